mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/repro_subset.py 1024 1440 1449 6 1 2 5 17 44 89 120 150 179 211 250 301 333 358 359 > gpurun_out/subset.log 2>&1; echo "rc=$?" >> gpurun_out/subset.log
timeout 1500 python -m pytest tests/test_gpu_parity_large.py tests/test_gpu_dropin.py -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
