mkdir -p gpurun_out
bash tools/gpu_bench_env.sh - IMASK_FWD_TWO_DET=0
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
