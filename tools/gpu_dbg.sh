mkdir -p gpurun_out
timeout 300 python tools/phase_times.py > gpurun_out/phase.log 2>&1
bash tools/gpu_bench_env.sh - -
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
