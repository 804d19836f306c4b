mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-microbench > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
