mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --gpus 1 --steps 20 --warmup 5 --no-microbench --no-cpu-baseline > gpurun_out/b20.log 2>&1
