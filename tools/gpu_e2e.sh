mkdir -p gpurun_out
for i in 1 2; do timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline >> gpurun_out/bench2.log 2>&1; done
