mkdir -p gpurun_out
set -x
timeout 600 python bench.py --steps 24 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 24 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1
echo "rc=$?"
