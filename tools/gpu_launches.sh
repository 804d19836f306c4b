mkdir -p gpurun_out
timeout 600 python bench.py --steps 24 --warmup 3 --steps-only > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 24 --warmup 3 --steps-only > gpurun_out/ncu.log 2>&1
echo "launches rc=$?" >> gpurun_out/plain.log
