# Round profile set: plain bench, launch list of the same bench command, full ncu of
# the f=1 forward and adjoint (the dominant kernels). Outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 60 --warmup 6 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 60 --warmup 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
timeout 600 python tools/prof_kernels.py --factors 1 --reps 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_adjoint$|k_forward" -c 2 \
  -o gpurun_out/prof_f1 -f python tools/prof_kernels.py --factors 1 --reps 1 > gpurun_out/ncu_f1.log 2>&1
echo "ncu rc=$?"
