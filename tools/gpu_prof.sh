mkdir -p gpurun_out
set -x
timeout 600 python tools/prof_kernels.py --factors 1 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_adjoint|k_forward" -c 4 -o gpurun_out/prof_f1 -f python tools/prof_kernels.py --factors 1 --reps 2 > gpurun_out/ncu_f1.log 2>&1
echo "ncu rc=$?"
timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
