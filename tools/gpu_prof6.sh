mkdir -p gpurun_out
timeout 600 python tools/prof_kernels.py --factors 1,2 --reps 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k k_adjoint -c 4 -o gpurun_out/prof_adj -f python tools/prof_kernels.py --factors 1,2 --reps 1 > gpurun_out/ncu_adj.log 2>&1
echo "ncu rc=$?"
