mkdir -p gpurun_out
timeout 600 python tools/prof_kernels.py --factors 32,8 --reps 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -c 30 -o gpurun_out/prof_coarse2 -f python tools/prof_kernels.py --factors 32,8 --reps 1 > gpurun_out/ncu_coarse2.log 2>&1
echo "ncu rc=$?"
