mkdir -p gpurun_out
timeout 300 python tools/prof_kernels.py --factors 2,4,8 --reps 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_adjoint -o gpurun_out/prof_adjc -f python tools/prof_kernels.py --factors 2,4,8 --reps 1 > gpurun_out/ncu_adjc.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_adjc.log
