# ncu --set full of the f=1 TMA forward on the full angle set (after a plain run)
mkdir -p gpurun_out
timeout 300 python tools/prof_kernels.py --factors 1,2 --reps 1 > gpurun_out/pf_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward_tma -c 2 -o gpurun_out/prof_fwd_full -f python tools/prof_kernels.py --factors 1,2 --reps 1 > gpurun_out/pf_ncu1.log 2>&1
echo "rc=$?" >> gpurun_out/pf_plain.log
