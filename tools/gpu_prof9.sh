mkdir -p gpurun_out
timeout 300 python tools/prof_step.py --levels 5 > gpurun_out/prof_step_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_adjoint -c 2 -o gpurun_out/prof_adj1 -f python tools/prof_step.py --levels 5 > gpurun_out/ncu_adj1.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_adj1.log
