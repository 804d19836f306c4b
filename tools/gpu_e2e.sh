mkdir -p gpurun_out
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; echo "rc=$?" >> gpurun_out/e2e_probe.log
