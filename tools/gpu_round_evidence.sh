# Round evidence: GPU tests, smoke, the default bench and the reference arm, then
# the launch list and one ncu --set full capture (each after its plain run exited 0).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
( time timeout 900 python bench.py ) > gpurun_out/bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/bench_default.log
( time timeout 900 python bench.py --impl reference ) > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 300 python tools/phase_times.py > gpurun_out/phase.log 2>&1
timeout 600 python bench.py --steps 24 --warmup 3 --steps-only > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 24 --warmup 3 --steps-only > gpurun_out/ncu.log 2>&1
echo "launches rc=$?" >> gpurun_out/plain.log
timeout 300 python tools/prof_step.py > gpurun_out/prof_step_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:k_forward|k_adjoint|k_saga_image|k_prepare|k_compensate|k_restrict' -o gpurun_out/prof_step -f python tools/prof_step.py > gpurun_out/ncu_step.log 2>&1
echo "full rc=$?" >> gpurun_out/prof_step_plain.log
