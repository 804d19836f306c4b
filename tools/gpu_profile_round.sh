# Evidence for profiles/: bench launch list + one ncu --set full capture of a step's kernels.
mkdir -p gpurun_out
set -x
timeout 600 python bench.py --steps 24 --warmup 3 --steps-only > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 24 --warmup 3 --steps-only > gpurun_out/ncu.log 2>&1
echo "launches rc=$?"
timeout 300 python tools/prof_step.py > gpurun_out/prof_step_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:k_forward|k_adjoint|k_saga_image|k_prepare|k_compensate|k_restrict' -o gpurun_out/prof_step -f python tools/prof_step.py > gpurun_out/ncu_step.log 2>&1
echo "full rc=$?"
