mkdir -p gpurun_out
for v in 8 1 4 2; do
  echo "== IMASK_ADJ_CLUSTER=$v" >> gpurun_out/phase_cl.log
  IMASK_ADJ_CLUSTER=$v timeout 300 python tools/phase_times.py >> gpurun_out/phase_cl.log 2>&1
done
bash tools/gpu_bench_env.sh IMASK_ADJ_CLUSTER=8 IMASK_ADJ_CLUSTER=1 IMASK_ADJ_CLUSTER=4
