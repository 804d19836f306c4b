mkdir -p gpurun_out
for t in 129 64 32; do
  echo "== IMASK_TMA_MIN_N=$t" >> gpurun_out/tma_n.log
  IMASK_TMA_MIN_N=$t timeout 300 python tools/phase_times.py >> gpurun_out/tma_n.log 2>&1
done
