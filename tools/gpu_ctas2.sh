mkdir -p gpurun_out
for t in "16:2,32:2" "16:3,32:3" "16:4,32:4" "16:6,32:6" "4:8,2:12"; do
  echo "== IMASK_ADJ_CTAS=$t" >> gpurun_out/ctas.log
  IMASK_ADJ_CTAS=$t timeout 300 python tools/phase_times.py >> gpurun_out/ctas.log 2>&1
done
