mkdir -p gpurun_out
for t in "" "1:7,2:7,4:7" "1:14,2:10,4:10" "1:28,2:24,4:24" "8:8,16:8,32:8" "8:32,16:32,32:32"; do
  echo "== IMASK_ADJ_CTAS=$t" >> gpurun_out/ctas.log
  IMASK_ADJ_CTAS=$t timeout 300 python tools/phase_times.py >> gpurun_out/ctas.log 2>&1
done
