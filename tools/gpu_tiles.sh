mkdir -p gpurun_out
for t in "" "8:16,16:16,32:16" "8:16,16:32,32:32" "4:32,8:32" "2:16,4:8"; do
  echo "== IMASK_ADJ_TILE=$t" >> gpurun_out/tiles.log
  IMASK_ADJ_TILE=$t timeout 300 python tools/phase_times.py >> gpurun_out/tiles.log 2>&1
done
