mkdir -p gpurun_out
for wr in "8 0" "4 0" "2 0" "1 0"; do
  set -- $wr
  for v in "IMASK_FWD_TWO_DET_MIN_WAVES=6" "IMASK_FWD_TWO_DET_MIN_WAVES=3" "IMASK_FWD_TWO_DET_MIN_WAVES=0"; do
    echo "== world $1 rank $2 $v" >> gpurun_out/shard_2d.log
    env $v timeout 300 python tools/phase_times.py --world $1 --rank $2 2>&1 | grep -E "f=  [248] " >> gpurun_out/shard_2d.log
  done
done
