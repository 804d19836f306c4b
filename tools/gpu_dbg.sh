mkdir -p gpurun_out
timeout 800 python tools/shard_probe.py > gpurun_out/shard_probe.log 2>&1
for wr in "8 0" "8 7" "4 0" "1 0"; do set -- $wr; echo "== world $1 rank $2" >> gpurun_out/phase_shards.log; timeout 300 python tools/phase_times.py --world $1 --rank $2 >> gpurun_out/phase_shards.log 2>&1; done
