# bench.py (100 steps, device-timed, L2 flushed) under environment settings given
# as arguments ("-" = none), twice each, in interleaved order.
mkdir -p gpurun_out
for round in 1 2; do
  for e in "$@"; do
    echo "== $e" >> gpurun_out/bench_env.log
    if [ "$e" = "-" ]; then envs=""; else envs="$e"; fi
    env $envs timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-microbench --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['per_level_ms'])" >> gpurun_out/bench_env.log
  done
done
