mkdir -p gpurun_out
L=paper_2412_10249_b200/libimask_b200.so
cp $L /tmp/lib_default.so
for round in 1 2; do
for lib in /tmp/lib_default.so tools/variants/lib_f1mb4.so tools/variants/lib_adj8.so tools/variants/lib_both.so; do
  cp $lib $L
  echo "== $lib" >> gpurun_out/ab.log
  timeout 300 python tools/phase_times.py 2>&1 | grep -E "f=  [12] " >> gpurun_out/ab.log
  timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-microbench --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['per_level_ms'])" >> gpurun_out/ab.log
done
done
cp /tmp/lib_default.so $L
