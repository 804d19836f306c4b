# Sweep adjoint build variants (launch-bounds min blocks) x window caps with short benches.
mkdir -p gpurun_out
L=paper_2412_10249_b200/libimask_b200.so
cp $L /tmp/lib_default.so
for lib in /tmp/lib_default.so tools/variants/lib_minb7.so tools/variants/lib_minb8.so; do
  cp $lib $L
  for kb in 40 20; do
    echo "== $lib kb=$kb" >> gpurun_out/variants.log
    IMASK_ADJ_WIN_KB=$kb timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/variants.log 2>&1
  done
done
cp /tmp/lib_default.so $L
