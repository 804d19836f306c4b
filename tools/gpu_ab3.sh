mkdir -p gpurun_out
L=paper_2412_10249_b200/libimask_b200.so
cp $L /tmp/lib_default.so
for lib in /tmp/lib_default.so tools/variants/lib_e8w96.so tools/variants/lib_e16w96.so tools/variants/lib_e16w72.so /tmp/lib_default.so; do
  cp $lib $L
  echo "== $lib" >> gpurun_out/ab.log
  timeout 300 python tools/phase_times.py >> gpurun_out/ab.log 2>&1
done
cp /tmp/lib_default.so $L
