mkdir -p gpurun_out
L=paper_2412_10249_b200/libimask_b200.so
cp $L /tmp/lib_default.so
for round in 1 2; do
for lib in tools/variants/lib_k4mb3.so tools/variants/lib_k4mb2.so; do
  cp $lib $L
  for v in 4 2; do
    echo "== $lib TWO_DET=$v" >> gpurun_out/ab.log
    IMASK_FWD_TWO_DET=$v timeout 300 python tools/phase_times.py 2>&1 | grep -E "f=  [48]|f= 16" >> gpurun_out/ab.log
  done
done
done
cp tools/variants/lib_k4mb3.so $L
timeout 900 python -m pytest tests/test_gpu_projector.py -q -x -p no:cacheprovider --timeout 400 -k "bit_identical or sampled or config_A" > gpurun_out/pytest_bi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bi.log
cp /tmp/lib_default.so $L
