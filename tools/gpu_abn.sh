# A/B/N: the built library vs tools/variants/lib_<name>.so for each name given,
# phase times for each (two rounds), then the GPU projector tests on the first variant.
mkdir -p gpurun_out
L=paper_2412_10249_b200/libimask_b200.so
cp $L /tmp/lib_default.so
for round in 1 2; do
  for lib in /tmp/lib_default.so $(for v in "$@"; do echo tools/variants/lib_$v.so; done); do
    cp $lib $L
    echo "== $lib" >> gpurun_out/ab.log
    timeout 300 python tools/phase_times.py >> gpurun_out/ab.log 2>&1
  done
done
cp tools/variants/lib_$1.so $L
timeout 600 python -m pytest tests/test_gpu_projector.py tests/test_gpu_solver.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
cp /tmp/lib_default.so $L
