# A/B/N with shard phase times: the built library vs tools/variants/lib_<name>.so
# for each name given, at world 1 and at ranks of 8- and 4-way angle shards.
mkdir -p gpurun_out
L=paper_2412_10249_b200/libimask_b200.so
cp $L /tmp/lib_default.so
for lib in /tmp/lib_default.so $(for v in "$@"; do echo tools/variants/lib_$v.so; done); do
  cp $lib $L
  for wr in "1 0" "8 0" "8 7" "4 0"; do
    set -- $wr
    echo "== $lib world $1 rank $2" >> gpurun_out/abs.log
    timeout 300 python tools/phase_times.py --world $1 --rank $2 >> gpurun_out/abs.log 2>&1
  done
done
cp /tmp/lib_default.so $L
timeout 600 python -m pytest tests/test_gpu_projector.py tests/test_gpu_solver.py -m gpu -q -x -p no:cacheprovider > gpurun_out/abs_tests.log 2>&1; echo "rc=$?" >> gpurun_out/abs_tests.log
