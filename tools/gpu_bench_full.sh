mkdir -p gpurun_out
( time timeout 900 python bench.py ) > gpurun_out/bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/bench_default.log
( time timeout 900 python bench.py --impl reference ) > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
