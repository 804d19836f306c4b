# A/B of an environment switch ("VAR" with values given) on phase times at world 1
# and on 2-, 4- and 8-way shard ranks, then the forward bit-identity check and the
# projector / solver GPU tests with the default setting.
mkdir -p gpurun_out
VAR=$1; shift
for v in "$@"; do
  for wr in ${WORLDS:-1:0 2:0 4:0 8:0}; do
    set -- ${wr/:/ }
    echo "== $VAR=$v world $1 rank $2" >> gpurun_out/abe.log
    env $VAR=$v timeout 300 python tools/phase_times.py --world $1 --rank $2 >> gpurun_out/abe.log 2>&1
  done
done
[ -n "$NOTEST" ] && exit 0
timeout 600 python tools/dbg_fwd.py > gpurun_out/dbg.log 2>&1
timeout 600 python -m pytest tests/test_gpu_projector.py tests/test_gpu_solver.py -m gpu -q -x -p no:cacheprovider > gpurun_out/abe_tests.log 2>&1; echo "rc=$?" >> gpurun_out/abe_tests.log
