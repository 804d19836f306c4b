mkdir -p gpurun_out
for g in "1024 1440 1449 1" "256 360 363 1" "256 360 363 2"; do
  echo "== $g" >> gpurun_out/rq.log
  OUT=gpurun_out/q.npy timeout 120 python tools/repro_quad.py $g >> gpurun_out/rq.log 2>&1; echo "quad rc=$?" >> gpurun_out/rq.log
  IMASK_NO_QUAD=1 OUT=gpurun_out/p.npy timeout 120 python tools/repro_quad.py $g >> gpurun_out/rq.log 2>&1; echo "pair rc=$?" >> gpurun_out/rq.log
  python -c "import numpy as np; a=np.load('gpurun_out/q.npy'); b=np.load('gpurun_out/p.npy'); print('rel', np.linalg.norm(a-b)/np.linalg.norm(b))" >> gpurun_out/rq.log 2>&1
done
