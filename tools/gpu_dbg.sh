mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_projector.py -q -x -p no:cacheprovider --timeout 300 -k "row_pairs or config_A or config_D or against_oracle" > gpurun_out/pytest_rp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rp.log
for v in 1 0; do echo "== ROW_PAIR=$v" >> gpurun_out/phase_rp.log; IMASK_ADJ_ROW_PAIR=$v timeout 300 python tools/phase_times.py 2>&1 | grep "f=  1" >> gpurun_out/phase_rp.log; IMASK_ADJ_ROW_PAIR=$v timeout 300 python tools/phase_times.py --world 8 --rank 0 2>&1 | grep "f=  1" >> gpurun_out/phase_rp.log; done
bash tools/gpu_bench_env.sh - IMASK_ADJ_ROW_PAIR=0
