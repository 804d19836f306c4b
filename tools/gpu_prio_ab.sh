# A/B of the step DAG's stream priorities (IMASK_PRIO) on the default bench.
bash tools/gpu_bench_env.sh - IMASK_PRIO=1 IMASK_PRIO=2
timeout 600 env IMASK_PRIO=2 python -m pytest tests/test_gpu_solver.py -m gpu -x -q > gpurun_out/prio_pytest.log 2>&1
