mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_projector.py tests/test_gpu_solver.py -q -x -p no:cacheprovider --timeout 400 -k "bit_identical or fused_staging" --durations=10 > gpurun_out/pytest_fs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fs.log
