mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/prof_kernels.py --factors 1,2,4,8 --reps 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_adjoint$|k_forward" -c 8 -o gpurun_out/prof_all -f python tools/prof_kernels.py --factors 1,2,4,8 --reps 1 > gpurun_out/ncu_all.log 2>&1
echo "ncu rc=$?"
timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
