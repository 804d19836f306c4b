# A/B of library variants: runs "$CMD" with the default library and each tools/variants/lib_NAME.so
# usage: CMD="python tools/image_probe.py" bash tools/gpu_ab_libs.sh NAME...
mkdir -p gpurun_out
L=paper_2412_10249_b200/libimask_b200.so
cp $L /tmp/lib_default.so
for round in 1 2; do
for name in default "$@"; do
  if [ $name = default ]; then cp /tmp/lib_default.so $L; else cp tools/variants/lib_$name.so $L; fi
  echo "== $name (round $round)" >> gpurun_out/ab.log
  timeout 600 $CMD >> gpurun_out/ab.log 2>&1
done
done
cp /tmp/lib_default.so $L
