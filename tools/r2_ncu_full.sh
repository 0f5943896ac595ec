#!/bin/bash
# ncu --set full captures (cold caches, serialized, one launch each) of the ResNet-50 s21 b512
# conv kernels: the stem+pool, stage-1/2 halo 3x3, pairs, stage-3 1x1/3x3.  Only after the
# same program exited 0 without ncu.  Reports land in gpurun_out/ncu/ (read here with
# ncu -i ... --page details / raw).
set -u
mkdir -p gpurun_out/ncu
tag=${1:-r2}
python tools/prof_step.py resnet50_s21_b512 1 > gpurun_out/ncu/ps.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_tc|conv_pair|conv_blk" \
  --launch-skip 0 --launch-count 14 -o gpurun_out/ncu/${tag}_s12 -f \
  python tools/prof_step.py resnet50_s21_b512 1 > gpurun_out/ncu/${tag}_s12.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_tc|conv_pair|conv_blk" \
  --launch-skip 17 --launch-count 6 -o gpurun_out/ncu/${tag}_s3 -f \
  python tools/prof_step.py resnet50_s21_b512 1 > gpurun_out/ncu/${tag}_s3.log 2>&1
ls -la gpurun_out/ncu
