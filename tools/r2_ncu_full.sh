#!/bin/bash
# ncu --set full captures (cold caches, serialized, one launch each) of the ResNet-50 s21 b512
# conv kernels from the stem through stage 3's first identity block, at the current build.
# Only after the same program exited 0 without ncu.  Reports land in gpurun_out/ncu/.
set -u
mkdir -p gpurun_out/ncu
tag=${1:-r2}
python tools/prof_step.py resnet50_s21_b512 1 > gpurun_out/ncu/ps.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"conv_tc|conv_pair" \
  --launch-skip 0 --launch-count 24 -o gpurun_out/ncu/${tag}_r50 -f \
  python tools/prof_step.py resnet50_s21_b512 1 > gpurun_out/ncu/${tag}_r50.log 2>&1
ls -la gpurun_out/ncu
