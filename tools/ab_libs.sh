#!/bin/bash
# Same-box A/B of switches on the ResNet-50 layer profile (current build).
for r in 1 2; do
  for v in "HAPI_BLOCK=0" "HAPI_BLOCK=1"; do
    tag=$(echo $v | tr ' =' '__')
    env $v timeout 300 python tools/layer_profile.py resnet50_s21_b512 5 > gpurun_out/lp_sw_${tag}_$r.txt 2>&1
    echo "$v : $(head -1 gpurun_out/lp_sw_${tag}_$r.txt)"
  done
done
