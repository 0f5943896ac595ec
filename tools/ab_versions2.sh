#!/bin/bash
for r in 1 2; do
  for c in e8dd633 3066285 e418590; do
    (cd abtest/$c && timeout 300 python tools/layer_profile.py resnet50_s21_b512 5 > ../../gpurun_out/lp_ab2_${c}_$r.txt 2>&1)
    echo "$c $(head -1 gpurun_out/lp_ab2_${c}_$r.txt) $(grep 'layer3.1.conv2' gpurun_out/lp_ab2_${c}_$r.txt | awk '{print $2}')"
  done
done
