#!/bin/bash
# Same-box A/B of the ResNet-50 layer profile across library versions (abtest/<commit> trees,
# gitignored, built in place) and the current tree, two alternating rounds.
for r in 1 2; do
  for c in e418590 b349825; do
    (cd abtest/$c && timeout 300 python tools/layer_profile.py resnet50_s21_b512 5 > ../../gpurun_out/lp_ab_${c}_$r.txt 2>&1)
    head -1 gpurun_out/lp_ab_${c}_$r.txt
  done
  timeout 300 python tools/layer_profile.py resnet50_s21_b512 5 > gpurun_out/lp_ab_head_$r.txt 2>&1
  head -1 gpurun_out/lp_ab_head_$r.txt
done
