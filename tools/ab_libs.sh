#!/bin/bash
# Same-box A/B of library builds (abtest/libhapi_*.so, gitignored) on the ResNet-50 layer profile.
for r in 1 2; do
  for lib in D E; do
    HAPI_LIB=abtest/libhapi_$lib.so timeout 300 python tools/layer_profile.py resnet50_s21_b512 5 > gpurun_out/lp_lib_${lib}_$r.txt 2>&1
    echo "$lib : $(head -1 gpurun_out/lp_lib_${lib}_$r.txt) stem $(sed -n 4p gpurun_out/lp_lib_${lib}_$r.txt | awk '{print $2}')"
  done
done
