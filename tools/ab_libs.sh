#!/bin/bash
# Same-box A/B of library builds (abtest/libhapi_*.so, gitignored) on the ResNet-50 layer profile.
for r in 1 2; do
  for v in "A" "C HAPI_DUAL_M256=0" "C"; do
    set -- $v; lib=$1; shift
    env HAPI_LIB=abtest/libhapi_$lib.so "$@" timeout 300 python tools/layer_profile.py resnet50_s21_b512 5 > gpurun_out/lp_lib_${lib}_${1:-def}_$r.txt 2>&1
    echo "$lib $* : $(head -1 gpurun_out/lp_lib_${lib}_${1:-def}_$r.txt)"
  done
done
