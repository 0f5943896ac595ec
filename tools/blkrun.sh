timeout 900 python -m pytest tests/test_gpu_fusion_bits.py -q -k "DUAL_M32 or DUAL_M-" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "densenet" 2>&1 | tail -1
for wl in densenet121_s20_b512 densenet121_s9_b512; do
for v in "HAPI_X=0" "HAPI_DUAL_M32=0"; do
  env $v timeout 300 python tools/layer_profile.py $wl 5 > gpurun_out/dm32.txt 2>&1
  echo "$v: $(head -1 gpurun_out/dm32.txt | cut -c1-80)"
done
done
