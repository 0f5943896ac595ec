timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_fusion_bits.py -q -x -k "DUAL_M" 2>&1 | tail -1
for wl in resnet18_s10_b200 resnet50_s21_b512 resnet50_s20_b512; do
  timeout 300 python tools/layer_profile.py $wl 5 > gpurun_out/halo.txt 2>&1
  echo "$wl: $(head -1 gpurun_out/halo.txt | cut -c1-80)"
done
