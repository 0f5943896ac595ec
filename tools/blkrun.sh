timeout 900 python -m pytest tests/test_gpu_block.py -q -x 2>&1 | tail -3
for r in 1 2; do
for v in "HAPI_X=0" "HAPI_BLOCK_DS=0"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python tools/layer_profile.py resnet50_s21_b512 5 > gpurun_out/ds_$tag.txt 2>&1
  echo "$v : $(head -1 gpurun_out/ds_$tag.txt)"
done
done
grep -h "block\[layer1.0\|layer1.0" gpurun_out/ds_HAPI_X_0.txt | cut -c1-120
