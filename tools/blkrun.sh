timeout 300 python -m pytest tests/test_gpu_block.py -x -q 2>&1 | tail -1
for e in 0 0u0 0 0u0; do
  HAPI_BLOCK=1 HAPI_LIB=abtest/libhapi_blk$e.so timeout 300 python tools/layer_profile.py resnet50_s21_b512 5 > gpurun_out/blk_exp$e.txt 2>&1
  echo "exp $e: $(head -1 gpurun_out/blk_exp$e.txt | cut -c1-80) | $(grep -h 'block\[layer1.1' gpurun_out/blk_exp$e.txt | cut -c1-30)"
done
