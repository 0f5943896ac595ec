# A/B: VGG11 stem (mode 4 + 2x2 pool epilogue) with pipelined TMEM loads and constant-bank bias
for L in abtest/libhapi_base.so paper_2210_08650_b200/libhapi.so; do
  HAPI_LIB=$L timeout 300 python tools/outhash.py vgg11_s21_b256 2>&1 | tail -2
done
for r in 1 2; do for L in abtest/libhapi_base.so paper_2210_08650_b200/libhapi.so; do
  echo "$L"; HAPI_LIB=$L timeout 300 python tools/layer_profile.py vgg11_s21_b256 10 2>&1 | sed -n '1p;4p'
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_u8.py tests/test_gpu_fusion_bits.py -q -k "vgg" 2>&1 | tail -1
