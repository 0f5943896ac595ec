# A/B: VGG11 stem pool epilogue: tile coordinates carried forward (no per-tile divisions)
for L in abtest/libhapi_base.so paper_2210_08650_b200/libhapi.so; do
  HAPI_LIB=$L timeout 300 python tools/outhash.py vgg11_s21_b256 2>&1 | tail -2
done
for r in 1 2; do for L in abtest/libhapi_base.so paper_2210_08650_b200/libhapi.so; do
  echo "$L"; HAPI_LIB=$L timeout 300 python tools/layer_profile.py vgg11_s21_b256 10 2>&1 | sed -n '1p;4p'
done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_u8.py tests/test_gpu_fusion_bits.py tests/test_gpu_large_inputs.py -q -x -k "vgg or u8" 2>&1 | tail -1
