timeout 900 python -m pytest tests/test_gpu_fusion_bits.py -q -k "DUAL_M_PRO or DUAL_M32" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_suffix.py tests/test_gpu_large_inputs.py -q -k "densenet" 2>&1 | tail -1
timeout 300 python tools/layer_profile.py densenet121_s9_b512 5 2>&1 | head -1
