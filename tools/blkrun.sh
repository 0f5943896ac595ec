timeout 1500 python -m pytest tests/test_gpu_large_inputs.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 800 python tools/size_sweep.py 2>&1 | tee gpurun_out/size_sweep.txt
