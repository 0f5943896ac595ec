timeout 900 python -m pytest tests/test_gpu_block.py -q 2>&1 | tail -3
