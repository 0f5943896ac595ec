timeout 900 python -m pytest tests/test_gpu_block.py -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python tools/race_check.py resnet50 21 512 20 2>&1 | tail -3
