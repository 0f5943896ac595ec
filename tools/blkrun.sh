timeout 900 python -m pytest tests/test_gpu_strong_subset.py tests/test_gpu_u8.py -q 2>&1 | tail -3
timeout 600 python bench.py --workload resnet50_s21_64k --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), d['parity_subset'])"
