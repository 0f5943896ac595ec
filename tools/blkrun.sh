timeout 900 python -m pytest tests/test_gpu_u8.py -q 2>&1 | tail -5
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_u8.json 2> gpurun_out/bench_u8.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_u8.json').read().strip().splitlines()[-1]); e=d['e2e']
print(round(d['value']), round(e['value']), round(e['sync_per_step_value']), round(e['u8']['value']), e['u8']['h2d_bytes_per_step'])"
