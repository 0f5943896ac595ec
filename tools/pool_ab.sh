set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fusion_bits.py -k "POOL_GENERIC" tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pool_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/pool_tests.log
for r in 1 2; do
  HAPI_POOL_GENERIC=1 python bench.py --workload vgg11_s21_b256 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pab_gen_$r.json 2>/dev/null
  python bench.py --workload vgg11_s21_b256 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pab_new_$r.json 2>/dev/null
  HAPI_POOL_GENERIC=1 python bench.py --workload densenet121_s20_b512 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pab_dgen_$r.json 2>/dev/null
  python bench.py --workload densenet121_s20_b512 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pab_dnew_$r.json 2>/dev/null
done
python tools/layer_profile.py vgg11_s21_b256 5 > gpurun_out/lp_vgg_new.txt 2>&1
HAPI_POOL_GENERIC=1 python tools/layer_profile.py vgg11_s21_b256 5 > gpurun_out/lp_vgg_gen.txt 2>&1
python bench.py --workload vgg11_s21_b256 > gpurun_out/v11_bench_vgg.json 2>/dev/null
python bench.py > gpurun_out/v11_bench_r50.json 2>/dev/null
