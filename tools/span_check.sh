# Verify the span pack for HW % 8 != 0 splits: parity tests, layer profiles and bench lines
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -m gpu -x -q > gpurun_out/v14_pytest.log 2>&1; echo tests=$?; tail -2 gpurun_out/v14_pytest.log
python tools/layer_profile.py resnet50_s20_b512 5 > gpurun_out/lp_r50s20_v14.txt 2>&1
python tools/layer_profile.py vgg11_s21_b256 5 > gpurun_out/lp_vgg_v14.txt 2>&1
python bench.py --workload resnet50_s20_b512 --no-cpu-baseline > gpurun_out/v14_bench_r50s20.json 2>/dev/null
python bench.py --workload vgg11_s21_b256 > gpurun_out/v14_bench_vgg.json 2>/dev/null
python bench.py > gpurun_out/v14_bench_r50.json 2>/dev/null
