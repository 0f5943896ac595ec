# Verify the batched-load adaptive avgpool: GPU parity + determinism tests, ResNet50 layer profile and bench line
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/v12_pytest.log 2>&1; echo tests=$?; tail -2 gpurun_out/v12_pytest.log
python tools/layer_profile.py resnet50_s21_b512 5 > gpurun_out/lp_r50_v12.txt 2>&1
python bench.py > gpurun_out/v12_bench_r50.json 2>gpurun_out/v12_bench_r50.err
python bench.py --workload densenet121_s20_b512 --no-cpu-baseline > gpurun_out/v12_bench_d20.json 2>/dev/null
