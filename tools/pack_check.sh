# Verify the swizzled pack_output tile: GPU parity tests, DenseNet121 s=9 layer profile and bench line
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -m gpu -x -q > gpurun_out/v13_pytest.log 2>&1; echo tests=$?; tail -2 gpurun_out/v13_pytest.log
python tools/layer_profile.py densenet121_s9_b512 5 > gpurun_out/lp_d9_v13.txt 2>&1
python tools/layer_profile.py resnet18_s10_b200 5 > gpurun_out/lp_r18_v13.txt 2>&1
for r in 1 2; do
python bench.py --workload densenet121_s9_b512 --no-cpu-baseline --no-e2e > gpurun_out/v13_bench_d9_$r.json 2>/dev/null
done
python bench.py --workload densenet121_s9_b512 > gpurun_out/v13_bench_d9.json 2>/dev/null
python bench.py --workload resnet18_s10_b200 > gpurun_out/v13_bench_r18.json 2>/dev/null
