set -x
python paper_2210_08650_b200/build.py
./tools/micro/mma_rate2 > gpurun_out/mma_rate2.txt 2>&1; cat gpurun_out/mma_rate2.txt
./tools/micro/mma_rate > gpurun_out/mma_rate.txt 2>&1; head -8 gpurun_out/mma_rate.txt
for v in 1 0 1 0; do HAPI_STEM_SEG=$v timeout 300 python tools/layer_profile.py resnet50_s21_b512 5 > gpurun_out/lp_r2e_seg$v.txt 2>&1; sed -n 1p gpurun_out/lp_r2e_seg$v.txt; sed -n 4p gpurun_out/lp_r2e_seg$v.txt; done
timeout 900 python -m pytest tests/test_gpu_fusion_bits.py tests/test_gpu_suffix.py tests/test_gpu_server.py -q -p no:cacheprovider > gpurun_out/pytest_r2e.log 2>&1; tail -3 gpurun_out/pytest_r2e.log
timeout 300 python bench.py --workload densenet121_s9_b512 --no-cpu-baseline > gpurun_out/bench_r2e_d9.json 2>/dev/null; tail -c 300 gpurun_out/bench_r2e_d9.json
bash tools/sanitize.sh
