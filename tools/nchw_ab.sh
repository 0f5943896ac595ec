# A/B: NCHW-storing last-conv epilogue vs NHWC store + split pack (HAPI_NCHW_EPI=0)
set -x
mkdir -p gpurun_out
HAPI_NCHW_EPI=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/v15_pytest_epi0.log 2>&1; echo tests=$?; tail -2 gpurun_out/v15_pytest_epi0.log
for r in 1 2; do
for wl in resnet50_s20_b512 resnet18_s10_b200; do
  python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/nab_on_${wl}_$r.json 2>/dev/null
  HAPI_NCHW_EPI=0 python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/nab_off_${wl}_$r.json 2>/dev/null
done
done
HAPI_NCHW_EPI=0 python tools/layer_profile.py resnet50_s20_b512 5 > gpurun_out/lp_r50s20_epi0.txt 2>&1
