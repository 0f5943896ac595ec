#!/bin/bash
# Closing verification: full GPU suite, smoke(), default bench line (cpu_baseline + e2e), the
# reference (oracle) arm, per-workload bench lines, and the ResNet-50 launch list under ncu.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin_pytest.log 2>&1; echo tests=$?; tail -2 gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
timeout 600 python bench.py > gpurun_out/fin_bench_r50.json 2> gpurun_out/fin_bench_r50.err; tail -c 600 gpurun_out/fin_bench_r50.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_ref.json 2>&1
for wl in resnet18_s10_b200 densenet121_s9_b512 vgg11_s21_b256 resnet50_s20_b512; do
  timeout 300 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/fin_bench_$wl.json 2> /dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin_ncu_l.log 2>&1
echo done
