#!/bin/bash
# Final check after the last kernel change: full GPU suite, smoke(), bench lines for the default
# workload and VGG11, and the ncu launch list of the VGG11 bench command.
set -u
mkdir -p gpurun_out/fin2
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin2/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/fin2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin2/smoke.log 2>&1; tail -1 gpurun_out/fin2/smoke.log
timeout 600 python bench.py > gpurun_out/fin2/bench_resnet50_s21_b512.json 2> gpurun_out/fin2/bench_resnet50_s21_b512.err
timeout 600 python bench.py --workload vgg11_s21_b256 --no-cpu-baseline > gpurun_out/fin2/bench_vgg11_s21_b256.json 2> gpurun_out/fin2/bench_vgg11_s21_b256.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin2/launches_vgg11_s21_b256.csv \
  python bench.py --workload vgg11_s21_b256 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin2/ncu_l.log 2>&1
echo done
