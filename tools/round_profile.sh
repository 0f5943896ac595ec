#!/bin/bash
# One GPU call: bench lines for every workload, the ResNet-50 ncu launch list and per-launch
# DRAM traffic (each ncu pass only after the same command exited 0 without ncu).
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err || exit 1
for wl in resnet18_s10_b200 densenet121_s9_b512 densenet121_s20_b512 vgg11_s21_b256 alexnet_s13_b8_f32 resnet50_s20_b512; do
  python bench.py --workload $wl --no-cpu-baseline > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l.log 2>&1
python tools/prof_step.py resnet50_s21_b512 1 > gpurun_out/ps.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/traffic.csv python tools/prof_step.py resnet50_s21_b512 1 > gpurun_out/ncu_t.log 2>&1
echo done
