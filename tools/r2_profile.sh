#!/bin/bash
# One GPU call (round 2): GPU suite, bench lines for every workload, and per workload the ncu
# DRAM traffic of the dominant kernel class (profiles/traffic_<wl>.json, bench.py's
# roofline.traffic) -- each ncu pass only after the same workload's bench exited 0.
set -u
mkdir -p gpurun_out/r2p
tag=${1:-r2p}
for wl in resnet50_s21_b512 resnet18_s10_b200 densenet121_s9_b512 densenet121_s20_b512 vgg11_s21_b256 alexnet_s13_b8_f32 resnet50_s20_b512; do
  extra="--no-cpu-baseline"; [ $wl = resnet50_s21_b512 ] && extra=""
  timeout 600 python bench.py --workload $wl $extra > gpurun_out/r2p/bench_${tag}_$wl.json 2> gpurun_out/r2p/bench_${tag}_$wl.err || continue
  kern=conv_; [ $wl = alexnet_s13_b8_f32 ] && kern=conv_simt
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2p/traffic_$wl.csv python tools/prof_step.py $wl 1 > gpurun_out/r2p/ncu_t_$wl.log 2>&1 && \
    python tools/ncu_traffic.py gpurun_out/r2p/traffic_$wl.csv $wl $kern > gpurun_out/r2p/traffic_$wl.sum 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2p/launches_resnet50_s21_b512.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2p/ncu_l.log 2>&1
cp profiles/traffic_*.json gpurun_out/r2p/ 2>/dev/null
echo done
