#!/bin/bash
# Round-2 closing verification at the final tree (one GPU call): full GPU suite, smoke(), the
# default bench line (cpu_baseline + e2e) and the reference (oracle) arm, bench lines + DRAM
# traffic of the dominant class for every workload, the ResNet-50 launch list under ncu, and an
# ncu --set full capture of the ResNet-50 conv launches through stage 2 (stem, blocks, pairs).
# Every ncu pass runs only after the same program exited 0 without ncu.
set -u
mkdir -p gpurun_out/fin gpurun_out/ncu
python paper_2210_08650_b200/build.py > /dev/null
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/fin/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin/smoke.log 2>&1; tail -1 gpurun_out/fin/smoke.log
timeout 600 python bench.py > gpurun_out/fin/bench_resnet50_s21_b512.json 2> gpurun_out/fin/bench_resnet50_s21_b512.err
tail -c 300 gpurun_out/fin/bench_resnet50_s21_b512.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin/ref.json 2> gpurun_out/fin/ref.err; tail -c 200 gpurun_out/fin/ref.json
for wl in resnet18_s10_b200 densenet121_s9_b512 densenet121_s20_b512 vgg11_s21_b256 alexnet_s13_b8_f32 resnet50_s20_b512 resnet50_s21_b512; do
  if [ $wl != resnet50_s21_b512 ]; then
    timeout 600 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/fin/bench_$wl.json 2> gpurun_out/fin/bench_$wl.err || continue
  fi
  kern=conv_; [ $wl = alexnet_s13_b8_f32 ] && kern=conv_simt
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/fin/traffic_$wl.csv python tools/prof_step.py $wl 1 > gpurun_out/fin/ncu_t_$wl.log 2>&1 && \
    python tools/ncu_traffic.py gpurun_out/fin/traffic_$wl.csv $wl $kern > gpurun_out/fin/traffic_$wl.sum 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin/launches_resnet50_s21_b512.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin/ncu_l.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"conv_tc|conv_pair|conv_block" \
  --launch-skip 0 --launch-count 16 -o gpurun_out/ncu/fin_r50 -f \
  python tools/prof_step.py resnet50_s21_b512 1 > gpurun_out/ncu/fin_r50.log 2>&1
cp profiles/traffic_*.json gpurun_out/fin/ 2>/dev/null
ls gpurun_out/fin | wc -l
echo done
