# ncu --set full capture of the 2x2 pool and split-pack kernels (one launch each) after a clean run
set -x
mkdir -p gpurun_out
python tools/prof_step.py densenet121_s9_b512 1 > gpurun_out/ps_d9.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"pool2x2|pack_output_v8" -c 2 \
  -o gpurun_out/ncu_pool_pack_d9 python tools/prof_step.py densenet121_s9_b512 1 > gpurun_out/ncu_pp.log 2>&1
echo ncu=$?
python tools/prof_step.py vgg11_s21_b256 1 > gpurun_out/ps_vgg.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_vgg.csv \
  python tools/prof_step.py vgg11_s21_b256 1 > gpurun_out/ncu_lv.log 2>&1
echo ncu2=$?
