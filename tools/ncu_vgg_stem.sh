# ncu --set full capture of the VGG11 stem (+2x2 maxpool) launch
set -x
mkdir -p gpurun_out
python tools/prof_step.py vgg11_s21_b256 1 > gpurun_out/ps_vgg.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"conv_tc_kernel" -c 1 \
  -o gpurun_out/ncu_vgg_stem python tools/prof_step.py vgg11_s21_b256 1 > gpurun_out/ncu_vs.log 2>&1
echo ncu=$?
