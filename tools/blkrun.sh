mkdir -p gpurun_out/ncu
timeout 300 python tools/prof_step.py vgg11_s21_b256 1 > gpurun_out/ncu/psv.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_tc" --launch-skip 0 --launch-count 1 \
  -o gpurun_out/ncu/vggstem -f python tools/prof_step.py vgg11_s21_b256 1 > gpurun_out/ncu/vggstem.log 2>&1
tail -1 gpurun_out/ncu/vggstem.log
