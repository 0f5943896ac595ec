#!/bin/bash
# Weak scaling (512 images per GPU) and the config-5 strong-scaling sets on N = 1, 2, 4 GPUs of
# one box, each N launched as the driver does; NCCL INIT lines go to stderr (nRanks check).
mkdir -p gpurun_out/scale
python paper_2210_08650_b200/build.py > /dev/null
for n in 1 2 4; do
  for wl in resnet50_s21_b512 resnet50_s21_64k densenet121_s9_64k; do
    if [ $n = 1 ]; then
      timeout 600 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/scale/${wl}_n$n.json 2> gpurun_out/scale/${wl}_n$n.err
    else
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29500 + n)) bench.py --gpus $n --workload $wl --no-cpu-baseline \
        > gpurun_out/scale/${wl}_n$n.json 2> gpurun_out/scale/${wl}_n$n.err
    fi
    python -c "
import json,sys
d=json.loads(open('gpurun_out/scale/${wl}_n$n.json').read().strip().splitlines()[-1])
print('$wl', $n, round(d['value']), (d.get('e2e') or {}).get('value'), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
" 2>&1 | tail -1
    grep -c "nRanks $n\|nranks $n" gpurun_out/scale/${wl}_n$n.err | sed "s/^/  nccl nRanks=$n lines: /"
  done
done
