# Multi-GPU weak/strong scaling on one box (run under gpurun --gpus 4)
set -x
nvidia-smi -L
for N in 1 2 4; do
  if [ $N = 1 ]; then
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_w_n$N.json 2> gpurun_out/bench_w_n$N.err
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_w_n$N.json 2> gpurun_out/bench_w_n$N.err
  fi
  echo W$N $?; cut -c1-160 gpurun_out/bench_w_n$N.json
done
for N in 1 2 4; do
  if [ $N = 1 ]; then
    timeout 300 python bench.py --workload resnet50_s21_64k --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s_n$N.json 2> gpurun_out/bench_s_n$N.err
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --workload resnet50_s21_64k --steps 5 --warmup 3 > gpurun_out/bench_s_n$N.json 2> gpurun_out/bench_s_n$N.err
  fi
  echo S$N $?; cut -c1-160 gpurun_out/bench_s_n$N.json
done
for N in 1 2 4; do
  if [ $N = 1 ]; then
    timeout 300 python bench.py --workload densenet121_s9_64k --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_d_n$N.json 2> gpurun_out/bench_d_n$N.err
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --workload densenet121_s9_64k --steps 5 --warmup 3 > gpurun_out/bench_d_n$N.json 2> gpurun_out/bench_d_n$N.err
  fi
  echo D$N $?; cut -c1-160 gpurun_out/bench_d_n$N.json
done
