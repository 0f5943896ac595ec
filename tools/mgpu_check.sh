set -x
nvidia-smi -L
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo N2_EXIT $?
cat gpurun_out/bench_n2.json; tail -3 gpurun_out/bench_n2.err
timeout 300 python bench.py --workload resnet50_s21_64k --steps 10 --warmup 3 > gpurun_out/bench_64k_n1.json 2> gpurun_out/bench_64k_n1.err; echo S1_EXIT $?
cat gpurun_out/bench_64k_n1.json; tail -3 gpurun_out/bench_64k_n1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --workload resnet50_s21_64k --steps 10 --warmup 3 > gpurun_out/bench_64k_n2.json 2> gpurun_out/bench_64k_n2.err; echo S2_EXIT $?
cat gpurun_out/bench_64k_n2.json; tail -3 gpurun_out/bench_64k_n2.err
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_n2.json 2> gpurun_out/bench_ref_n2.err; echo R2_EXIT $?
cut -c1-200 gpurun_out/bench_ref_n2.json
