for i in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + i)) bench.py --gpus 4 --no-cpu-baseline 2> gpurun_out/s4_$i.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); e=d['e2e']; print(round(d['value']), round(e['value']), round(e['sync_per_step_value']), round(e['u8']['value']), e['host_cores'])"
done
