"""Throughput of one 512-image forward when the library executes it in chunks of
max_batch images through a small (L2-resident) arena.  Usage: chunk_sweep.py [workload]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import hapi_inputs  # noqa: E402
import paper_2210_08650_b200 as H  # noqa: E402
from bench import WORKLOADS  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "resnet50_s21_b512"
arch, act, split, batch, seed = WORKLOADS[wl]
P = list(hapi_inputs.params(arch, 1000 + seed).values())
x = torch.from_numpy(hapi_inputs.images(batch, seed)).cuda()
for mb in [int(v) for v in (sys.argv[2:] or ["16", "32", "64", "128", "256", "512"])]:
    m = H.Model(arch, act, P, mb, split, split)
    st = torch.cuda.current_stream()
    m.set_stream(st.cuda_stream)
    es = 4 if act == "f32" else 2
    out = torch.empty(m.out_bytes[split - 1] // es * batch, dtype=torch.float32 if act == "f32" else torch.bfloat16,
                      device="cuda")
    for _ in range(3):
        m.forward(split, x, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record(st)
    for _ in range(n):
        m.forward(split, x, out)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{wl} max_batch={mb:4d}: {ms:.3f} ms per {batch} images -> {batch / ms * 1e3:.0f} img/s, "
          f"arena {m.device_bytes()[1] / 2**20:.0f} MiB", flush=True)
    m.close()
