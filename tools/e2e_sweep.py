"""End-to-end (pinned host buffers in and out) throughput of the host-buffer calls for several
staging chunk sizes (desc.host_chunk): a stream of requests through
hapi_prefix_forward_host_async + one hapi_host_sync, and the synchronous call per request.
Usage: e2e_sweep.py [workload] [chunks...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import hapi_inputs  # noqa: E402
import paper_2210_08650_b200 as H  # noqa: E402
from bench import WORKLOADS  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "resnet50_s21_b512"
chunks = [int(c) for c in sys.argv[2:]] or [96, 128, 176, 256, 512]
arch, act, split, batch, seed = WORKLOADS[wl]
P = list(hapi_inputs.params(arch, 1000 + seed).values())
xs = [torch.from_numpy(hapi_inputs.images(batch, seed)).pin_memory() for _ in range(2)]
es = 4 if act == "f32" else 2
for c in chunks:
    m = H.Model(arch, act, P, batch, split, split, host_chunk=c)
    os_ = [torch.empty(m.out_bytes[split - 1] // es * batch, dtype=torch.float32 if act == "f32" else torch.bfloat16)
           .pin_memory() for _ in range(2)]
    for i in range(3):
        m.forward_host(split, xs[i & 1], os_[i & 1])
    n = 10
    t0 = time.perf_counter()
    for i in range(n):
        m.forward_host_async(split, xs[i & 1], os_[i & 1])
    m.host_sync()
    da = (time.perf_counter() - t0) / n
    t0 = time.perf_counter()
    for i in range(n):
        m.forward_host(split, xs[i & 1], os_[i & 1])
    ds = (time.perf_counter() - t0) / n
    print(f"{wl} host_chunk={c}: streamed {da * 1e3:.2f} ms/step -> {batch / da:.0f} img/s, "
          f"sync {ds * 1e3:.2f} ms -> {batch / ds:.0f} img/s", flush=True)
    m.close()
