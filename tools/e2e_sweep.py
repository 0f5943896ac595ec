"""End-to-end (pinned host buffers in and out) throughput of hapi_prefix_forward_host for
several host chunk sizes (HAPI_HOST_CHUNK).  Usage: e2e_sweep.py [workload] [chunks...]"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 2 and sys.argv[2] == "--one":
    import torch
    import hapi_inputs
    import paper_2210_08650_b200 as H
    from bench import WORKLOADS
    wl = sys.argv[1]
    arch, act, split, batch, seed = WORKLOADS[wl]
    m = H.Model(arch, act, list(hapi_inputs.params(arch, 1000 + seed).values()), batch, split, split)
    x = torch.from_numpy(hapi_inputs.images(batch, seed)).pin_memory()
    es = 4 if act == "f32" else 2
    o = torch.empty(m.out_bytes[split - 1] // es * batch, dtype=torch.float32 if act == "f32" else torch.bfloat16).pin_memory()
    for _ in range(3):
        m.forward_host(split, x, o)
    t0 = time.perf_counter()
    n = 10
    for _ in range(n):
        m.forward_host(split, x, o)
    dt = (time.perf_counter() - t0) / n
    print(f"{wl} chunk={os.environ.get('HAPI_HOST_CHUNK', 'default')}: {dt * 1e3:.2f} ms -> {batch / dt:.0f} img/s e2e",
          flush=True)
    m.close()
else:
    wl = sys.argv[1] if len(sys.argv) > 1 else "resnet50_s21_b512"
    for c in (sys.argv[2:] or ["default", "32", "64", "128", "256"]):
        env = dict(os.environ)
        if c != "default":
            env["HAPI_HOST_CHUNK"] = c
        subprocess.run([sys.executable, __file__, wl, "--one"], env=env, check=False)
