"""Pinned host->device copy bandwidth with the 308 MB step split over 1, 2 or 4 streams (copy
engines), and with a concurrent device->host stream (full duplex), to see whether one H2D stream
is the e2e ceiling."""
import time

import torch

n = 512 * 3 * 224 * 224
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    part = n // ns
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            for k, s in enumerate(streams):
                with torch.cuda.stream(s):
                    d[k * part:(k + 1) * part].copy_(h[k * part:(k + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
    print(f"H2D over {ns} stream(s): {n * 4 / dt / 1e9:.1f} GB/s", flush=True)
