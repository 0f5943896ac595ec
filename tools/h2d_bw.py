"""Pinned host->device copy bandwidth (the e2e ceiling): 308 MB (512 fp32 224x224 images)."""
import torch

n = 512 * 3 * 224 * 224
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for chunk in (n, n // 4, n // 16):
    for _ in range(2):
        for c0 in range(0, n, chunk):
            d[c0:c0 + chunk].copy_(h[c0:c0 + chunk], non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        for c0 in range(0, n, chunk):
            d[c0:c0 + chunk].copy_(h[c0:c0 + chunk], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"H2D chunk {chunk * 4 / 2**20:.0f} MiB: {n * 4 / ms / 1e6:.1f} GB/s")
