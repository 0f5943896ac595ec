"""Throughput of the prefix forward at larger input sizes: ResNet50 s=21 and
DenseNet121 s=9 at 224..640 px, batch scaled so each step handles ~the same pixel count as
b512 at 224; device-resident inputs, CUDA events around K graph-replayed steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import hapi_inputs  # noqa: E402
import paper_2210_08650_b200 as H  # noqa: E402

for arch, split, seed in (("resnet50", 21, 3), ("densenet121", 9, 4)):
    P = list(hapi_inputs.params(arch, 1000 + seed).values())
    for size in (224, 320, 448, 640):
        batch = max(8, int(512 * (224 / size) ** 2) // 8 * 8)
        m = H.Model(arch, "bf16", P, batch, split, split, in_h=size, in_w=size)
        x = torch.randn(batch, 3, size, size, device="cuda")
        out = torch.empty(m.out_bytes[split - 1] // 2 * batch, dtype=torch.bfloat16, device="cuda")
        for _ in range(3):
            m.forward(split, x, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = 10
        e0.record()
        for _ in range(k):
            m.forward(split, x, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        info = m.plan_info(split)
        print(f"{arch} s={split} {size}px b{batch}: {ms:.3f} ms/step, {batch / ms * 1e3:.0f} img/s, "
              f"{batch * size * size / ms / 1e6:.1f} Gpx/s, {info['n']} launches", flush=True)
        m.close()
