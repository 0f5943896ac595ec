"""Minimal driver for ncu: build a workload's model and run `n` forwards (no timing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import hapi_inputs  # noqa: E402
import paper_2210_08650_b200 as H  # noqa: E402
from bench import WORKLOADS  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "resnet50_s21_b512"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
arch, act, split, batch, seed = WORKLOADS[wl]
m = H.Model(arch, act, list(hapi_inputs.params(arch, 1000 + seed).values()), batch, split, split)
x = torch.from_numpy(hapi_inputs.images(batch, seed)).cuda()
es = 4 if act == "f32" else 2
out = torch.empty(m.out_bytes[split - 1] // es * batch, dtype=torch.float32 if act == "f32" else torch.bfloat16,
                  device="cuda")
for _ in range(n):
    m.forward(split, x, out)
torch.cuda.synchronize()
m.close()
print("ok")
