"""Determinism stress: the same forward repeated; any bit that changes between runs is a race.
Usage: python tools/race_check.py [arch] [split] [batch] [reps] [size]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import hapi_inputs  # noqa: E402
import paper_2210_08650_b200 as H  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
split = int(sys.argv[2]) if len(sys.argv) > 2 else 21
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 512
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
size = int(sys.argv[5]) if len(sys.argv) > 5 else 224
P = hapi_inputs.params(arch, 1003)
m = H.Model(arch, "bf16", list(P.values()), batch, split, split, in_h=size, in_w=size)
x = torch.from_numpy(hapi_inputs.images(batch, 3, size, size)).cuda()
out = torch.empty(m.out_bytes[split - 1] // 2 * batch, dtype=torch.bfloat16, device="cuda")
m.forward(split, x, out)
torch.cuda.synchronize()
ref = out.clone()
bad = 0
for i in range(reps):
    m.forward(split, x, out)
    torch.cuda.synchronize()
    d = (out.view(torch.int16) != ref.view(torch.int16)).sum().item()
    if d:
        bad += 1
        print(f"rep {i}: {d} elements differ")
flags = {k: v for k, v in os.environ.items() if k.startswith("HAPI_")}
print(f"{arch} s{split} b{batch} {flags}: {bad}/{reps} runs differ")
m.close()
