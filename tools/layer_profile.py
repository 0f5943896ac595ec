"""Per-launch profile of one workload: CUDA events between launches (hapi_prefix_forward_timed),
algorithmic FLOPs/bytes from hapi_plan_info.  Usage: python tools/layer_profile.py [workload] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import hapi_inputs  # noqa: E402
import paper_2210_08650_b200 as H  # noqa: E402
from bench import WORKLOADS  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "resnet50_s21_b512"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
arch, act, split, batch, seed = WORKLOADS[wl]
P = hapi_inputs.params(arch, 1000 + seed)
m = H.Model(arch, act, list(P.values()), batch, split, split)
x = torch.from_numpy(hapi_inputs.images(batch, seed)).cuda()
es = 4 if act == "f32" else 2
out = torch.empty(m.out_bytes[split - 1] // es * batch, dtype=torch.float32 if act == "f32" else torch.bfloat16,
                  device="cuda")
info = m.plan_info(split)
for _ in range(3):
    m.forward(split, x, out)
torch.cuda.synchronize()
ms = np.zeros(info["n"])
for _ in range(reps):
    ms += np.array(m.forward_timed(split, x, out))
ms /= reps
tot = ms.sum()
print(f"{wl}: {info['n']} launches, {tot:.3f} ms/step -> {batch / tot * 1e3:.0f} img/s")
print(f"{'#':>3} {'ms':>8} {'%':>5} {'TFLOP/s':>8} {'GB/s':>7}  op")
for i in range(info["n"]):
    tf = info["flops"][i] * batch / (ms[i] / 1e3) / 1e12
    gb = info["bytes"][i] * batch / (ms[i] / 1e3) / 1e9
    print(f"{i:3d} {ms[i]:8.4f} {100 * ms[i] / tot:5.1f} {tf:8.1f} {gb:7.0f}  {info['desc'][i]}")
