"""Device time of back-to-back forwards (graph replay) vs the sum of per-launch times, for
one workload: the difference is launch/prologue/tail overhead between kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import hapi_inputs  # noqa: E402
import paper_2210_08650_b200 as H  # noqa: E402
from bench import WORKLOADS  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "resnet50_s21_b512"
arch, act, split, batch, seed = WORKLOADS[wl]
m = H.Model(arch, act, list(hapi_inputs.params(arch, 1000 + seed).values()), batch, split, split)
st = torch.cuda.current_stream()
m.set_stream(st.cuda_stream)
x = torch.from_numpy(hapi_inputs.images(batch, seed)).cuda()
es = 4 if act == "f32" else 2
out = torch.empty(m.out_bytes[split - 1] // es * batch, dtype=torch.float32 if act == "f32" else torch.bfloat16,
                  device="cuda")
for _ in range(5):
    m.forward(split, x, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
e0.record(st)
for _ in range(n):
    m.forward(split, x, out)
e1.record(st)
torch.cuda.synchronize()
step = e0.elapsed_time(e1) / n
per = np.zeros(m.plan_info(split)["n"])
for _ in range(5):
    per += np.array(m.forward_timed(split, x, out))
per /= 5
print(f"{wl} PDL={os.environ.get('HAPI_PDL', '1')} GRAPH={os.environ.get('HAPI_GRAPH', '1')}: step {step:.3f} ms, "
      f"sum of launches {per.sum():.3f} ms, overhead {step - per.sum():.3f} ms over {len(per)} launches")
