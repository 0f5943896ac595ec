import hashlib, os, sys
sys.path.insert(0, os.getcwd())
import torch, hapi_inputs, paper_2210_08650_b200 as H
from bench import WORKLOADS
arch, act, split, batch, seed = WORKLOADS[sys.argv[1]]
P = hapi_inputs.params(arch, 1000 + seed)
m = H.Model(arch, act, list(P.values()), batch, 1, split)
x = torch.from_numpy(hapi_inputs.images(batch, seed)).cuda()
for s in (1, split):
    out = torch.empty(m.out_bytes[s - 1] // 2 * batch, dtype=torch.bfloat16, device="cuda")
    m.forward(s, x, out); torch.cuda.synchronize()
    print(sys.argv[1], s, hashlib.md5(out.view(torch.int16).cpu().numpy().tobytes()).hexdigest())
