"""Small forwards of every arch through the C ABI for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): bf16 tcgen05 kernels, the fp32 SIMT path, pools, packs, the suffix and
the host path.  Usage: compute-sanitizer --tool memcheck python tools/sanitize_fwd.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import hapi_inputs  # noqa: E402
import paper_2210_08650_b200 as H  # noqa: E402

CASES = [("resnet50", "bf16", 21, 96, 2), ("resnet50", "bf16", 20, 64, 2), ("resnet18", "bf16", 10, 64, 2),
         ("densenet121", "bf16", 9, 64, 2), ("vgg11", "bf16", 21, 64, 2), ("alexnet", "f32", 13, 224, 1),
         ("resnet18", "f32", 10, 64, 1)]
only = sys.argv[1:] or None
for arch, act, s, sz, n in CASES:
    if only and arch not in only:
        continue
    P = hapi_inputs.params(arch, 1)
    m = H.Model(arch, act, list(P.values()), n, s, s, in_h=sz, in_w=sz, host_chunk=n)
    x = torch.from_numpy(hapi_inputs.images(n, 2, sz, sz)).cuda()
    es = 4 if act == "f32" else 2
    out = torch.empty(n * m.out_bytes[s - 1] // es, dtype=torch.float32 if act == "f32" else torch.bfloat16, device="cuda")
    m.forward(s, x, out)
    torch.cuda.synchronize()
    oh = torch.empty(out.numel(), dtype=out.dtype)
    m.forward_host(s, x.cpu(), oh)
    assert torch.equal(oh.view(torch.int16 if es == 2 else torch.int32), out.cpu().view(torch.int16 if es == 2 else torch.int32))
    m.close()
    print("ok", arch, act, s, sz, flush=True)
