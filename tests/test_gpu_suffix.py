"""Client-side frozen suffix on the GPU: a suffix model consumes the
storage side's send buffer (layer s output, NCHW act dtype) and computes layers s+1..e.

* bf16: prefix(s) -> suffix(s..e) is bitwise equal to prefix(e) (same kernels, fusions are
  bitwise neutral, the split activation is the same bf16 tensor either way);
* both dtypes: the suffix matches the oracle's suffix applied to the same input activations
  (rel-L2 <= 2e-2 bf16, <= 1e-5 fp32);
* argument errors.
"""
import numpy as np
import pytest

import hapi_inputs
from oracle import prefix
from tests.gpu_helpers import rel_l2
from tests.parity_check import check_close

pytestmark = pytest.mark.gpu

CASES = [("resnet50", 5, 21, 96, 3), ("resnet50", 13, 20, 96, 3), ("densenet121", 4, 9, 64, 3),
         ("densenet121", 9, 14, 64, 2), ("alexnet", 6, 17, 224, 2), ("vgg11", 11, 25, 64, 2),
         ("resnet18", 4, 10, 64, 3)]


def _run(arch, act, s, e, size, n):
    import torch
    import paper_2210_08650_b200 as H
    P = hapi_inputs.params(arch, 31)
    x = torch.from_numpy(hapi_inputs.images(n, 32, size, size)).cuda()
    es = 4 if act == "f32" else 2
    tdt = torch.float32 if act == "f32" else torch.bfloat16
    pre = H.Model(arch, act, list(P.values()), n, s, e, in_h=size, in_w=size)
    a = torch.empty(pre.out_bytes[s - 1] // es * n, dtype=tdt, device="cuda")
    full = torch.empty(pre.out_bytes[e - 1] // es * n, dtype=tdt, device="cuda")
    pre.forward(s, x, a)
    pre.forward(e, x, full)
    suf = H.Model(arch, act, list(P.values()), n, e, e, in_h=size, in_w=size, start_idx=s)
    got = torch.empty_like(full)
    suf.forward_suffix(e, a.view(n, -1), got)
    torch.cuda.synchronize()
    pre.close()
    suf.close()
    return P, a, full, got


@pytest.mark.parametrize("arch,s,e,size,n", CASES)
def test_suffix_bf16_bitwise_composition_and_oracle(arch, s, e, size, n):
    P, a, full, got = _run(arch, "bf16", s, e, size, n)
    import torch
    assert torch.equal(got.view(torch.int16), full.view(torch.int16))
    # oracle suffix from the same (bf16) split activations
    a64 = a.float().cpu().numpy().astype(np.float64)
    shape = prefix.prefix_forward(arch, P, hapi_inputs.images(1, 32, size, size), s).shape[1:]
    ref = prefix.suffix_forward(arch, P, a64.reshape((n,) + shape), s, e)
    check_close(got.float().cpu().numpy(), ref, "bf16", f"suffix {arch} {s}..{e}")


@pytest.mark.parametrize("arch,s,e,size,n", [c for c in CASES if c[0] in ("resnet18", "alexnet", "densenet121")])
def test_suffix_f32_matches_oracle(arch, s, e, size, n):
    P, a, full, got = _run(arch, "f32", s, e, size, n)
    a64 = a.cpu().numpy().astype(np.float64)
    shape = prefix.prefix_forward(arch, P, hapi_inputs.images(1, 32, size, size), s).shape[1:]
    ref = prefix.suffix_forward(arch, P, a64.reshape((n,) + shape), s, e)
    check_close(got.cpu().numpy(), ref, "f32", f"suffix {arch} {s}..{e}")
    assert rel_l2(got.cpu().numpy(), full.cpu().numpy()) <= 1e-5


def test_suffix_argument_errors():
    import torch
    import paper_2210_08650_b200 as H
    P = list(hapi_inputs.params("resnet18", 1).values())
    with pytest.raises(H.HapiError):
        H.Model("resnet18", "bf16", P, 2, 5, 5, in_h=64, in_w=64, start_idx=5)    # start must be < min_split
    m = H.Model("resnet18", "bf16", P, 2, 6, 8, in_h=64, in_w=64, start_idx=4)
    x = torch.zeros(2, 3, 64, 64, device="cuda")
    out = torch.zeros(1 << 16, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(H.HapiError):
        m.forward(6, x, out)                                                      # prefix entry on a suffix model
    acts = torch.zeros(2 * m.out_bytes[3] // 2, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(H.HapiError):
        m.forward_suffix(9, acts.view(2, -1), out)                                            # end outside [6, 8]
    with pytest.raises(ValueError):
        m.forward_suffix(7, out, out)                                             # acts not 2 layer-4 outputs
    m.close()
