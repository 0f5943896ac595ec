"""Run-to-run determinism at bench-like sizes (GPU): the same forward repeated on the same
inputs must give the same bits.  A data race between epilogue warps, a
mis-ordered smem buffer reuse or a missing inter-kernel dependency shows up here as
changing bits -- at small test sizes the warps rarely overlap enough to expose it."""
import numpy as np
import pytest

import hapi_inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("arch,split,batch,reps", [
    ("resnet50", 21, 256, 6),
    ("resnet50", 8, 128, 4),
    ("densenet121", 9, 128, 4),
    ("resnet18", 10, 200, 4),
    ("vgg11", 21, 64, 3),
])
def test_repeated_forward_is_bitwise_stable(arch, split, batch, reps):
    import torch
    import paper_2210_08650_b200 as H
    P = hapi_inputs.params(arch, 77)
    m = H.Model(arch, "bf16", list(P.values()), batch, split, split)
    x = torch.from_numpy(hapi_inputs.images(batch, 78)).cuda()
    out = torch.empty(m.out_bytes[split - 1] // 2 * batch, dtype=torch.bfloat16, device="cuda")
    m.forward(split, x, out)
    torch.cuda.synchronize()
    ref = out.clone()
    try:
        for r in range(reps):
            m.forward(split, x, out)
            torch.cuda.synchronize()
            diff = int((out.view(torch.int16) != ref.view(torch.int16)).sum().item())
            assert diff == 0, (arch, split, r, diff)
    finally:
        m.close()
