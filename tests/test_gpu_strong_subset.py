"""Config 5 (strong scaling over a 65,536-image set generated on device): the parity subset of a
shard -- its first and last 16 images, drawn on the host per global index
(hapi_inputs.parity_subset) and written over the device-generated images exactly as bench.py's
strong path does -- against the oracle, for a shard in the middle of the set."""
import numpy as np
import pytest

import hapi_inputs
from oracle import prefix
from tests.parity_check import check_close

pytestmark = pytest.mark.gpu


def test_strong_shard_parity_subset():
    import torch
    import paper_2210_08650_b200 as H
    from paper_2210_08650_b200.parallel import shard_range
    arch, act, split, seed, total, world, rank = "resnet50", "bf16", 21, 7, 65536, 1024, 517
    a, b = shard_range(total, world, rank)                 # 64 images: [33088, 33152)
    n = b - a
    P = hapi_inputs.params(arch, 1000 + seed)
    m = H.Model(arch, act, list(P.values()), 32, split, split)   # COS batch 32: the shard runs in 2 chunks
    try:
        x = torch.randn(n, 3, 224, 224, generator=torch.Generator(device="cuda").manual_seed(seed), device="cuda")
        idx, sub = hapi_inputs.parity_subset(seed, a, b)
        assert len(idx) == 32 and idx[0] == a and idx[-1] == b - 1
        pos = [g - a for g in idx]
        x[pos] = torch.from_numpy(sub).cuda()
        out = torch.empty(m.out_bytes[split - 1] // 2 * n, dtype=torch.bfloat16, device="cuda")
        m.forward(split, x, out)
        torch.cuda.synchronize()
        got = out.view(n, -1)[pos].float().cpu().numpy()
        sel = [0, 15, 16, 31]                              # both ends of both halves (oracle ~0.1 s / image)
        ref = prefix.prefix_forward(arch, P, sub[sel], split)
        check_close(got[sel].reshape(ref.shape), ref, act, "strong-scaling parity subset")
        # the subset is independent of the shard layout: the same global index gives the same image
        idx2, sub2 = hapi_inputs.parity_subset(seed, a - 48, b)
        assert np.array_equal(sub2[idx2.index(b - 1)], sub[idx.index(b - 1)])
    finally:
        m.close()
