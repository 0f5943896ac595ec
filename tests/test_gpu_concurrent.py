"""Multi-request serving on one GPU: the batch adaptation
assigns each queued request a COS batch under one HBM budget, each request runs its own
model on its own stream concurrently, and

* every request's split output is bitwise identical to running it alone (requests share no
  state: separate arenas, weights and streams), and matches the oracle on sampled images;
* the device memory the models own together stays within the budget the adaptation was given
  (Eq. 4's constraint, with est = W + b*P over-estimating each model, section 4.3).
"""
import numpy as np
import pytest

import hapi_inputs
from oracle import planner
from tests.gpu_helpers import oracle_all
from tests.parity_check import check_close

pytestmark = pytest.mark.gpu


def test_concurrent_requests_match_sequential_and_fit_budget():
    import torch
    import paper_2210_08650_b200 as H

    queue = [("resnet50", 21, 40), ("densenet121", 9, 64), ("resnet18", 10, 48)]   # (arch, split, images)
    reqs = []
    for seq, (arch, s, _) in enumerate(queue):
        sz = planner.layer_sizes(arch, act="bf16")
        reqs.append((seq, sz.weight_bytes[s - 1], sz.peak_bytes[s - 1], 4, 32))
    budget = sum(r[1] + 12 * r[2] for r in reqs)          # room for ~12 images per request
    batches, used = H.hapi_adapt_batches(reqs, budget, max_concurrency=8)
    assert all(4 <= b <= 32 for b in batches) and used <= budget

    models, inputs, outs = [], [], []
    for (arch, s, n), b in zip(queue, batches):
        P = hapi_inputs.params(arch, 21)
        m = H.Model(arch, "bf16", list(P.values()), b, s, s)
        x = torch.from_numpy(hapi_inputs.images(n, 22 + s, 224, 224)).cuda()
        out = torch.empty(m.out_bytes[s - 1] // 2 * n, dtype=torch.bfloat16, device="cuda")
        models.append(m)
        inputs.append(x)
        outs.append(out)
    owned = sum(sum(m.device_bytes()) for m in models)
    assert owned <= budget, (owned, budget)

    # alone, one after another
    alone = []
    for (arch, s, n), m, x, out in zip(queue, models, inputs, outs):
        m.forward(s, x, out)
        torch.cuda.synchronize()
        alone.append(out.clone())
    # concurrently, one stream per request
    streams = [torch.cuda.Stream() for _ in queue]
    for (arch, s, n), m, x, out, st in zip(queue, models, inputs, outs, streams):
        out.zero_()
        m.set_stream(st.cuda_stream)
    torch.cuda.synchronize()
    for (arch, s, n), m, x, out, st in zip(queue, models, inputs, outs, streams):
        m.forward(s, x, out)
    torch.cuda.synchronize()
    for a, out in zip(alone, outs):
        assert torch.equal(a.view(torch.int16), out.view(torch.int16))
    for (arch, s, n), out in zip(queue, outs):
        sel = [0, n - 1]
        ref = oracle_all(arch, 21, 22 + s, n, upto=s, sel=sel)[s - 1]
        got = out.float().cpu().numpy().reshape(n, -1)[sel]
        check_close(got, ref, "bf16", f"concurrent {arch} s={s}")
    for m in models:
        m.close()
