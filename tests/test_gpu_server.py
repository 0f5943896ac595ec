"""The serving loop on the GPU: requests of three frozen
models, staggered arrivals, a memory budget that cannot hold them all at once.

* the scheduler's rounds decide admission/deferral (the C loop is the oracle-pinned
  hapi_scheduler); deferred requests run after earlier ones finish (carry-over);
* requests of one model share a single copy of its weights (hapi_model_create_shared);
* the device bytes the server holds never exceed the registered weights plus what Eq. 4
  accounts for the running requests, sum of W_r + b_r * P_r (each request's own memory
  stays within its estimate; the weights exist once);
* every request's output equals running it alone, and matches the oracle on sampled images.
"""
import numpy as np
import pytest

import hapi_inputs
from oracle import planner
from tests.gpu_helpers import oracle_all
from tests.parity_check import check_close

pytestmark = pytest.mark.gpu


def test_server_loop_admits_defers_and_matches_oracle():
    import torch
    import paper_2210_08650_b200 as H

    specs = {"resnet50": (21, 21), "densenet121": (9, 9), "resnet18": (10, 10)}
    P = {a: hapi_inputs.params(a, 61) for a in specs}
    # (arrival us, arch, split, n images, b_max)
    trace = [(0, "resnet50", 21, 60, 32), (10, "densenet121", 9, 40, 64), (20, "resnet18", 10, 50, 50),
             (30, "resnet50", 21, 30, 40), (5000, "densenet121", 9, 20, 20)]
    sz = {a: planner.layer_sizes(a, act="bf16") for a in specs}
    need = [sz[a].weight_bytes[s - 1] + 25 * sz[a].peak_bytes[s - 1] for _, a, s, _, _ in trace]
    budget = need[0] + need[1] + need[2] // 2          # the first round cannot admit everything
    srv = H.Server(budget, 0, max_concurrency=3, wait_us=100, b_min=25)
    mids = {a: srv.add_model(a, "bf16", list(P[a].values()), lo, hi) for a, (lo, hi) in specs.items()}
    weights = srv.device_bytes()
    reqs = []
    for t, a, s, n, bmax in trace:
        x = torch.from_numpy(hapi_inputs.images(n, 62 + t % 97)).cuda()
        out = torch.empty(n * sz[a].out_bytes[s - 1] // 2, dtype=torch.bfloat16, device="cuda")
        reqs.append([t, a, s, n, bmax, x, out, None])
    now, admitted_at, seen_deferred = 0, {}, False
    pending = list(range(len(reqs)))
    while True:
        while pending and reqs[pending[0]][0] <= now:
            r = reqs[pending.pop(0)]
            r[7] = srv.submit(now, mids[r[1]], r[2], r[4], r[5], r[6])
        active = srv.step(now)
        running_data = 0
        for r in reqs:
            if r[7] is None:
                continue
            st, b = srv.state(r[7])
            seen_deferred |= st == H.Scheduler.DEFERRED
            if st == H.Scheduler.RUNNING:
                admitted_at.setdefault(r[7], now)
                running_data += sz[r[1]].weight_bytes[r[2] - 1] + b * sz[r[1]].peak_bytes[r[2] - 1]
                assert 25 <= b <= r[4] or b == r[4]
        assert srv.device_bytes() <= weights + running_data, (srv.device_bytes(), weights, running_data)
        if not pending and active == 0:
            break
        now += 50
        assert now < 10_000_000
    torch.cuda.synchronize()
    assert seen_deferred                               # the budget forced a carry-over round
    for t, a, s, n, bmax, x, out, rid in reqs:
        m = H.Model(a, "bf16", list(P[a].values()), n, s, s)
        alone = torch.empty_like(out)
        m.forward(s, x, alone)
        torch.cuda.synchronize()
        m.close()
        assert torch.equal(alone.view(torch.int16), out.view(torch.int16)), (a, rid)
        sel = [0, n - 1]
        ref = oracle_all(a, 61, 62 + t % 97, n, upto=s, sel=sel)[s - 1]
        check_close(out.float().cpu().numpy().reshape(n, -1)[sel], ref, "bf16", f"server {a} s={s}")
    srv.close()


def test_shared_model_uses_one_weight_copy():
    import torch
    import paper_2210_08650_b200 as H
    P = hapi_inputs.params("resnet50", 3)
    base = H.Model("resnet50", "bf16", list(P.values()), 4, 21, 21, in_h=96, in_w=96)
    a = base.shared(8)
    wb, ab = a.device_bytes()
    assert wb == 0 and ab > 0
    x = torch.from_numpy(hapi_inputs.images(8, 4, 96, 96)).cuda()
    o1 = torch.empty(8 * base.out_bytes[20] // 2, dtype=torch.bfloat16, device="cuda")
    o2 = torch.empty_like(o1)
    base.forward(21, x, o1)
    base.close()                                       # the shared model keeps the weights alive
    a.forward(21, x, o2)
    torch.cuda.synchronize()
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))
    a.close()
