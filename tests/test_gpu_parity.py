"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element on
the same seeded inputs.  Tolerances are BASELINE.json's north_star: relative L2 <= 1e-5
on the fp32 path and <= 2e-2 on the bf16 tensor-core path (reading A21: over the whole
split output of the call, fp64) -- plus, through tests/parity_check.check_close, the same
bound per image, a per-channel bound and an element-wise bound, so an error confined to
one channel, one row or one element fails.  Shapes/bytes, split choices and batch sizes
are exact.
"""
import numpy as np
import pytest

import hapi_inputs
from oracle import archs, planner
from tests.gpu_helpers import gpu_forward, oracle_all, rel_l2
from tests.parity_check import check_close

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "bf16": 2e-2}
SMALL = {"alexnet": 224, "resnet18": 64, "resnet50": 96, "vgg11": 64, "densenet121": 64}


def _H():
    import paper_2210_08650_b200 as H
    return H


@pytest.mark.parametrize("act", ["f32", "bf16"])
@pytest.mark.parametrize("arch", list(archs.ARCHS))
def test_every_split_small(arch, act):
    """Every canonical split s = 1..L (fusion legality at every boundary, H3), ragged tiles."""
    H = _H()
    sz, n = SMALL[arch], 3
    P = hapi_inputs.params(arch, 21)
    x = hapi_inputs.images(n, 22, sz, sz)
    L = len(archs.layers(arch))
    ref = oracle_all(arch, 21, 22, n, sz, sz)
    model = H.Model(arch, act, list(P.values()), n, 1, L, in_h=sz, in_w=sz)
    for s in range(1, L + 1):
        got, _ = gpu_forward(arch, act, s, x, P, model=model)
        want = ref[s - 1]
        assert got.shape == (n, want[0].size)
        assert model.out_bytes[s - 1] == want[0].size * (4 if act == "f32" else 2)
        check_close(got, want, act, f"{arch} s={s} {sz}px")
    model.close()


@pytest.mark.parametrize("act", ["f32", "bf16"])
@pytest.mark.parametrize("arch", list(archs.ARCHS))
def test_every_split_224(arch, act):
    """Every canonical split at the paper's 224x224 input (reading A10), batch 2: the
    split-specific epilogue variants (NCHW store, pack, pools fused or not) on full-size
    maps, which the small-size sweep above does not reach."""
    H = _H()
    n = 2
    P = hapi_inputs.params(arch, 23)
    x = hapi_inputs.images(n, 24)
    L = len(archs.layers(arch))
    ref = oracle_all(arch, 23, 24, n)
    model = H.Model(arch, act, list(P.values()), n, 1, L)
    for s in range(1, L + 1):
        got, _ = gpu_forward(arch, act, s, x, P, model=model)
        assert model.out_bytes[s - 1] == ref[s - 1][0].size * (4 if act == "f32" else 2)
        check_close(got, ref[s - 1], act, f"{arch} s={s} 224px")
    model.close()


def test_config1_alexnet_fp32_full_batch():
    """configs[0]: AlexNet features prefix s=13, batch 8, fp32, full-batch parity."""
    P = hapi_inputs.params("alexnet", 1001)
    x = hapi_inputs.images(8, 1)
    got, m = gpu_forward("alexnet", "f32", 13, x, P)
    ref = oracle_all("alexnet", 1001, 1, 8, upto=13)[12]
    assert got.shape == (8, 9216)
    check_close(got, ref, "f32", "config1 alexnet s=13 b8")


SAMPLE = {"resnet18": (200, [0, 1, 198, 199]), "resnet50": (512, [0, 1, 510, 511])}


@pytest.mark.parametrize("arch,split", [("resnet18", 10), ("resnet50", 21), ("resnet50", 20)])
def test_configs_2_3_bench_size_sampled(arch, split):
    """configs[1]/[2] at the bench's launch configuration (batch 200 / 512): sampled
    outputs checked against the oracle one by one, and batch invariance (bitwise) ties the
    sampled images to their rows of the full-batch launch."""
    H = _H()
    batch, sel = SAMPLE[arch]
    seed = 2 if arch == "resnet18" else 3
    P = hapi_inputs.params(arch, 1000 + seed)
    x = hapi_inputs.images(batch, seed)
    model = H.Model(arch, "bf16", list(P.values()), batch, split, split)
    got, _ = gpu_forward(arch, "bf16", split, x, P, model=model)
    ref = oracle_all(arch, 1000 + seed, seed, batch, upto=split, sel=sel)[split - 1]
    check_close(got[sel], ref, "bf16", f"{arch} s={split} b{batch} sampled")
    small, _ = gpu_forward(arch, "bf16", split, np.ascontiguousarray(x[sel]), P, model=model)
    np.testing.assert_array_equal(small, got[sel])
    assert np.isfinite(got).all()
    model.close()


def _free_hbm():
    import torch
    return torch.cuda.mem_get_info()[0]


@pytest.mark.parametrize("arch,splits", [("vgg11", [11] + list(range(16, 26))),
                                         ("densenet121", [4, 9] + list(range(13, 21)))])
def test_config4_split_sweep_budgeted(arch, splits):
    """configs[3]: bf16 split sweep over the candidate layers with the HBM-budgeted COS
    batch (budgets: free HBM, 16 GiB = the paper's T4, 2 GiB).  Split/batch choices come
    from hapi_choose_split and must equal the oracle planner; activations within 2e-2;
    library-owned device bytes <= est(b, s) (reading R8)."""
    H = _H()
    P = hapi_inputs.params(arch, 1004)
    n = 2
    x = hapi_inputs.images(n, 4)
    ref = oracle_all(arch, 1004, 4, n, upto=max(splits))
    for budget in (_free_hbm() // 2, 16 << 30, 2 << 30):
        for s in splits:
            # freeze = s and a 1 B/s link: no candidate passes, Alg. 1 returns the freeze index s
            st, r, _ = H.hapi_choose_split(arch, s, 2000, 1, budget, b_min=25, b_max=2000, act="bf16")
            q = planner.choose_split(planner.SplitQuery(arch, s, 2000, 1, budget, b_min=25, b_max=2000, act="bf16"))
            assert (st, r["split_idx"], r["cos_batch"], r["est_bytes"]) == (q.status, q.split_idx, q.cos_batch,
                                                                             q.est_bytes)
            assert r["split_idx"] == s
            b = r["cos_batch"]
            model = H.Model(arch, "bf16", list(P.values()), b, s, s)
            wb, ab = model.device_bytes()
            est = planner.estimate(arch, s, b, "bf16")
            assert wb + ab <= est, (arch, s, b, wb, ab, est)
            if budget == (2 << 30):
                got, _ = gpu_forward(arch, "bf16", s, x, P, model=model)
                check_close(got, ref[s - 1], "bf16", f"{arch} s={s} cos_batch={b}")
            model.close()


@pytest.mark.parametrize("arch,split,act", [("resnet50", 21, "bf16"), ("alexnet", 13, "f32"), ("resnet18", 10, "bf16"),
                                            ("densenet121", 9, "bf16"), ("resnet50", 4, "bf16")])
def test_memory_bound(arch, split, act):
    """Device bytes owned by the model <= est(b, s) = W(s) + b*P(s) (section 4.3 'we
    always over-estimate')."""
    H = _H()
    P = hapi_inputs.params(arch, 7)
    for b in (1, 25, 200):
        model = H.Model(arch, act, list(P.values()), b, split, split)
        wb, ab = model.device_bytes()
        assert wb + ab <= planner.estimate(arch, split, b, act), (b, wb, ab)
        model.close()


@pytest.mark.parametrize("act", ["bf16", "f32"])
def test_chunking_batch_shard_invariance_determinism(act):
    """a8 + H6: chunked (batch > max_batch), sharded (contiguous ranges) and
    repeated runs give bit-identical outputs."""
    H = _H()
    arch, s, n = "resnet50", 21, 7
    P = hapi_inputs.params(arch, 8)
    x = hapi_inputs.images(n, 9, 96, 96)
    big = H.Model(arch, act, list(P.values()), n, s, s, in_h=96, in_w=96)
    small = H.Model(arch, act, list(P.values()), 3, s, s, in_h=96, in_w=96)
    full, _ = gpu_forward(arch, act, s, x, P, model=big)
    again, _ = gpu_forward(arch, act, s, x, P, model=big)
    chunked, _ = gpu_forward(arch, act, s, x, P, model=small)
    np.testing.assert_array_equal(full, again)
    np.testing.assert_array_equal(full, chunked)
    shards = [gpu_forward(arch, act, s, np.ascontiguousarray(x[a:b]), P, model=big)[0]
              for a, b in [(0, 2), (2, 5), (5, 7)]]
    np.testing.assert_array_equal(np.concatenate(shards), full)


@pytest.mark.parametrize("n,max_batch", [(9, 4), (200, 64)])   # (200, 64): ramped chunks 32, 64, 64, 40
def test_host_path_matches_oracle_and_device_path(n, max_batch):
    """f2: the host-buffer call (pinned H2D, compute, D2H on copy streams) against the
    oracle on sampled images (first, last and chunk-boundary images), and bitwise against
    the device-buffer call."""
    H = _H()
    arch, s = "resnet18", 10
    P = hapi_inputs.params(arch, 10)
    x = hapi_inputs.images(n, 11, 64, 64)
    m = H.Model(arch, "bf16", list(P.values()), max_batch, s, s, in_h=64, in_w=64, host_chunk=max_batch)
    host, _ = gpu_forward(arch, "bf16", s, x, P, model=m, host=True)
    sel = sorted({0, 1, n // 2, n - 2, n - 1} | ({31, 32, 95, 96, 159, 160} if n == 200 else set()))
    ref = oracle_all(arch, 10, 11, n, 64, 64, upto=s, sel=sel)[s - 1]
    check_close(host[sel], ref, "bf16", f"host path n={n}")
    dev, _ = gpu_forward(arch, "bf16", s, x, P, model=m)
    np.testing.assert_array_equal(dev, host)


@pytest.mark.parametrize("arch,split,b", [("resnet50", 21, 512), ("resnet50", 21, 25), ("densenet121", 9, 200),
                                          ("resnet18", 10, 1)])
def test_memory_bound_with_host_staging(arch, split, b):
    """With the host path's staging (allocated at create time, counted in device_bytes), the
    model stays within est(b, s) plus the closed-form staging term 2 * c * (l_0 + l_s) -- the
    double-buffered DRAM<->GPU copies of Eq. 1's C11 * B * (l_0 + l_split) (
    reading A14: a term added to both sides)."""
    H = _H()
    P = hapi_inputs.params(arch, 7)
    m = H.Model(arch, "bf16", list(P.values()), b, split, split, host_chunk=-1)
    wb, ab = m.device_bytes()
    c = b if b < 256 else min(b, max(64, (b * 3 // 16 + 15) // 16 * 16))
    sz = planner.layer_sizes(arch, act="bf16")
    assert wb + ab <= planner.estimate(arch, split, b, "bf16") + 2 * c * (sz.input_bytes + sz.out_bytes[split - 1])
    m.close()


def test_python_argument_validation():
    """The binding checks dtype, shape, device and output size before any pointer reaches
    the library: ValueError, never an out-of-bounds access."""
    import torch
    H = _H()
    P = hapi_inputs.params("resnet18", 0)
    m = H.Model("resnet18", "bf16", list(P.values()), 2, 10, 10, in_h=64, in_w=64)
    x = torch.zeros(2, 3, 64, 64, device="cuda")
    out = torch.zeros(2 * m.out_bytes[9] // 2, dtype=torch.bfloat16, device="cuda")
    m.forward(10, x, out)
    for bad_x, bad_out in ((x.half(), out), (x[:, :2].contiguous(), out), (x.cpu(), out),
                           (torch.zeros(2, 3, 32, 32, device="cuda"), out), (x, out[:-1]), (x, out.float()),
                           (x, out.cpu())):
        with pytest.raises(ValueError):
            m.forward(10, bad_x, bad_out)
    with pytest.raises(H.HapiError) as e:
        m.forward_host(10, x.cpu(), out.cpu())          # no staging was requested (host_chunk = 0)
    assert e.value.status == 1
    m.close()


def test_models_on_two_devices_in_one_process():
    """Per-device kernel attributes and the device guard: two models on two GPUs
    driven from one thread give the same bits as each alone, and the caller's current
    device is left unchanged."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    H = _H()
    P = hapi_inputs.params("resnet50", 5)
    x = hapi_inputs.images(3, 6, 96, 96)
    outs = []
    torch.cuda.set_device(0)
    for dev in (0, 1):
        m = H.Model("resnet50", "bf16", list(P.values()), 3, 21, 21, in_h=96, in_w=96, device=dev)
        assert torch.cuda.current_device() == 0
        xd = torch.from_numpy(x).to(f"cuda:{dev}")
        o = torch.empty(3 * m.out_bytes[20] // 2, dtype=torch.bfloat16, device=f"cuda:{dev}")
        m.forward(21, xd, o)
        torch.cuda.synchronize(dev)
        assert torch.cuda.current_device() == 0
        outs.append(o.cpu())
        m.close()
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))


def test_gpu_argument_errors():
    import torch
    H = _H()
    P = hapi_inputs.params("alexnet", 0)
    m = H.Model("alexnet", "f32", list(P.values()), 2, 5, 13)
    x = torch.zeros(2, 3, 224, 224, device="cuda")
    out = torch.zeros(2 * 200000, device="cuda")
    for bad in (4, 14):
        with pytest.raises(H.HapiError) as e:
            m.forward(bad, x, out)
        assert e.value.status == 1
    with pytest.raises(H.HapiError):
        m.forward(13, x[:0], out)


def test_host_async_stream_matches_sync_and_oracle():
    """hapi_prefix_forward_host_async: back-to-back calls share the staging slots (chunk
    numbering continues across calls) -- every call's output equals the synchronous call's,
    bitwise, and the oracle on sampled images."""
    import torch
    H = _H()
    arch, s = "resnet18", 10
    P = hapi_inputs.params(arch, 12)
    m = H.Model(arch, "bf16", list(P.values()), 64, s, s, in_h=64, in_w=64, host_chunk=40)
    xs = [torch.from_numpy(hapi_inputs.images(n, 13 + n, 64, 64)) for n in (100, 37, 64, 5)]
    outs = [torch.empty(x.shape[0] * m.out_bytes[s - 1] // 2, dtype=torch.bfloat16) for x in xs]
    for x, o in zip(xs, outs):
        m.forward_host_async(s, x, o)
    m.host_sync()
    for x, o in zip(xs, outs):
        ref_sync = torch.empty_like(o)
        m.forward_host(s, x, ref_sync)
        assert torch.equal(o.view(torch.int16), ref_sync.view(torch.int16))
        n = x.shape[0]
        sel = [0, n - 1]
        ref = oracle_all(arch, 12, 13 + n, n, 64, 64, upto=s, sel=sel)[s - 1]
        check_close(o.float().numpy().reshape(n, -1)[sel], ref, "bf16", f"host async n={n}")
    m.close()
