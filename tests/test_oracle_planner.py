"""Pins for oracle/planner.py: paper anchors (tests/golden/paper_anchors.json), Table 2
counts, torchvision shapes (library), the paper's own profiling procedure (one random
sample through the forward, Alg. 1 lines 1-5), closed forms, brute force and
hypothesis properties (SPEC.md:134-139 as test ideas)."""
import json
import os

import numpy as np
import pytest
import torch
import torchvision
from hypothesis import given, settings, strategies as st

import hapi_inputs
from oracle import archs, planner, prefix

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_anchors.json")))
GBPS = GOLD["defaults"]["gbps_bytes"]
ARCHS = list(archs.ARCHS)


def q(arch, batch, gbps, budget=1 << 40, act="f32", **kw):
    return planner.SplitQuery(arch, archs.FREEZE[arch], batch, int(round(gbps * GBPS)), budget, act=act, **kw)


@pytest.mark.parametrize("anchor", GOLD["split_anchors"])
def test_paper_split_anchors(anchor):
    r = planner.choose_split(q(anchor["arch"], anchor["training_batch"], anchor["gbps"]))
    assert r.split_idx == anchor["split_idx"]
    sz = planner.layer_sizes(anchor["arch"])
    if "mb_per_iteration" in anchor:
        mib = r.bytes_per_iteration / 2 ** 20
        assert 0 <= anchor["mb_per_iteration"] - mib <= GOLD["mb_tolerance_rel"] * anchor["mb_per_iteration"]
    if "data_ratio_vs_freeze" in anchor:
        assert sz.out_bytes[r.split_idx - 1] == anchor["data_ratio_vs_freeze"] * sz.out_bytes[anchor["freeze_idx"] - 1]


def test_table2_counts_and_freeze():
    t2 = GOLD["table2"]
    for a in t2["n_layers_matching_canonical"]:
        assert len(archs.layers(a)) == t2["n_layers"][a]
    for a, n in t2["n_layers_known_mismatch"].items():
        if not a.startswith("_"):
            assert len(archs.layers(a)) == n
    for a in ARCHS:
        assert archs.FREEZE[a] == t2["freeze"][a]


def test_table4_trend():
    t4 = GOLD["table4"]
    got = [planner.choose_split(q("alexnet", 8000, g)).split_idx for g in t4["gbps"]]
    assert got[0] == 17 == t4["split_idx"][0]
    assert all(a >= b for a, b in zip(got, got[1:]))
    assert got == [17, 17, 17, 17, 16, 13, 13, 6, 3]  # reading A7 (values differ from Table 4)


def test_qualitative_sizes():
    for a in ARCHS:
        sz = planner.layer_sizes(a)
        assert any(sz.out_bytes[s - 1] < sz.input_bytes for s in range(1, archs.FREEZE[a] + 1))
        diffs = np.diff(sz.out_bytes)
        assert (diffs > 0).any() and (diffs < 0).any()


@pytest.mark.parametrize("arch", ARCHS)
def test_shapes_vs_torchvision(arch):
    """Library pin: the shapes torchvision produces layer by layer (batch 1, 224x224)."""
    from tests.test_oracle_models import TV, tv_layers
    model = TV[arch](weights=None).eval()
    t = torch.zeros(1, 3, 224, 224)
    sz = planner.layer_sizes(arch)
    with torch.no_grad():
        for s, (name, fn) in enumerate(tv_layers(arch, model), start=1):
            t = fn(t)
            assert t[0].numel() * 4 == sz.out_bytes[s - 1], (arch, s, name)
    bf = planner.layer_sizes(arch, act="bf16")
    assert [2 * b for b in bf.out_bytes] == sz.out_bytes


@pytest.mark.parametrize("arch", ["alexnet", "resnet18"])
def test_profiling_run_pin(arch):
    """Alg. 1 profile_model literally: one random input point through the forward,
    record the per-layer output sizes."""
    P = hapi_inputs.params(arch, 4)
    outs = prefix.prefix_forward_all(arch, P, hapi_inputs.images(1, 4))
    assert [o[0].size * 4 for o in outs] == planner.layer_sizes(arch).out_bytes


def test_weight_bytes_closed_form():
    """W(L) in fp32 = 4 x (torchvision parameter count minus BN running buffers)."""
    for a in ARCHS:
        n = sum(int(np.prod(s)) for _, s, k in hapi_inputs.param_table(a) if k not in ("m", "v"))
        assert planner.layer_sizes(a).weight_bytes[-1] == 4 * n
        # bf16: weights 2 bytes, vectors stay 4
        nw = sum(int(np.prod(s)) for _, s, k in hapi_inputs.param_table(a) if k == "w")
        assert planner.layer_sizes(a, act="bf16").weight_bytes[-1] == 4 * n - 2 * nw


def test_peak_closed_form():
    sz = planner.layer_sizes("resnet50")
    seq = [sz.input_bytes] + sz.out_bytes
    for s in range(1, 23):
        assert sz.peak_bytes[s - 1] == max(seq[i - 1] + seq[i] for i in range(1, s + 1))
    # W(21) bf16 = 47,122,304 B
    assert planner.layer_sizes("resnet50", act="bf16").weight_bytes[20] == 47122304


def brute_split(sizes, l0, freeze, batch, C):
    for s in range(1, freeze + 1):
        if sizes[s - 1] < l0 and sizes[s - 1] * batch < C:
            return s
    return freeze


@settings(max_examples=300, deadline=None)
@given(arch=st.sampled_from(ARCHS), batch=st.integers(1, 20000), bw=st.integers(1, 5 * 10 ** 9),
       act=st.sampled_from(["f32", "bf16"]), freeze_off=st.integers(0, 5))
def test_split_properties(arch, batch, bw, act, freeze_off):
    L = len(archs.layers(arch))
    freeze = max(1, archs.FREEZE[arch] - freeze_off)
    sz = planner.layer_sizes(arch, act=act)
    qq = planner.SplitQuery(arch, freeze, batch, bw, 1 << 50, act=act)
    r = planner.choose_split(qq)
    assert 1 <= r.split_idx <= freeze <= L
    assert r.split_idx == brute_split(sz.out_bytes, sz.input_bytes, freeze, batch, bw)
    assert all(sz.out_bytes[c - 1] < sz.input_bytes for c in r.candidates)
    assert r.candidates == sorted(r.candidates)
    assert r.bytes_per_iteration < bw or r.split_idx == freeze
    # bandwidth monotonicity and batch monotonicity
    r2 = planner.choose_split(planner.SplitQuery(arch, freeze, batch, bw * 2, 1 << 50, act=act))
    assert r2.split_idx <= r.split_idx
    r3 = planner.choose_split(planner.SplitQuery(arch, freeze, batch * 2, bw, 1 << 50, act=act))
    assert r3.split_idx >= r.split_idx


@settings(max_examples=200, deadline=None)
@given(arch=st.sampled_from(ARCHS), s=st.integers(1, 21), b=st.integers(1, 10 ** 4))
def test_est_linear(arch, s, b):
    s = min(s, len(archs.layers(arch)))
    est = lambda bb: planner.estimate(arch, s, bb)  # noqa: E731
    assert est(2 * b) - est(b) == est(3 * b) - est(2 * b)


@settings(max_examples=150, deadline=None)
@given(arch=st.sampled_from(ARCHS), extra=st.integers(0, 80), bmin=st.integers(1, 30),
       bmax=st.integers(30, 90), jitter=st.integers(0, 10 ** 6))
def test_cos_batch_brute_force(arch, extra, bmin, bmax, jitter):
    qq = q(arch, 2000, 1, budget=0, b_min=bmin, b_max=bmax)
    s = planner.choose_split(planner.SplitQuery(**{**qq.__dict__, "hbm_budget_bytes": 1 << 50})).split_idx
    sz = planner.layer_sizes(arch)
    W, P = sz.weight_bytes[s - 1], sz.peak_bytes[s - 1]
    budget = W + extra * P + jitter
    r = planner.choose_split(planner.SplitQuery(**{**qq.__dict__, "hbm_budget_bytes": budget}))
    best = 0
    for b in range(bmin, bmax + 1):  # linear scan for the largest feasible b
        if W + b * P <= budget:
            best = b
    if best == 0:
        assert r.status == "infeasible" and r.cos_batch == 0
    else:
        assert r.status == "ok" and r.cos_batch == best and r.est_bytes == W + best * P <= budget


def test_errors():
    with pytest.raises(ValueError):
        planner.choose_split(planner.SplitQuery("alexnet", 0, 1, 1, 1))
    with pytest.raises(ValueError):
        planner.choose_split(planner.SplitQuery("alexnet", 22, 1, 1, 1))
    with pytest.raises(ValueError):
        planner.choose_split(planner.SplitQuery("alexnet", 17, 0, 1, 1))
    with pytest.raises(ValueError):
        planner.choose_split(planner.SplitQuery("alexnet", 17, 1, 0, 1))
    with pytest.raises(ValueError):
        planner.choose_split(planner.SplitQuery("alexnet", 17, 1, 1, 1, b_min=5, b_max=4))
    with pytest.raises(OverflowError):
        planner.choose_split(planner.SplitQuery("alexnet", 17, 1 << 62, 1, 1 << 40))
    with pytest.raises(ValueError):
        planner.layer_sizes("alexnet", 16, 16)  # empty output


def test_no_candidate_defaults_to_freeze():
    r = planner.choose_split(planner.SplitQuery("vgg11", 25, 1, 1, 1 << 40))
    assert r.split_idx == archs.FREEZE["vgg11"]
