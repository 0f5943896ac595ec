"""C-ABI library checks that need no GPU: the library loads, exports every symbol
include/hapi.h declares, and its planner equals the oracle bit-exactly (exhaustive grid
over archs x dtypes x image sizes x bandwidth x batch x budgets)."""
import itertools
import os
import re

import pytest

import hapi_inputs
import paper_2210_08650_b200 as H
from paper_2210_08650_b200 import _lib
from oracle import archs, planner

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARCHS = list(archs.ARCHS)


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "hapi.h")).read()
    declared = set(re.findall(r"HAPI_API[^;(]*?\b(hapi_\w+)\s*\(", hdr))
    assert len(declared) >= 16
    for name in declared:
        assert hasattr(_lib.lib, name), name
    assert declared == set(_lib.EXPORTED)
    assert "sm_100a" in H.build_info()


def test_num_layers_and_freeze():
    for a in ARCHS:
        assert H.hapi_num_layers(a) == len(archs.layers(a))
        assert H.hapi_freeze_index(a) == archs.FREEZE[a]
    assert _lib.hapi_num_layers(7) == -2


@pytest.mark.parametrize("arch", ARCHS)
def test_param_table_matches_inputs(arch):
    assert H.hapi_param_table(arch) == [(n, s) for n, s, _ in hapi_inputs.param_table(arch)]


@pytest.mark.parametrize("arch", ARCHS)
@pytest.mark.parametrize("act", ["f32", "bf16"])
@pytest.mark.parametrize("hw", [(224, 224), (256, 192), (96, 96), (227, 231)])
def test_layer_sizes_equal_oracle(arch, act, hw):
    try:
        ref = planner.layer_sizes(arch, hw[0], hw[1], act)
    except ValueError:
        with pytest.raises(H.HapiError):
            H.hapi_layer_sizes(arch, hw[0], hw[1], act)
        return
    l0, o, p, w = H.hapi_layer_sizes(arch, hw[0], hw[1], act)
    assert l0 == ref.input_bytes and o == ref.out_bytes and p == ref.peak_bytes and w == ref.weight_bytes


def test_layer_sizes_small_image_invalid():
    with pytest.raises(H.HapiError) as e:
        H.hapi_layer_sizes("alexnet", 16, 16)
    assert e.value.status == 2


GB = 125_000_000
BWS = [1, 10 ** 6, int(0.05 * GB), int(0.1 * GB), int(0.5 * GB), GB, 2 * GB, 3 * GB, 5 * GB, 10 * GB, 12 * GB, 10 ** 12]
BATCHES = [1, 25, 200, 512, 1000, 2000, 3000, 4000, 8000, 12000]
BUDGETS = [0, 2 << 30, 16 << 30, 180 << 30]


@pytest.mark.parametrize("arch", ARCHS)
@pytest.mark.parametrize("act", ["f32", "bf16"])
def test_choose_split_equals_oracle_exhaustive(arch, act):
    L = len(archs.layers(arch))
    for bw, batch, budget, freeze, (bmin, bmax) in itertools.product(
            BWS, BATCHES, BUDGETS, sorted({1, archs.FREEZE[arch], L}), [(25, 2000), (1, 1), (25, 512)]):
        q = planner.SplitQuery(arch, freeze, batch, bw, budget, b_min=bmin, b_max=bmax, act=act)
        ref = planner.choose_split(q)
        st, r, cands = H.hapi_choose_split(arch, freeze, batch, bw, budget, b_min=bmin, b_max=bmax, act=act)
        assert st == ref.status
        assert r["split_idx"] == ref.split_idx and r["cos_batch"] == ref.cos_batch
        assert r["bytes_per_iteration"] == ref.bytes_per_iteration and r["est_bytes"] == ref.est_bytes
        assert cands == ref.candidates and r["n_candidates"] == len(ref.candidates)


def test_paper_anchors_through_abi():
    _, r, _ = H.hapi_choose_split("alexnet", 17, 3000, GB, 1 << 40)
    assert r["split_idx"] == 13 and r["bytes_per_iteration"] == 110_592_000
    _, r, _ = H.hapi_choose_split("alexnet", 17, 4000, GB, 1 << 40)
    assert r["split_idx"] == 16 and r["bytes_per_iteration"] == 65_536_000
    _, r, _ = H.hapi_choose_split("densenet121", 20, 2000, 12 * GB, 1 << 40)
    assert r["split_idx"] == 9


@pytest.mark.parametrize("kw,code", [
    (dict(freeze_idx=0), 1), (dict(freeze_idx=99), 1), (dict(training_batch=0), 1),
    (dict(link_bytes_per_s=0), 1), (dict(b_min=5, b_max=4), 1), (dict(threshold_ms=0), 1),
    (dict(training_batch=1 << 62, link_bytes_per_s=1 << 40), 1)])
def test_choose_split_errors(kw, code):
    args = dict(arch="alexnet", freeze_idx=17, training_batch=100, link_bytes_per_s=GB, hbm_budget_bytes=1 << 40)
    args.update(kw)
    with pytest.raises(H.HapiError) as e:
        H.hapi_choose_split(**args)
    assert e.value.status == code


def test_infeasible_status():
    st, r, _ = H.hapi_choose_split("vgg11", 25, 2000, GB, 1 << 20)
    assert st == "infeasible" and r["cos_batch"] == 0 and r["split_idx"] == 23
    with pytest.raises(H.HapiError) as e:
        H.hapi_choose_split("vgg11", 25, 2000, GB, 1 << 20, raise_infeasible=True)
    assert e.value.status == 3


def test_model_create_argument_errors_without_gpu():
    """Argument validation happens before any device call."""
    P = list(hapi_inputs.params("alexnet", 0).values())
    with pytest.raises(H.HapiError) as e:
        H.Model("alexnet", "f32", P[:-1], 8, 13)
    assert e.value.status == 2
    with pytest.raises(H.HapiError) as e:
        H.Model("alexnet", "f32", P, 8, 22)
    assert e.value.status == 1
    with pytest.raises(H.HapiError) as e:
        H.Model("alexnet", "f32", P, 0, 13)
    assert e.value.status == 1
