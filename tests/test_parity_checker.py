"""The parity checker (tests/parity_check.py) is itself pinned on CPU: it must accept the
error a legitimate bf16 implementation makes and reject the localized mistakes a
whole-call relative L2 lets through (VERDICT r1 'What's weak' 1: a 20% error confined to
one of 256 channels adds only ~1e-2 to the whole-call norm).

The 'legitimate' output is a bf16 emulation of the prefix: the oracle's own layer
definitions evaluated with every conv/linear weight and every layer output rounded to
bf16 (round-to-nearest-even, reading A19) -- the error model of SURVEY 8(c)'s feasibility
row (4e-3 .. 1.4e-2 rel-L2), which is *worse* than the fused GPU path (fewer roundings).
"""
import numpy as np
import pytest

import hapi_inputs
from oracle import archs, prefix
from tests.parity_check import bounds, check_close, stats


def bf16(a):
    """fp64/fp32 -> nearest bf16 (RNE), returned as fp64."""
    f = np.asarray(a, np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def emulate_bf16(arch, P, x, split):
    Pb = {k: (bf16(v) if k.endswith("weight") and v.ndim >= 2 else v) for k, v in P.items()}
    y = bf16(x)
    for m in archs.layers(arch)[:split]:
        y = bf16(m.fwd(y, Pb))
    return y


CASES = [("resnet18", 10, 64), ("resnet50", 11, 64), ("densenet121", 9, 64), ("vgg11", 11, 64)]


@pytest.fixture(scope="module", params=CASES, ids=[f"{a}_s{s}" for a, s, _ in CASES])
def case(request):
    arch, s, sz = request.param
    P = hapi_inputs.params(arch, 41)
    x = hapi_inputs.images(2, 42, sz, sz)
    ref = prefix.prefix_forward(arch, P, x, s)
    emu = emulate_bf16(arch, P, x, s)
    return arch, s, ref, emu


def test_accepts_bf16_emulation(case):
    arch, s, ref, emu = case
    st = check_close(emu, ref, "bf16", f"{arch} s={s} emulated")
    assert st["whole"] > 1e-3  # the emulation really carries bf16-sized error


def _channel(ref):
    # a typical channel: the median by norm (not the largest, where a mistake is least diluted)
    n = np.linalg.norm(np.moveaxis(ref, 1, 0).reshape(ref.shape[1], -1), axis=1)
    return int(np.argsort(n)[len(n) // 2])


def test_rejects_single_channel_scale_error(case):
    """BN-fold scale off by 20% in one channel."""
    arch, s, ref, emu = case
    bad = emu.copy()
    c = _channel(ref)
    bad[:, c] *= 1.2
    assert stats(bad, ref)["whole"] <= bounds("bf16")["whole"]  # the old norm-only check passes it
    with pytest.raises(AssertionError):
        check_close(bad, ref, "bf16")


def test_rejects_single_channel_bias_error(case):
    """Folded bias off by 0.2 x the channel's RMS in one channel."""
    arch, s, ref, emu = case
    bad = emu.copy()
    c = _channel(ref)
    bad[:, c] += 0.2 * np.sqrt(np.mean(ref[:, c] ** 2))
    assert stats(bad, ref)["whole"] <= bounds("bf16")["whole"]
    with pytest.raises(AssertionError):
        check_close(bad, ref, "bf16")


def test_rejects_corrupted_row_and_swapped_channels(case):
    arch, s, ref, emu = case
    bad = emu.copy()
    bad[1, :, ref.shape[2] // 2, :] = 0.0          # one output row of one image lost (a skipped tile)
    with pytest.raises(AssertionError):
        check_close(bad, ref, "bf16")
    bad = emu.copy()
    c = _channel(ref)
    bad[:, [c, c + 1]] = bad[:, [c + 1, c]]         # a channel permutation slip
    with pytest.raises(AssertionError):
        check_close(bad, ref, "bf16")


def test_rejects_one_wrong_element(case):
    arch, s, ref, emu = case
    bad = emu.copy()
    i = np.unravel_index(int(np.argmax(np.abs(ref))), ref.shape)
    bad[i] = 0.0                                    # one element never stored (a missed store)
    with pytest.raises(AssertionError):
        check_close(bad, ref, "bf16")


def test_fp32_bounds_accept_fp32_rounding_and_reject_bias_error():
    arch, s = "resnet18", 10
    P = hapi_inputs.params(arch, 43)
    x = hapi_inputs.images(2, 44, 64, 64)
    ref = prefix.prefix_forward(arch, P, x, s)
    P32 = {k: np.asarray(v, np.float32) for k, v in P.items()}
    y = np.asarray(x, np.float32)
    for m in archs.layers(arch)[:s]:
        y = np.asarray(m.fwd(y, P32), np.float32)   # every layer output rounded to fp32
    check_close(y, ref, "f32", "fp32 rounding")
    bad = y.astype(np.float64)
    c = _channel(ref)
    bad[:, c] += 1e-3 * np.sqrt(np.mean(ref[:, c] ** 2))
    with pytest.raises(AssertionError):
        check_close(bad, ref, "f32")


def test_classifier_outputs_use_elementwise_bound():
    rng = np.random.default_rng(0)
    ref = rng.standard_normal((3, 4096))
    ok = ref + 1e-3 * rng.standard_normal(ref.shape)
    check_close(ok, ref, "bf16")
    bad = ok.copy()
    bad[0, 7] += 5.0
    with pytest.raises(AssertionError):
        check_close(bad, ref, "bf16")
