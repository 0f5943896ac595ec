"""Pins for oracle/ops.py that do not rely on the oracle itself.

* brute force: pure-Python nested loops written straight from the definitions, on
  tiny tensors (exact up to fp64 rounding);
* library: torch CPU float64 functional ops (F.conv2d, max_pool2d, avg_pool2d,
  batch_norm(training=False), adaptive_avg_pool2d, linear).

Every (kernel, stride, pad) combination of the canonical layer lists is covered.
"""
import itertools

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import ops

CONV_CASES = [  # (k, stride, pad) used by AlexNet/ResNet/VGG/DenseNet (Appendix A)
    (11, 4, 2), (5, 1, 2), (3, 1, 1), (7, 2, 3), (1, 1, 0), (1, 2, 0), (3, 2, 1)]


def brute_conv(x, w, b, stride, pad):
    n, c, h, wd = x.shape
    o, _, r, s = w.shape
    oh = (h + 2 * pad - r) // stride + 1
    ow = (wd + 2 * pad - s) // stride + 1
    out = np.zeros((n, o, oh, ow))
    for i, oo, y, xx in itertools.product(range(n), range(o), range(oh), range(ow)):
        acc = 0.0 if b is None else float(b[oo])
        for cc, dr, ds in itertools.product(range(c), range(r), range(s)):
            iy, ix = y * stride + dr - pad, xx * stride + ds - pad
            if 0 <= iy < h and 0 <= ix < wd:
                acc += float(w[oo, cc, dr, ds]) * float(x[i, cc, iy, ix])
        out[i, oo, y, xx] = acc
    return out


def brute_pool(x, k, stride, pad, mode):
    n, c, h, w = x.shape
    oh = (h + 2 * pad - k) // stride + 1
    ow = (w + 2 * pad - k) // stride + 1
    out = np.zeros((n, c, oh, ow))
    for i, cc, y, xx in itertools.product(range(n), range(c), range(oh), range(ow)):
        vals = []
        for dr, ds in itertools.product(range(k), range(k)):
            iy, ix = y * stride + dr - pad, xx * stride + ds - pad
            if 0 <= iy < h and 0 <= ix < w:
                vals.append(float(x[i, cc, iy, ix]))
        out[i, cc, y, xx] = max(vals) if mode == "max" else sum(vals) / (k * k)
    return out


@pytest.mark.parametrize("k,stride,pad", CONV_CASES)
@pytest.mark.parametrize("bias", [False, True])
def test_conv_brute_force(k, stride, pad, bias):
    g = np.random.default_rng(100 + k * 10 + stride + pad)
    h = max(k + 2, 9) + 1  # ragged (odd) sizes
    x = g.standard_normal((2, 3, h, h - 1))
    w = g.standard_normal((4, 3, k, k))
    b = g.standard_normal(4) if bias else None
    np.testing.assert_allclose(ops.conv2d(x, w, b, stride, pad), brute_conv(x, w, b, stride, pad),
                               rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("k,stride,pad", CONV_CASES)
def test_conv_torch_fp64(k, stride, pad):
    g = np.random.default_rng(7 + k)
    x = g.standard_normal((2, 5, 23, 19))
    w = g.standard_normal((6, 5, k, k))
    b = g.standard_normal(6)
    ref = F.conv2d(torch.from_numpy(x), torch.from_numpy(w), torch.from_numpy(b), stride, pad).numpy()
    np.testing.assert_allclose(ops.conv2d(x, w, b, stride, pad), ref, rtol=1e-11, atol=1e-11)


def test_conv_asymmetric_weight_catches_transpose():
    """A transposed kernel (r<->s) or flipped kernel must fail: use a single tap."""
    x = np.zeros((1, 1, 5, 5))
    x[0, 0, 1, 3] = 1.0
    w = np.zeros((1, 1, 3, 3))
    w[0, 0, 0, 2] = 1.0  # out[y,x] = in[y-1, x+1]
    out = ops.conv2d(x, w, None, 1, 1)
    assert out[0, 0, 2, 2] == 1.0 and out.sum() == 1.0


@pytest.mark.parametrize("k,stride,pad", [(3, 2, 0), (3, 2, 1), (2, 2, 0)])
def test_maxpool(k, stride, pad):
    g = np.random.default_rng(k + pad)
    x = g.standard_normal((2, 3, 13, 12)) - 5.0  # all negative near borders: padding must be -inf
    np.testing.assert_array_equal(ops.maxpool2d(x, k, stride, pad), brute_pool(x, k, stride, pad, "max"))
    ref = F.max_pool2d(torch.from_numpy(x), k, stride, pad).numpy()
    np.testing.assert_array_equal(ops.maxpool2d(x, k, stride, pad), ref)


def test_avgpool():
    g = np.random.default_rng(3)
    x = g.standard_normal((2, 4, 11, 10))
    np.testing.assert_allclose(ops.avgpool2d(x, 2, 2), brute_pool(x, 2, 2, 0, "avg"), rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(ops.avgpool2d(x, 2, 2), F.avg_pool2d(torch.from_numpy(x), 2, 2).numpy(), atol=1e-15,
                               rtol=1e-14)


@pytest.mark.parametrize("h,w,oh,ow", [(13, 13, 6, 6), (6, 6, 6, 6), (7, 7, 7, 7), (7, 7, 1, 1),
                                       (9, 5, 7, 7), (3, 3, 6, 6)])
def test_adaptive_avgpool(h, w, oh, ow):
    g = np.random.default_rng(h * 100 + w)
    x = g.standard_normal((2, 3, h, w))
    ref = F.adaptive_avg_pool2d(torch.from_numpy(x), (oh, ow)).numpy()
    np.testing.assert_allclose(ops.adaptive_avgpool2d(x, oh, ow), ref, rtol=1e-13, atol=1e-14)
    if (h, w) == (oh, ow):  # identity at matching size (AlexNet 6x6, VGG 7x7 at 224)
        np.testing.assert_array_equal(ops.adaptive_avgpool2d(x, oh, ow), x)


def test_batchnorm_eval():
    g = np.random.default_rng(5)
    x = g.standard_normal((3, 4, 5, 6))
    gam, bet, mu = g.uniform(0.8, 1.2, 4), g.uniform(-.1, .1, 4), g.uniform(-.1, .1, 4)
    var = g.uniform(0.8, 1.2, 4)
    ref = F.batch_norm(torch.from_numpy(x), torch.from_numpy(mu), torch.from_numpy(var),
                       torch.from_numpy(gam), torch.from_numpy(bet), training=False, eps=1e-5).numpy()
    np.testing.assert_allclose(ops.batchnorm_eval(x, gam, bet, mu, var), ref, rtol=1e-13, atol=1e-14)
    # closed form: gamma=1, beta=0, mean=0, var=1-eps is the identity
    np.testing.assert_allclose(ops.batchnorm_eval(x, np.ones(4), np.zeros(4), np.zeros(4),
                                                  np.full(4, 1 - 1e-5)), x, rtol=1e-15)


def test_linear_brute():
    g = np.random.default_rng(9)
    x = g.standard_normal((3, 2, 2, 3))
    w = g.standard_normal((5, 12))
    b = g.standard_normal(5)
    xf = x.reshape(3, 12)
    want = np.array([[sum(xf[i, k] * w[o, k] for k in range(12)) + b[o] for o in range(5)] for i in range(3)])
    np.testing.assert_allclose(ops.linear(x, w, b), want, rtol=1e-13)


def test_relu():
    x = np.array([-1.0, 0.0, 2.5, -0.0])
    np.testing.assert_array_equal(ops.relu(x), [0.0, 0.0, 2.5, 0.0])


def test_transition_pool_commutes_with_bias_free_1x1_conv():
    """The identity the executor's commuted DenseNet transition relies on (SURVEY
    K5): for a bias-free 1x1 conv W and the 2x2/s2 mean, avgpool(conv(y)) = conv(avgpool(y))
    for any y = relu(bn(x)) -- checked on the oracle's own operators, where it holds to
    rounding."""
    import numpy as np
    from oracle import ops
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 12, 8, 6))
    g, b, m, v = rng.uniform(0.8, 1.2, 12), rng.uniform(-.1, .1, 12), rng.uniform(-.1, .1, 12), rng.uniform(.8, 1.2, 12)
    w = rng.standard_normal((5, 12, 1, 1))
    y = ops.relu(ops.batchnorm_eval(x, g, b, m, v))
    a = ops.avgpool2d(ops.conv2d(y, w, None, 1, 0), 2, 2)
    c = ops.conv2d(ops.avgpool2d(y, 2, 2), w, None, 1, 0)
    np.testing.assert_allclose(a, c, rtol=1e-12, atol=1e-12)
    # and it fails with a bias-carrying or non-1x1 conv (why the planner checks both)
    k3 = rng.standard_normal((5, 12, 3, 3))
    assert not np.allclose(ops.avgpool2d(ops.conv2d(y, k3, None, 1, 1), 2, 2), ops.conv2d(ops.avgpool2d(y, 2, 2), k3, None, 1, 1))
