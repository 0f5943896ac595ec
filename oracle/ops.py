"""Oracle operators: the textbook eval-mode definitions, NCHW, float64 (FLOAT).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this package.
The product path (``paper_2210_08650_b200``) never imports it.

Each operator is the plain definition the paper's PyTorch layers compute
("we use PyTorch"; the storage side "executes the feature extraction
part up to the split index").  Eval-mode semantics (reading R5/A9,
PAPER.md:683 "its weights are frozen"): BatchNorm uses running statistics with
eps = 1e-5, Dropout is the identity.  A library primitive (np.matmul) is used as
the contraction step of the convolution, after an explicit im2col.
"""
from __future__ import annotations

import numpy as np

BN_EPS = 1e-5

# Working precision of every operator: float64 for parity (the oracle proper).  bench.py's
# cpu_baseline leg alone switches to float32 ("the same code in fp32 mode").
FLOAT = np.float64


class precision:
    """with ops.precision(np.float32): ... -- run the same definitions at another width."""

    def __init__(self, dt):
        self.dt = dt

    def __enter__(self):
        global FLOAT
        self.prev, FLOAT = FLOAT, self.dt
        return self

    def __exit__(self, *a):
        global FLOAT
        FLOAT = self.prev


def out_size(h: int, k: int, stride: int, pad: int) -> int:
    """H_out = floor((H + 2p - k) / s) + 1 (no dilation, ceil_mode=False)."""
    return (h + 2 * pad - k) // stride + 1


def conv2d(x: np.ndarray, w: np.ndarray, b, stride: int, pad: int) -> np.ndarray:
    """out[n,o,y,x] = b[o] + sum_{c,r,t} W[o,c,r,t] * in[n,c,y*s+r-p,x*s+t-p], zero padding.

    Explicit im2col (every (r,t) tap gathered into its own column block) followed by
    one matmul per image over K = C*R*S."""
    x = np.asarray(x, dtype=FLOAT)
    w = np.asarray(w, dtype=FLOAT)
    n, c, h, wd = x.shape
    o, c2, r, s = w.shape
    assert c == c2, (x.shape, w.shape)
    oh, ow = out_size(h, r, stride, pad), out_size(wd, s, stride, pad)
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    wm = w.reshape(o, c * r * s)
    out = np.empty((n, o, oh, ow), dtype=FLOAT)
    for i in range(n):  # one image at a time bounds the im2col buffer
        cols = np.empty((c, r, s, oh, ow), dtype=FLOAT)
        for dr in range(r):
            for ds in range(s):
                cols[:, dr, ds] = xp[i, :, dr: dr + stride * (oh - 1) + 1: stride,
                                     ds: ds + stride * (ow - 1) + 1: stride]
        out[i] = (wm @ cols.reshape(c * r * s, oh * ow)).reshape(o, oh, ow)
    if b is not None:
        out += np.asarray(b, dtype=FLOAT)[None, :, None, None]
    return out


def batchnorm_eval(x, gamma, beta, mean, var, eps: float = BN_EPS):
    """gamma * (x - mean) / sqrt(var + eps) + beta, per channel (axis 1)."""
    sh = (1, -1) + (1,) * (x.ndim - 2)
    g = np.asarray(gamma, FLOAT).reshape(sh)
    b = np.asarray(beta, FLOAT).reshape(sh)
    m = np.asarray(mean, FLOAT).reshape(sh)
    v = np.asarray(var, FLOAT).reshape(sh)
    return g * (np.asarray(x, FLOAT) - m) / np.sqrt(v + eps) + b


def relu(x):
    return np.maximum(x, 0.0)


def maxpool2d(x, k: int, stride: int, pad: int):
    """max over the k x k window; padding = -inf; ceil_mode=False."""
    n, c, h, w = x.shape
    oh, ow = out_size(h, k, stride, pad), out_size(w, k, stride, pad)
    xp = np.pad(np.asarray(x, FLOAT), ((0, 0), (0, 0), (pad, pad), (pad, pad)),
                constant_values=-np.inf)
    out = np.full((n, c, oh, ow), -np.inf, dtype=FLOAT)
    for dr in range(k):
        for ds in range(k):
            out = np.maximum(out, xp[:, :, dr: dr + stride * (oh - 1) + 1: stride,
                                     ds: ds + stride * (ow - 1) + 1: stride])
    return out


def avgpool2d(x, k: int, stride: int):
    """mean over the k x k window, no padding (DenseNet transition: k = s = 2)."""
    n, c, h, w = x.shape
    oh, ow = out_size(h, k, stride, 0), out_size(w, k, stride, 0)
    acc = np.zeros((n, c, oh, ow), dtype=FLOAT)
    for dr in range(k):
        for ds in range(k):
            acc += np.asarray(x, FLOAT)[:, :, dr: dr + stride * (oh - 1) + 1: stride,
                                             ds: ds + stride * (ow - 1) + 1: stride]
    return acc / (k * k)


def adaptive_bins(insz: int, outsz: int):
    """PyTorch adaptive pooling bins: [floor(i*H/o), ceil((i+1)*H/o))."""
    return [((i * insz) // outsz, -((-(i + 1) * insz) // outsz)) for i in range(outsz)]


def adaptive_avgpool2d(x, oh: int, ow: int):
    n, c, h, w = x.shape
    out = np.empty((n, c, oh, ow), dtype=FLOAT)
    for i, (h0, h1) in enumerate(adaptive_bins(h, oh)):
        for j, (w0, w1) in enumerate(adaptive_bins(w, ow)):
            out[:, :, i, j] = np.asarray(x, FLOAT)[:, :, h0:h1, w0:w1].mean(axis=(2, 3))
    return out


def flatten(x):
    return np.asarray(x, FLOAT).reshape(x.shape[0], -1)


def linear(x, w, b):
    """x W^T + b on the flattened input."""
    return flatten(x) @ np.asarray(w, FLOAT).T + np.asarray(b, FLOAT)[None, :]
