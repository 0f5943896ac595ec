"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no convolution, pooling, BN, split
selection or size computation).  It only draws random numbers:

* ``images(n, seed)``: i.i.d. N(0,1) fp32 NCHW 3xHxW tensors -- the paper's
  "random_tensor(input_size)" / "Dataset: Synthetic" (
  reading R6/A10 in DESIGN.md).
* ``parity_subset(seed, a, b)``: the first/last 16 images of a shard, host-drawn per global
  index (the oracle-checked subset of the on-device generated strong-scaling set).
* ``images_u8(n, seed)``: i.i.d. uniform 0..255 uint8 NCHW images (the optional u8
  ingest of SURVEY 8(f) f2).
* ``params(arch, seed)``: fp32 weight tensors in torchvision ``state_dict`` order
  (PAPER.md:873 -- the paper used PyTorch; reading A12/A16).  Weights are *data*:
  the same arrays are handed to the oracle (as a name->array dict) and to
  ``hapi_model_create`` (as an ordered pointer list).

The parameter table below lists names and shapes only; it is pinned against
torchvision's own ``state_dict`` in ``tests/test_inputs.py``.
"""
from __future__ import annotations

from collections import OrderedDict

import numpy as np

ARCHS = ("alexnet", "resnet18", "resnet50", "vgg11", "densenet121")


# ----------------------------------------------------------------------------------
# parameter table (names, shapes, kinds) in torchvision state_dict order
# kinds: "w" conv/linear weight, "b" bias, "g" BN gamma, "bb" BN beta, "m" BN running
# mean, "v" BN running var.  num_batches_tracked buffers are excluded (int64, unused
# in eval mode).
# ----------------------------------------------------------------------------------

def _bn(name, c):
    return [(f"{name}.weight", (c,), "g"), (f"{name}.bias", (c,), "bb"),
            (f"{name}.running_mean", (c,), "m"), (f"{name}.running_var", (c,), "v")]


def _conv(name, cin, cout, k, bias):
    t = [(f"{name}.weight", (cout, cin, k, k), "w")]
    if bias:
        t.append((f"{name}.bias", (cout,), "b"))
    return t


def _linear(name, fin, fout):
    return [(f"{name}.weight", (fout, fin), "w"), (f"{name}.bias", (fout,), "b")]


def _alexnet():
    t = []
    t += _conv("features.0", 3, 64, 11, True)
    t += _conv("features.3", 64, 192, 5, True)
    t += _conv("features.6", 192, 384, 3, True)
    t += _conv("features.8", 384, 256, 3, True)
    t += _conv("features.10", 256, 256, 3, True)
    t += _linear("classifier.1", 256 * 6 * 6, 4096)
    t += _linear("classifier.4", 4096, 4096)
    t += _linear("classifier.6", 4096, 1000)
    return t


def _resnet(block, layers):
    t = _conv("conv1", 3, 64, 7, False) + _bn("bn1", 64)
    inplanes = 64
    expansion = 1 if block == "basic" else 4
    for li, (planes, n) in enumerate(zip((64, 128, 256, 512), layers)):
        for bi in range(n):
            stride = 2 if (li > 0 and bi == 0) else 1
            p = f"layer{li + 1}.{bi}"
            if block == "basic":
                t += _conv(f"{p}.conv1", inplanes, planes, 3, False) + _bn(f"{p}.bn1", planes)
                t += _conv(f"{p}.conv2", planes, planes, 3, False) + _bn(f"{p}.bn2", planes)
            else:
                t += _conv(f"{p}.conv1", inplanes, planes, 1, False) + _bn(f"{p}.bn1", planes)
                t += _conv(f"{p}.conv2", planes, planes, 3, False) + _bn(f"{p}.bn2", planes)
                t += _conv(f"{p}.conv3", planes, planes * 4, 1, False) + _bn(f"{p}.bn3", planes * 4)
            if stride != 1 or inplanes != planes * expansion:
                t += _conv(f"{p}.downsample.0", inplanes, planes * expansion, 1, False)
                t += _bn(f"{p}.downsample.1", planes * expansion)
            inplanes = planes * expansion
    t += _linear("fc", 512 * expansion, 1000)
    return t


def _vgg11():
    cfg = [64, "M", 128, "M", 256, 256, "M", 512, 512, "M", 512, 512, "M"]
    t, idx, cin = [], 0, 3
    for v in cfg:
        if v == "M":
            idx += 1
        else:
            t += _conv(f"features.{idx}", cin, v, 3, True)
            cin = v
            idx += 2
    t += _linear("classifier.0", 512 * 7 * 7, 4096)
    t += _linear("classifier.3", 4096, 4096)
    t += _linear("classifier.6", 4096, 1000)
    return t


def _densenet121():
    growth, bn_size = 32, 4
    t = _conv("features.conv0", 3, 64, 7, False) + _bn("features.norm0", 64)
    c = 64
    for bi, n in enumerate((6, 12, 24, 16)):
        for li in range(n):
            p = f"features.denseblock{bi + 1}.denselayer{li + 1}"
            cin = c + li * growth
            t += _bn(f"{p}.norm1", cin) + _conv(f"{p}.conv1", cin, bn_size * growth, 1, False)
            t += _bn(f"{p}.norm2", bn_size * growth) + _conv(f"{p}.conv2", bn_size * growth, growth, 3, False)
        c += n * growth
        if bi != 3:
            p = f"features.transition{bi + 1}"
            t += _bn(f"{p}.norm", c) + _conv(f"{p}.conv", c, c // 2, 1, False)
            c //= 2
    t += _bn("features.norm5", c)
    t += _linear("classifier", c, 1000)
    return t


_TABLES = {"alexnet": _alexnet, "resnet18": lambda: _resnet("basic", (2, 2, 2, 2)),
           "resnet50": lambda: _resnet("bottleneck", (3, 4, 6, 3)), "vgg11": _vgg11,
           "densenet121": _densenet121}


def param_table(arch: str):
    """[(name, shape, kind)] in torchvision state_dict order (no num_batches_tracked)."""
    return _TABLES[arch]()


# ----------------------------------------------------------------------------------
# generators
# ----------------------------------------------------------------------------------

def images(n: int, seed: int, h: int = 224, w: int = 224) -> np.ndarray:
    """fp32 NCHW images, i.i.d. N(0,1), NumPy PCG64."""
    g = np.random.Generator(np.random.PCG64(seed))
    return g.standard_normal((n, 3, h, w), dtype=np.float32)


def parity_subset(seed: int, a: int, b: int, k: int = 16, h: int = 224, w: int = 224):
    """The parity subset of the image shard [a, b) of a large generated set (SURVEY 8(d), config
    5): its first and last k images, each drawn on the host from its own stream keyed by its
    global index, so the oracle side regenerates exactly what the device run used.
    -> (global indices, fp32 NCHW array)."""
    idx = sorted(set(range(a, min(a + k, b))) | set(range(max(b - k, a), b)))
    arr = np.stack([images(1, 7_000_003 * (seed + 1) + g, h, w)[0] for g in idx]) if idx else \
        np.zeros((0, 3, h, w), np.float32)
    return idx, arr


def images_u8(n: int, seed: int, h: int = 224, w: int = 224) -> np.ndarray:
    """uint8 NCHW images (the u8-ingest calls), i.i.d. uniform over 0..255, NumPy PCG64."""
    g = np.random.Generator(np.random.PCG64(seed))
    return g.integers(0, 256, size=(n, 3, h, w), dtype=np.uint8)


def params(arch: str, seed: int) -> "OrderedDict[str, np.ndarray]":
    """fp32 parameters (reading A16): conv/linear weights He-normal N(0, 2/fan_in);
    biases U(-0.1, 0.1); BN gamma U(0.8,1.2), beta U(-0.1,0.1), running_mean
    U(-0.1,0.1), running_var U(0.8,1.2) so that BN folding is exercised.
    Each tensor has its own stream (SeedSequence([seed, index])) so the values do not
    depend on generation order."""
    out = OrderedDict()
    for i, (name, shape, kind) in enumerate(param_table(arch)):
        g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, i])))
        if kind == "w":
            fan_in = int(np.prod(shape[1:]))
            a = g.standard_normal(shape, dtype=np.float32) * np.float32(np.sqrt(2.0 / fan_in))
        elif kind in ("b", "bb", "m"):
            a = g.uniform(-0.1, 0.1, size=shape).astype(np.float32)
        elif kind in ("g", "v"):
            a = g.uniform(0.8, 1.2, size=shape).astype(np.float32)
        else:  # pragma: no cover
            raise ValueError(kind)
        out[name] = np.ascontiguousarray(a)
    return out
