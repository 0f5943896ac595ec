"""Oracle prefix forward: y = f_s o ... o f_1 (x), each image independently.

TEST INFRASTRUCTURE ONLY (see oracle/ops.py header).

This is the storage-side hot path's definition: the server "executes the feature
extraction part up to the split index" and "sends back the outputs of the split
index layer", using "custom DNN models that run the forward pass
between arbitrary start and end layers".  Split index s = number of
leading layers run on storage, 1-based, inclusive (reading R1/A1).  The output is
the layer-s tensor for the whole batch, NCHW (or [b, F] inside a classifier) --
reading R11/A18.  Accumulation is float64.
"""
from __future__ import annotations

import numpy as np

from . import archs, ops


def prefix_forward(arch: str, params, images: np.ndarray, split_idx: int) -> np.ndarray:
    mods = archs.layers(arch)
    if not 1 <= split_idx <= len(mods):
        raise ValueError(f"split_idx {split_idx} not in [1, {len(mods)}]")
    x = np.asarray(images, dtype=ops.FLOAT)
    for m in mods[:split_idx]:
        x = m.fwd(x, params)
    return x


def normalize_u8(images_u8: np.ndarray, scale, shift) -> np.ndarray:
    """u8 ingest (optional; the data the client moves to the GPU,
    PAPER.md:911): uint8 NCHW images become x[n, c] = scale[c] * u[n, c] + shift[c] before
    layer 1 -- a caller's per-channel normalisation (u / 255 - mean) / std is
    scale = 1 / (255 std), shift = -mean / std."""
    u = np.asarray(images_u8)
    if u.dtype != np.uint8 or u.ndim != 4 or u.shape[1] != 3:
        raise ValueError("images_u8 must be uint8 [N,3,H,W]")
    sc = np.asarray(scale, dtype=ops.FLOAT).reshape(1, 3, 1, 1)
    sh = np.asarray(shift, dtype=ops.FLOAT).reshape(1, 3, 1, 1)
    return sc * u.astype(ops.FLOAT) + sh


def prefix_forward_all(arch: str, params, images: np.ndarray, upto: int | None = None):
    """Outputs of every layer 1..upto (one pass; used by the profiling-run pin)."""
    mods = archs.layers(arch)
    upto = len(mods) if upto is None else upto
    x = np.asarray(images, dtype=ops.FLOAT)
    outs = []
    for m in mods[:upto]:
        x = m.fwd(x, params)
        outs.append(x)
    return outs


def suffix_forward(arch: str, params, acts: np.ndarray, start_idx: int, end_idx: int) -> np.ndarray:
    """Layers start_idx+1 .. end_idx applied to layer start_idx's output (the client-side
    frozen suffix, PAPER.md:734 / SURVEY 8(f) f3): the same per-layer definitions, begun
    later.  acts: [B, C, H, W] (or [B, F]) as layer start_idx produces it."""
    mods = archs.layers(arch)
    x = np.asarray(acts, dtype=ops.FLOAT)
    for m in mods[start_idx:end_idx]:
        x = m.fwd(x, params)
    return x
