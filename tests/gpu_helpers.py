"""Shared helpers for the GPU parity tests (and the debug script).  The oracle side and
the CUDA side only share the seeded inputs from hapi_inputs."""
from __future__ import annotations

import numpy as np

import hapi_inputs
from oracle import prefix

_ORACLE_CACHE = {}


def rel_l2(got, ref) -> float:
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def oracle_all(arch, pseed, iseed, n, h=224, w=224, upto=None, sel=None):
    """Outputs of every layer 1..upto for images `sel` (indices) of images(n, iseed)."""
    key = (arch, pseed, iseed, n, h, w, upto, tuple(sel) if sel is not None else None)
    if key not in _ORACLE_CACHE:
        P = hapi_inputs.params(arch, pseed)
        x = hapi_inputs.images(n, iseed, h, w)
        if sel is not None:
            x = x[list(sel)]
        _ORACLE_CACHE[key] = prefix.prefix_forward_all(arch, P, x, upto)
    return _ORACLE_CACHE[key]


def gpu_forward(arch, act, split, images: np.ndarray, params, max_batch=None, min_split=None, max_split=None,
                model=None, host=False):
    import torch
    import paper_2210_08650_b200 as H
    n, _, h, w = images.shape
    if model is None:
        model = H.Model(arch, act, list(params.values()), max_batch or n, min_split or split, max_split or split,
                        in_h=h, in_w=w)
    es = 4 if act == "f32" else 2
    numel = model.out_bytes[split - 1] // es * n
    tdt = torch.float32 if act == "f32" else torch.bfloat16
    if host:
        xh = torch.from_numpy(images).contiguous()
        out = torch.empty(numel, dtype=tdt)
        model.forward_host(split, xh, out)
    else:
        x = torch.from_numpy(images).cuda()
        out = torch.empty(numel, dtype=tdt, device="cuda")
        model.forward(split, x, out)
        torch.cuda.synchronize()
    return out.float().cpu().numpy().reshape(n, -1), model
