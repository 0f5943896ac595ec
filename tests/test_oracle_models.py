"""Library pin for the whole oracle prefix: torchvision models in float64 eval mode with
the same weights, sliced at every canonical layer boundary s (reading R2), must agree
with oracle.prefix_forward to <= 1e-12 relative L2.

The torchvision slicing below is an independent construction of the canonical layer
list (from torchvision's own module tree), not a re-use of oracle/archs.py.
"""
import numpy as np
import pytest
import torch
import torch.nn as nn
import torch.nn.functional as F
import torchvision

import hapi_inputs
from oracle import archs, prefix

TV = {"alexnet": torchvision.models.alexnet, "resnet18": torchvision.models.resnet18,
      "resnet50": torchvision.models.resnet50, "vgg11": torchvision.models.vgg11,
      "densenet121": torchvision.models.densenet121}


class _DenseTail(nn.Module):
    """torchvision DenseNet.forward's functional tail + classifier."""

    def __init__(self, fc):
        super().__init__()
        self.fc = fc

    def forward(self, x):
        return self.fc(torch.flatten(F.adaptive_avg_pool2d(F.relu(x), (1, 1)), 1))


def tv_layers(arch, model):
    """Canonical layer list from the torchvision module tree: returns [(name, fn)]."""
    flat = lambda m: (lambda x: m(torch.flatten(x, 1)))  # noqa: E731
    if arch in ("alexnet", "vgg11"):
        L = [(f"features.{i}", m) for i, m in enumerate(model.features)]
        L.append(("avgpool", model.avgpool))
        L += [(f"classifier.{i}", flat(m) if i == 0 else m) for i, m in enumerate(model.classifier)]
        return L
    if arch.startswith("resnet"):
        L = [("conv1", model.conv1), ("bn1", model.bn1), ("relu", model.relu), ("maxpool", model.maxpool)]
        for li in range(1, 5):
            for bi, blk in enumerate(getattr(model, f"layer{li}")):
                L.append((f"layer{li}.{bi}", blk))
        L += [("avgpool", model.avgpool), ("fc", flat(model.fc))]
        return L
    L = []
    for name, m in model.features.named_children():
        if name.startswith("transition"):
            L += [(f"features.{name}.{n2}", m2) for n2, m2 in m.named_children()]
        else:
            L.append((f"features.{name}", m))
    L.append(("classifier", _DenseTail(model.classifier)))
    return L


SIZES = {"alexnet": 224, "resnet18": 224, "resnet50": 96, "vgg11": 64, "densenet121": 64}


@pytest.mark.parametrize("arch", list(TV))
def test_prefix_matches_torchvision_fp64_every_split(arch):
    P = hapi_inputs.params(arch, 11)
    model = TV[arch](weights=None).double().eval()
    model.load_state_dict({k: torch.from_numpy(v.astype(np.float64)) for k, v in P.items()}, strict=False)
    layers = tv_layers(arch, model)
    mods = archs.layers(arch)
    assert [n for n, _ in layers] == [m.name for m in mods]
    sz = SIZES[arch]
    x = hapi_inputs.images(2, 12, sz, sz)
    ours = prefix.prefix_forward_all(arch, P, x)
    t = torch.from_numpy(x.astype(np.float64))
    with torch.no_grad():
        for s, (name, fn) in enumerate(layers, start=1):
            t = fn(t)
            ref = t.numpy()
            got = ours[s - 1]
            assert got.shape == ref.shape, (s, name)
            rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)
            assert rel <= 1e-12, (arch, s, name, rel)
    # prefix_forward at a single split equals the running pass
    s_mid = len(mods) // 2
    np.testing.assert_array_equal(prefix.prefix_forward(arch, P, x, s_mid), ours[s_mid - 1])


def test_split_idx_bounds():
    P = hapi_inputs.params("alexnet", 1)
    x = hapi_inputs.images(1, 1)
    for bad in (0, 22):
        with pytest.raises(ValueError):
            prefix.prefix_forward("alexnet", P, x, bad)


def test_batch_invariance_oracle():
    """Each image is processed independently (eval mode)."""
    P = hapi_inputs.params("resnet18", 2)
    x = hapi_inputs.images(3, 3, 64, 64)
    full = prefix.prefix_forward("resnet18", P, x, 10)
    one = prefix.prefix_forward("resnet18", P, x[1:2], 10)
    np.testing.assert_allclose(full[1:2], one, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("act", ["f32", "bf16"])
@pytest.mark.parametrize("arch", list(TV))
def test_estimate_matches_torchvision_brute_force(arch, act):
    """planner.estimate(arch, s, b) = W(s) + b * P(s) (section 4.3), pinned
    against a construction that shares nothing with oracle/archs.py or oracle/planner.py:
    W(s) sums torchvision's own parameters of the first s layers of tv_layers (weights of
    rank >= 2 at the activation width, biases / BN affine at 4 bytes; running buffers are
    buffers, not parameters), P(s) = max over i <= s of input + output bytes of layer i
    measured by running the torchvision modules on one 224x224 image (Alg. 1 lines 1-5's
    profiling run), l_0 = the fp32 input.  Every s and three batches, and the split
    planner's est_bytes for the batch it picks equals the same value (an index slip such as
    W(s+1) or P(s-1) fails here)."""
    from oracle import planner
    ab = 2 if act == "bf16" else 4
    model = TV[arch](weights=None).float().eval()
    layers = tv_layers(arch, model)
    names = [n for n, _ in layers]
    owner = {}
    for pname, prm in model.named_parameters():
        mod = max((n for n in names if pname.startswith(n + ".")), key=len)
        owner.setdefault(mod, []).append(prm)
    t = torch.zeros(1, 3, 224, 224)
    sizes = [3 * 224 * 224 * 4]
    with torch.no_grad():
        for _, fn in layers:
            t = fn(t)
            sizes.append(t.numel() * ab)
    W = P = 0
    for s, n in enumerate(names, start=1):
        W += sum(p.numel() * (ab if p.dim() >= 2 else 4) for p in owner.get(n, []))
        P = max(P, sizes[s - 1] + sizes[s])
        for b in (1, 25, 512):
            assert planner.estimate(arch, s, b, act) == W + b * P, (arch, s, b)
        budget = W + 77 * P + 5
        r = planner.choose_split(planner.SplitQuery(arch, s, 1, 1, budget, b_min=1, b_max=100, act=act))
        assert r.split_idx == s and r.cos_batch == 77 and r.est_bytes == W + 77 * P
