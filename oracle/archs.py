"""Oracle layer lists: the canonical module sequences of reading R2.

TEST INFRASTRUCTURE ONLY (see oracle/ops.py header).

"Layer" = torchvision module order (the paper used PyTorch), flattened
through ``nn.Sequential`` containers, with BasicBlock / Bottleneck / _DenseBlock kept
atomic ("For DNNs structured as a sequence of blocks (e.g. ResNets) we split at block
boundary", Table 2).  DenseNet's functional tail (relu -> adaptive
avgpool(1) -> flatten) is folded into its classifier; flatten is not a layer.  The
resulting counts are AlexNet 21, ResNet18 14, ResNet50 22, VGG11 29, DenseNet121 22
(Table 2, lists 22/14/22/28/22; the AlexNet and VGG11 mismatches are
recorded as paper inconsistency A2 in DESIGN.md).

Each module knows: its per-image output shape given the input shape (closed-form
shape rules), its forward on a batch (using oracle.ops and the parameter dict), and
how many weight elements / bias+BN-affine elements it owns (for W(s), section 8(b)).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Tuple

import numpy as np

from . import ops

FREEZE = {"alexnet": 17, "resnet18": 11, "resnet50": 21, "vgg11": 25, "densenet121": 20}
"""Table 2 freeze indices (PAPER.md:935)."""


@dataclass
class Module:
    name: str                      # torchvision module name (Appendix A of SURVEY.md)
    kind: str
    shape_fn: Callable             # (C,H,W) or (F,) -> output shape
    fwd: Callable                  # (x batch, params) -> y batch
    weight_elems: int = 0          # conv / linear weight elements
    vec_elems: int = 0             # bias + BN gamma/beta elements
    meta: dict = field(default_factory=dict)


def _numel(shape):
    n = 1
    for d in shape:
        n *= d
    return n


# ---------------------------------------------------------------- module builders

def conv(name, cin, cout, k, stride, pad, bias):
    def shape_fn(s):
        c, h, w = s
        assert c == cin, (name, s)
        return (cout, ops.out_size(h, k, stride, pad), ops.out_size(w, k, stride, pad))

    def fwd(x, P):
        return ops.conv2d(x, P[f"{name}.weight"], P[f"{name}.bias"] if bias else None, stride, pad)

    return Module(name, "conv", shape_fn, fwd, cout * cin * k * k, cout if bias else 0,
                  dict(cin=cin, cout=cout, k=k, stride=stride, pad=pad, bias=bias))


def bn_apply(x, P, name):
    return ops.batchnorm_eval(x, P[f"{name}.weight"], P[f"{name}.bias"],
                              P[f"{name}.running_mean"], P[f"{name}.running_var"])


def bn(name, c):
    return Module(name, "bn", lambda s: s, lambda x, P: bn_apply(x, P, name), 0, 2 * c, dict(c=c))


def relu(name):
    return Module(name, "relu", lambda s: s, lambda x, P: ops.relu(x))


def maxpool(name, k, stride, pad):
    def shape_fn(s):
        c, h, w = s
        return (c, ops.out_size(h, k, stride, pad), ops.out_size(w, k, stride, pad))
    return Module(name, "maxpool", shape_fn, lambda x, P: ops.maxpool2d(x, k, stride, pad),
                  meta=dict(k=k, stride=stride, pad=pad))


def avgpool(name, k, stride):
    def shape_fn(s):
        c, h, w = s
        return (c, ops.out_size(h, k, stride, 0), ops.out_size(w, k, stride, 0))
    return Module(name, "avgpool", shape_fn, lambda x, P: ops.avgpool2d(x, k, stride),
                  meta=dict(k=k, stride=stride))


def adaptive_avgpool(name, oh, ow):
    return Module(name, "adaptive_avgpool", lambda s: (s[0], oh, ow),
                  lambda x, P: ops.adaptive_avgpool2d(x, oh, ow), meta=dict(oh=oh, ow=ow))


def dropout(name):
    """Dropout = identity in eval mode; the classifier's first module sees the
    flattened input (torchvision forward calls torch.flatten before classifier)."""
    return Module(name, "dropout", lambda s: (_numel(s),), lambda x, P: ops.flatten(x))


def linear(name, fin, fout):
    def shape_fn(s):
        assert _numel(s) == fin, (name, s)
        return (fout,)
    return Module(name, "linear", shape_fn,
                  lambda x, P: ops.linear(x, P[f"{name}.weight"], P[f"{name}.bias"]),
                  fout * fin, fout, dict(fin=fin, fout=fout))


def basic_block(name, cin, planes, stride):
    ds = stride != 1 or cin != planes

    def shape_fn(s):
        c, h, w = s
        assert c == cin
        return (planes, ops.out_size(h, 3, stride, 1), ops.out_size(w, 3, stride, 1))

    def fwd(x, P):
        # relu(bn2(conv2(relu(bn1(conv1 x)))) + ds(x))
        t = ops.relu(bn_apply(ops.conv2d(x, P[f"{name}.conv1.weight"], None, stride, 1), P, f"{name}.bn1"))
        t = bn_apply(ops.conv2d(t, P[f"{name}.conv2.weight"], None, 1, 1), P, f"{name}.bn2")
        idn = x
        if ds:
            idn = bn_apply(ops.conv2d(x, P[f"{name}.downsample.0.weight"], None, stride, 0), P,
                           f"{name}.downsample.1")
        return ops.relu(t + idn)

    we = planes * cin * 9 + planes * planes * 9 + (planes * cin if ds else 0)
    ve = 2 * planes * 2 + (2 * planes if ds else 0)
    return Module(name, "basic_block", shape_fn, fwd, we, ve,
                  dict(cin=cin, planes=planes, stride=stride, ds=ds))


def bottleneck(name, cin, planes, stride):
    cout = planes * 4
    ds = stride != 1 or cin != cout

    def shape_fn(s):
        c, h, w = s
        assert c == cin
        return (cout, ops.out_size(h, 3, stride, 1), ops.out_size(w, 3, stride, 1))

    def fwd(x, P):
        # torchvision v1.5: the stride sits on the 3x3 conv (reading A12)
        t = ops.relu(bn_apply(ops.conv2d(x, P[f"{name}.conv1.weight"], None, 1, 0), P, f"{name}.bn1"))
        t = ops.relu(bn_apply(ops.conv2d(t, P[f"{name}.conv2.weight"], None, stride, 1), P, f"{name}.bn2"))
        t = bn_apply(ops.conv2d(t, P[f"{name}.conv3.weight"], None, 1, 0), P, f"{name}.bn3")
        idn = x
        if ds:
            idn = bn_apply(ops.conv2d(x, P[f"{name}.downsample.0.weight"], None, stride, 0), P,
                           f"{name}.downsample.1")
        return ops.relu(t + idn)

    we = planes * cin + planes * planes * 9 + cout * planes + (cout * cin if ds else 0)
    ve = 2 * (planes + planes + cout) + (2 * cout if ds else 0)
    return Module(name, "bottleneck", shape_fn, fwd, we, ve,
                  dict(cin=cin, planes=planes, stride=stride, ds=ds))


def dense_block(name, nlayers, cin, growth=32, bn_size=4):
    cout = cin + nlayers * growth
    mid = bn_size * growth

    def shape_fn(s):
        c, h, w = s
        assert c == cin
        return (cout, h, w)

    def fwd(x, P):
        feats = [x]
        for j in range(nlayers):
            p = f"{name}.denselayer{j + 1}"
            cat = np.concatenate(feats, axis=1)
            # concat[x, conv2(relu(bn2(conv1(relu(bn1 x)))))]
            t = ops.conv2d(ops.relu(bn_apply(cat, P, f"{p}.norm1")), P[f"{p}.conv1.weight"], None, 1, 0)
            t = ops.conv2d(ops.relu(bn_apply(t, P, f"{p}.norm2")), P[f"{p}.conv2.weight"], None, 1, 1)
            feats.append(t)
        return np.concatenate(feats, axis=1)

    we = sum(mid * (cin + j * growth) + growth * mid * 9 for j in range(nlayers))
    ve = sum(2 * (cin + j * growth) + 2 * mid for j in range(nlayers))
    return Module(name, "dense_block", shape_fn, fwd, we, ve,
                  dict(cin=cin, nlayers=nlayers, growth=growth, bn_size=bn_size))


def densenet_classifier(name, fin, fout):
    """relu -> adaptive_avg_pool(1) -> flatten -> linear (torchvision DenseNet.forward)."""
    def fwd(x, P):
        t = ops.adaptive_avgpool2d(ops.relu(x), 1, 1)
        return ops.linear(t, P[f"{name}.weight"], P[f"{name}.bias"])
    return Module(name, "densenet_classifier", lambda s: (fout,), fwd, fout * fin, fout,
                  dict(fin=fin, fout=fout))


# ---------------------------------------------------------------- architectures

def alexnet() -> List[Module]:
    return [
        conv("features.0", 3, 64, 11, 4, 2, True), relu("features.1"), maxpool("features.2", 3, 2, 0),
        conv("features.3", 64, 192, 5, 1, 2, True), relu("features.4"), maxpool("features.5", 3, 2, 0),
        conv("features.6", 192, 384, 3, 1, 1, True), relu("features.7"),
        conv("features.8", 384, 256, 3, 1, 1, True), relu("features.9"),
        conv("features.10", 256, 256, 3, 1, 1, True), relu("features.11"), maxpool("features.12", 3, 2, 0),
        adaptive_avgpool("avgpool", 6, 6),
        dropout("classifier.0"), linear("classifier.1", 9216, 4096), relu("classifier.2"),
        dropout("classifier.3"), linear("classifier.4", 4096, 4096), relu("classifier.5"),
        linear("classifier.6", 4096, 1000),
    ]


def _resnet(block, layers) -> List[Module]:
    mods = [conv("conv1", 3, 64, 7, 2, 3, False), bn("bn1", 64), relu("relu"), maxpool("maxpool", 3, 2, 1)]
    cin, exp = 64, (1 if block is basic_block else 4)
    for li, (planes, n) in enumerate(zip((64, 128, 256, 512), layers)):
        for bi in range(n):
            stride = 2 if (li > 0 and bi == 0) else 1
            mods.append(block(f"layer{li + 1}.{bi}", cin, planes, stride))
            cin = planes * exp
    mods.append(adaptive_avgpool("avgpool", 1, 1))
    fc = linear("fc", cin, 1000)
    mods.append(fc)
    return mods


def resnet18():
    return _resnet(basic_block, (2, 2, 2, 2))


def resnet50():
    return _resnet(bottleneck, (3, 4, 6, 3))


def vgg11() -> List[Module]:
    cfg = [64, "M", 128, "M", 256, 256, "M", 512, 512, "M", 512, 512, "M"]
    mods, idx, cin = [], 0, 3
    for v in cfg:
        if v == "M":
            mods.append(maxpool(f"features.{idx}", 2, 2, 0))
            idx += 1
        else:
            mods += [conv(f"features.{idx}", cin, v, 3, 1, 1, True), relu(f"features.{idx + 1}")]
            cin = v
            idx += 2
    mods.append(adaptive_avgpool("avgpool", 7, 7))
    mods += [linear("classifier.0", 25088, 4096), relu("classifier.1"), dropout("classifier.2"),
             linear("classifier.3", 4096, 4096), relu("classifier.4"), dropout("classifier.5"),
             linear("classifier.6", 4096, 1000)]
    return mods


def densenet121() -> List[Module]:
    mods = [conv("features.conv0", 3, 64, 7, 2, 3, False), bn("features.norm0", 64),
            relu("features.relu0"), maxpool("features.pool0", 3, 2, 1)]
    c = 64
    for bi, n in enumerate((6, 12, 24, 16)):
        mods.append(dense_block(f"features.denseblock{bi + 1}", n, c))
        c += 32 * n
        if bi != 3:
            p = f"features.transition{bi + 1}"
            mods += [bn(f"{p}.norm", c), relu(f"{p}.relu"), conv(f"{p}.conv", c, c // 2, 1, 1, 0, False),
                     avgpool(f"{p}.pool", 2, 2)]
            c //= 2
    mods.append(bn("features.norm5", c))
    mods.append(densenet_classifier("classifier", c, 1000))
    return mods


ARCHS = {"alexnet": alexnet, "resnet18": resnet18, "resnet50": resnet50, "vgg11": vgg11,
         "densenet121": densenet121}


def layers(arch: str) -> List[Module]:
    return ARCHS[arch]()


def shapes(arch: str, in_h: int = 224, in_w: int = 224) -> List[Tuple[int, ...]]:
    """Per-image output shape of every layer s = 1..L (closed-form shape rules)."""
    s = (3, in_h, in_w)
    out = []
    for m in layers(arch):
        s = m.shape_fn(s)
        out.append(s)
    return out
