"""u8 ingest (optional): uint8 NCHW images normalised by the input pack kernel
(x = scale[c] * u + shift[c], one FFMA in fp32).  Checked against the oracle
(oracle.prefix.normalize_u8 then the fp64 prefix), bitwise against the fp32 path fed with the
same normalised values (single-rounded, as the FFMA does), host vs device paths bitwise, and a
scale/shift change after graph capture taking effect."""
import numpy as np
import pytest

import hapi_inputs
from oracle import prefix
from tests.parity_check import check_close

pytestmark = pytest.mark.gpu

# ImageNet normalisation as a caller would fold it: (u / 255 - mean) / std
MEAN = np.array([0.485, 0.456, 0.406])
STD = np.array([0.229, 0.224, 0.225])
SCALE = (1.0 / (255.0 * STD)).astype(np.float32)
SHIFT = (-MEAN / STD).astype(np.float32)


def _fp32_images(u8, scale, shift):
    # fmaf(u, scale, shift): the fp64 value of scale * u + shift is exact (24 + 8 bit
    # product), so one rounding to fp32 reproduces the kernel's FFMA bit for bit
    sc = np.asarray(scale, np.float32).astype(np.float64).reshape(1, 3, 1, 1)
    sh = np.asarray(shift, np.float32).astype(np.float64).reshape(1, 3, 1, 1)
    return (sc * u8.astype(np.float64) + sh).astype(np.float32)


def _out(model, split, n, act, host=False):
    import torch
    es = 4 if act == "f32" else 2
    return torch.empty(model.out_bytes[split - 1] // es * n, dtype=torch.float32 if act == "f32" else torch.bfloat16,
                       device="cpu" if host else "cuda")


@pytest.mark.parametrize("arch,act,size,splits", [
    ("resnet50", "bf16", 96, [1, 4, 21]),     # space-to-depth pack (layout 2)
    ("vgg11", "bf16", 64, [3, 11]),           # 3x3 stem packs (layout 3 / 4)
    ("densenet121", "bf16", 64, [9]),
    ("alexnet", "f32", 96, [2, 13]),          # fp32 NHWC pack (layout 0)
])
def test_u8_matches_oracle_and_fp32_path(arch, act, size, splits):
    import torch
    import paper_2210_08650_b200 as H
    n = 3
    P = hapi_inputs.params(arch, 61)
    u8 = hapi_inputs.images_u8(n, 62, size, size)
    m = H.Model(arch, act, list(P.values()), n, min(splits), max(splits), in_h=size, in_w=size)
    try:
        m.set_u8_norm(SCALE, SHIFT)
        xu = torch.from_numpy(u8).cuda()
        xf = torch.from_numpy(_fp32_images(u8, SCALE, SHIFT)).cuda()
        ref_all = prefix.prefix_forward_all(arch, P, prefix.normalize_u8(u8, SCALE, SHIFT), max(splits))
        for s in splits:
            a, b = _out(m, s, n, act), _out(m, s, n, act)
            m.forward_u8(s, xu, a)
            m.forward(s, xf, b)
            torch.cuda.synchronize()
            assert torch.equal(a.view(torch.int16 if act == "bf16" else torch.int32),
                               b.view(torch.int16 if act == "bf16" else torch.int32)), (arch, s)
            check_close(a.float().cpu().numpy().reshape(ref_all[s - 1].shape), ref_all[s - 1], act, f"u8 {arch} s={s}")
    finally:
        m.close()


def test_u8_host_paths_and_norm_change():
    import torch
    import paper_2210_08650_b200 as H
    arch, act, n, size, s = "resnet50", "bf16", 5, 96, 8
    P = hapi_inputs.params(arch, 63)
    u8 = hapi_inputs.images_u8(n, 64, size, size)
    m = H.Model(arch, act, list(P.values()), n, s, s, in_h=size, in_w=size, host_chunk=2)
    try:
        xu = torch.from_numpy(u8).cuda()
        dev = _out(m, s, n, act)
        m.forward_u8(s, xu, dev)                       # default scale 1/255, shift 0; graph captured
        torch.cuda.synchronize()
        want = _out(m, s, n, act)
        m.forward(s, torch.from_numpy(_fp32_images(u8, [1 / 255.0] * 3, [0.0] * 3)).cuda(), want)
        torch.cuda.synchronize()
        assert torch.equal(dev.view(torch.int16), want.view(torch.int16))
        m.set_u8_norm(SCALE, SHIFT)                    # must take effect on the captured graph's next replay
        m.forward_u8(s, xu, dev)
        torch.cuda.synchronize()
        m.forward(s, torch.from_numpy(_fp32_images(u8, SCALE, SHIFT)).cuda(), want)
        torch.cuda.synchronize()
        assert torch.equal(dev.view(torch.int16), want.view(torch.int16))
        hu = torch.from_numpy(u8).pin_memory()
        h1, h2 = _out(m, s, n, act, True).pin_memory(), _out(m, s, n, act, True).pin_memory()
        m.forward_host_u8(s, hu, h1)                   # 5 images in chunks of 2: ragged last chunk
        m.forward_host_async_u8(s, hu, h2)
        m.host_sync()
        d = dev.cpu()
        assert torch.equal(h1.view(torch.int16), d.view(torch.int16))
        assert torch.equal(h2.view(torch.int16), d.view(torch.int16))
        ref = prefix.prefix_forward(arch, P, prefix.normalize_u8(u8, SCALE, SHIFT), s)
        check_close(d.float().numpy().reshape(ref.shape), ref, act, "u8 host")
        with pytest.raises(ValueError):
            m.forward_u8(s, xu.float(), dev)           # wrong dtype
        with pytest.raises(ValueError):
            m.set_u8_norm([1.0, 2.0], [0.0, 0.0, 0.0])
    finally:
        m.close()


def test_u8_bench_size_sampled():
    """The u8 ingest at the bench's launch configuration (ResNet50 s=21, batch 512, the
    fused blocks on): the whole batch bitwise equal to the fp32 path fed the same
    normalised values, and sampled images checked against the oracle one by one."""
    import torch
    import paper_2210_08650_b200 as H
    arch, act, n, s, sel = "resnet50", "bf16", 512, 21, [0, 1, 510, 511]
    P = hapi_inputs.params(arch, 65)
    u8 = hapi_inputs.images_u8(n, 66, 224, 224)
    m = H.Model(arch, act, list(P.values()), n, s, s)
    try:
        m.set_u8_norm(SCALE, SHIFT)
        a, b = _out(m, s, n, act), _out(m, s, n, act)
        m.forward_u8(s, torch.from_numpy(u8).cuda(), a)
        m.forward(s, torch.from_numpy(_fp32_images(u8, SCALE, SHIFT)).cuda(), b)
        torch.cuda.synchronize()
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
        got = a.float().cpu().numpy().reshape(n, -1)[sel]
        ref = prefix.prefix_forward(arch, P, prefix.normalize_u8(np.ascontiguousarray(u8[sel]), SCALE, SHIFT), s)
        check_close(got.reshape(ref.shape), ref, act, "u8 resnet50 s=21 b512 sampled")
    finally:
        m.close()
