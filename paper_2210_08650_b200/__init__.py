"""HAPI (arXiv 2210.08650) storage-side prefix forward, B200-native.

Python face of the C ABI in include/hapi.h (same names, argument marshalling only).
PyTorch is used for device memory and streams; all compute runs in libhapi.so
(tcgen05/TMEM/TMA implicit-GEMM convolutions for bf16, SIMT FFMA for fp32).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

from . import _lib
from ._lib import SplitQuery, lib  # noqa: F401

ARCHS = {"alexnet": 0, "resnet18": 1, "resnet50": 2, "vgg11": 3, "densenet121": 4}
DTYPES = {"f32": 0, "bf16": 1}
STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "INVALID_MODEL", 3: "INFEASIBLE", 4: "OUT_OF_MEMORY", 5: "CUDA",
          6: "UNSUPPORTED"}


class HapiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"HAPI_ERR_{STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st: int):
    if st != 0:
        raise HapiError(st, _lib.hapi_last_error().decode())


def _arch(a) -> int:
    return ARCHS[a] if isinstance(a, str) else int(a)


def _dt(d) -> int:
    return DTYPES[d] if isinstance(d, str) else int(d)


def build_info() -> str:
    return _lib.hapi_build_info().decode()


def hapi_num_layers(arch) -> int:
    n = _lib.hapi_num_layers(_arch(arch))
    if n < 0:
        raise HapiError(-n, "unknown arch")
    return n


def hapi_freeze_index(arch) -> int:
    return _lib.hapi_freeze_index(_arch(arch))


def hapi_layer_sizes(arch, in_h: int = 224, in_w: int = 224, act="f32"):
    """-> (l0, out_bytes[L], peak_bytes[L], weight_bytes[L])"""
    L = hapi_num_layers(arch)
    o, p, w, l0 = (_lib.u64 * L)(), (_lib.u64 * L)(), (_lib.u64 * L)(), _lib.u64()
    _check(_lib.hapi_layer_sizes(_arch(arch), in_h, in_w, _dt(act), C.byref(l0), o, p, w, L))
    return l0.value, list(o), list(p), list(w)


def hapi_choose_split(arch, freeze_idx: int, training_batch: int, link_bytes_per_s: int, hbm_budget_bytes: int,
                      b_min: int = 25, b_max: int = 2000, threshold_ms: int = 1000, act="f32", in_h: int = 224,
                      in_w: int = 224, raise_infeasible: bool = False):
    """Alg. 1 + Eq. 4.  Returns (status, SplitResult-as-dict, candidates)."""
    L = hapi_num_layers(arch)
    q = SplitQuery(_arch(arch), in_h, in_w, _dt(act), freeze_idx, training_batch, link_bytes_per_s, threshold_ms,
                   hbm_budget_bytes, b_min, b_max)
    r = _lib.SplitResult()
    cands = (_lib.u32 * L)()
    st = _lib.hapi_choose_split(C.byref(q), C.byref(r), cands)
    if st not in (0, 3) or (st == 3 and raise_infeasible):
        _check(st)
    res = dict(split_idx=r.split_idx, cos_batch=r.cos_batch, bytes_per_iteration=r.bytes_per_iteration,
               est_bytes=r.est_bytes, n_candidates=r.n_candidates)
    return ("ok" if st == 0 else "infeasible"), res, list(cands)[: r.n_candidates]


def hapi_adapt_batches(requests, available_bytes: int, max_concurrency: int = 0):
    """Section 4.5 batch adaptation (Eq. 4 over queued requests).  requests: iterable of
    (arrival_seq, model_bytes, data_bytes, b_min, b_max).  Returns (batches, used_bytes);
    batch 0 = deferred."""
    reqs = list(requests)
    arr = (_lib.AdaptRequest * max(len(reqs), 1))(*[_lib.AdaptRequest(*r) for r in reqs])
    out = (_lib.u32 * max(len(reqs), 1))()
    used = _lib.u64()
    _check(_lib.hapi_adapt_batches(arr, len(reqs), available_bytes, max_concurrency, out, C.byref(used)))
    return list(out)[: len(reqs)], used.value


def hapi_partition_requests(n: int, n_gpus: int):
    """GPU of each request in arrival order (round-robin)."""
    out = (_lib.u32 * max(n, 1))()
    _check(_lib.hapi_partition_requests(n, n_gpus, out))
    return list(out)[:n]


class Scheduler:
    """hapi_scheduler handle: the section 4.5 batch-adaptation loop of one GPU (host-only;
    the caller supplies the clock in microseconds)."""

    QUEUED, DEFERRED, RUNNING, DONE = 0, 1, 2, 3

    def __init__(self, total_bytes: int, occupied_bytes: int = 0, max_concurrency: int = 0, wait_us: int = 0):
        cfg = _lib.SchedulerConfig(total_bytes, occupied_bytes, max_concurrency, wait_us)
        h = C.c_void_p()
        _check(_lib.hapi_scheduler_create(C.byref(cfg), C.byref(h)))
        self._h = h

    def close(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(_lib, "hapi_scheduler_destroy", None) is not None:
            _lib.hapi_scheduler_destroy(h)
        self._h = None

    __del__ = close

    def submit(self, now_us: int, model_bytes: int, data_bytes: int, b_min: int, b_max: int) -> int:
        rid = _lib.u64()
        r = _lib.AdaptRequest(0, model_bytes, data_bytes, b_min, b_max)
        _check(_lib.hapi_scheduler_submit(self._h, now_us, C.byref(r), C.byref(rid)))
        return rid.value

    def poll(self, now_us: int, cap: int = 4096):
        """-> [(request id, COS batch)] admitted by a round at now_us ([] if none ran)."""
        ids, bs, n = (_lib.u64 * cap)(), (_lib.u32 * cap)(), _lib.u32()
        _check(_lib.hapi_scheduler_poll(self._h, now_us, ids, bs, cap, C.byref(n)))
        return [(ids[i], bs[i]) for i in range(n.value)]

    def finish(self, rid: int):
        _check(_lib.hapi_scheduler_finish(self._h, rid))

    def state(self, rid: int):
        st, b = _lib.u32(), _lib.u32()
        _check(_lib.hapi_scheduler_query(self._h, rid, C.byref(st), C.byref(b), None))
        return st.value, b.value

    def available(self) -> int:
        a = _lib.u64()
        _check(_lib.hapi_scheduler_query(self._h, 0, None, None, C.byref(a)))
        return a.value


class Server:
    """hapi_server handle: the section 4.5 serving loop of one GPU.  Requests carry device
    tensors (kept alive here until the request is DONE)."""

    def __init__(self, total_bytes: int, occupied_bytes: int = 0, max_concurrency: int = 0, wait_us: int = 0,
                 device: int = 0, b_min: int = 25):
        cfg = _lib.ServerConfig(_lib.SchedulerConfig(total_bytes, occupied_bytes, max_concurrency, wait_us), device,
                                b_min)
        h = C.c_void_p()
        _check(_lib.hapi_server_create(C.byref(cfg), C.byref(h)))
        self._h, self.device, self._keep = h, device, {}

    def close(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(_lib, "hapi_server_destroy", None) is not None:
            _lib.hapi_server_destroy(h)
        self._h = None
        self._keep = {}

    __del__ = close

    def add_model(self, arch, act, params: Sequence, min_split: int, max_split: int, in_h: int = 224,
                  in_w: int = 224) -> int:
        import numpy as np
        keep = [np.ascontiguousarray(np.asarray(p, dtype=np.float32)) for p in params]
        ptrs = (C.c_void_p * len(keep))(*[p.ctypes.data for p in keep])
        d = _lib.ModelDesc(_arch(arch), _dt(act), in_h, in_w, min_split, max_split, 1, self.device, 0)
        mid = _lib.u32()
        _check(_lib.hapi_server_add_model(self._h, C.byref(d), ptrs, len(keep), C.byref(mid)))
        return mid.value

    def submit(self, now_us: int, model_id: int, split_idx: int, b_max: int, images, out) -> int:
        import torch
        _need(isinstance(images, torch.Tensor) and images.is_cuda and images.is_contiguous()
              and images.dtype == torch.float32 and images.dim() == 4, "images: contiguous CUDA fp32 [N,3,H,W]")
        _need(isinstance(out, torch.Tensor) and out.is_cuda and out.is_contiguous(), "out: contiguous CUDA tensor")
        rid = _lib.u64()
        _check(_lib.hapi_server_submit(self._h, now_us, model_id, split_idx, b_max, C.c_void_p(images.data_ptr()),
                                       images.shape[0], C.c_void_p(out.data_ptr()), C.byref(rid)))
        self._keep[rid.value] = (images, out)
        return rid.value

    def step(self, now_us: int) -> int:
        n = _lib.u32()
        _check(_lib.hapi_server_step(self._h, now_us, C.byref(n)))
        for rid in [r for r in self._keep if self.state(r)[0] == Scheduler.DONE]:
            del self._keep[rid]
        return n.value

    def state(self, rid: int):
        st, b = _lib.u32(), _lib.u32()
        _check(_lib.hapi_server_query(self._h, rid, C.byref(st), C.byref(b), None))
        return st.value, b.value

    def device_bytes(self) -> int:
        t = _lib.u64()
        _check(_lib.hapi_server_query(self._h, 0, None, None, C.byref(t)))
        return t.value


def hapi_param_table(arch):
    """[(name, shape)] the library expects, in torchvision state_dict order."""
    n = _lib.hapi_num_params(_arch(arch))
    out = []
    buf = C.create_string_buffer(256)
    dims = (_lib.i64 * 4)()
    nd = _lib.u32()
    for i in range(n):
        _check(_lib.hapi_param_info(_arch(arch), i, buf, 256, dims, C.byref(nd)))
        out.append((buf.value.decode(), tuple(dims[: nd.value])))
    return out


def _need(cond: bool, msg: str):
    if not cond:
        raise ValueError(msg)


class Model:
    """hapi_model handle.  `params`: sequence of fp32 C-contiguous arrays (numpy or CPU
    torch tensors) in hapi_param_table order."""

    def __init__(self, arch, act, params: Sequence, max_batch: int, min_split: int, max_split: Optional[int] = None,
                 in_h: int = 224, in_w: int = 224, device: int = 0, start_idx: int = 0, host_chunk: int = 0):
        """start_idx > 0: a client-side suffix model (input = layer start_idx's NCHW output,
        computes layers start_idx+1 .. split; use forward_suffix).  host_chunk > 0: staging
        for forward_host (chunks of that many images) is allocated here; -1 picks the
        measured default (3/16 of max_batch rounded to 16, at least 64, at most max_batch)."""
        import numpy as np
        max_split = min_split if max_split is None else max_split
        self.arch, self.act = arch, act
        self.in_h, self.in_w, self.max_batch = in_h, in_w, max_batch
        self.min_split, self.max_split = min_split, max_split
        keep = [np.ascontiguousarray(np.asarray(p, dtype=np.float32)) for p in params]
        ptrs = (C.c_void_p * len(keep))(*[p.ctypes.data for p in keep])
        if host_chunk < 0:
            host_chunk = max_batch if max_batch < 256 else min(max_batch, max(64, (max_batch * 3 // 16 + 15) // 16 * 16))
        d = _lib.ModelDesc(_arch(arch), _dt(act), in_h, in_w, min_split, max_split, max_batch, device, host_chunk)
        h = C.c_void_p()
        if start_idx:
            _check(_lib.hapi_model_create_suffix(C.byref(d), start_idx, ptrs, len(keep), C.byref(h)))
        else:
            _check(_lib.hapi_model_create(C.byref(d), ptrs, len(keep), C.byref(h)))
        self.start_idx = start_idx
        self._h = h
        self.device = device
        self.out_bytes = hapi_layer_sizes(arch, in_h, in_w, act)[1]

    def shared(self, max_batch: int, host_chunk: int = 0) -> "Model":
        """hapi_model_create_shared: a model over this model's device weights (no copy) with
        its own arena for max_batch images -- one per concurrent request."""
        if host_chunk < 0:
            host_chunk = max_batch if max_batch < 256 else min(max_batch, max(64, (max_batch * 3 // 16 + 15) // 16 * 16))
        h = C.c_void_p()
        _check(_lib.hapi_model_create_shared(self._h, max_batch, host_chunk, C.byref(h)))
        m = object.__new__(Model)
        m.__dict__.update({k: v for k, v in self.__dict__.items() if k != "_h"})
        m.max_batch, m._h = max_batch, h
        return m

    def close(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(_lib, "hapi_model_destroy", None) is not None:
            _lib.hapi_model_destroy(h)
        self._h = None

    __del__ = close

    def set_stream(self, stream_ptr: int):
        _check(_lib.hapi_model_set_stream(self._h, C.c_void_p(stream_ptr)))

    def out_shape(self, split_idx: int, batch: int):
        return batch, self.out_bytes[split_idx - 1] // (4 if self.act == "f32" else 2)

    def _split_bytes(self, idx: int) -> int:
        _need(1 <= idx <= len(self.out_bytes), f"layer index {idx} outside [1, {len(self.out_bytes)}]")
        return self.out_bytes[idx - 1]

    def _check_images(self, images, on_device: bool, u8: bool = False):
        import torch
        _need(isinstance(images, torch.Tensor), "images must be a torch tensor")
        want = torch.uint8 if u8 else torch.float32
        _need(images.dtype == want, f"images must be {want}, got {images.dtype}")
        _need(images.dim() == 4 and tuple(images.shape[1:]) == (3, self.in_h, self.in_w),
              f"images must be [N,3,{self.in_h},{self.in_w}], got {tuple(images.shape)}")
        _need(images.is_contiguous(), "images must be contiguous")
        if on_device:
            _need(images.is_cuda and images.device.index == self.device,
                  f"images must be on cuda:{self.device}, got {images.device}")
        else:
            _need(not images.is_cuda, "forward_host takes host (CPU) tensors")

    def _check_out(self, out, need_bytes: int, on_device: bool):
        import torch
        _need(isinstance(out, torch.Tensor), "out must be a torch tensor")
        want = torch.float32 if self.act == "f32" else torch.bfloat16
        _need(out.dtype == want, f"out must be {want}, got {out.dtype}")
        _need(out.is_contiguous(), "out must be contiguous")
        _need(out.numel() * out.element_size() >= need_bytes, f"out holds {out.numel() * out.element_size()} bytes, "
              f"needs {need_bytes}")
        if on_device:
            _need(out.is_cuda and out.device.index == self.device, f"out must be on cuda:{self.device}")
        else:
            _need(not out.is_cuda, "forward_host writes a host (CPU) tensor")

    def forward(self, split_idx: int, images, out):
        """images: CUDA fp32 [batch,3,H,W] contiguous tensor; out: CUDA tensor with room
        for the split output (act dtype).  Launches on the model's stream."""
        self._check_images(images, True)
        self._check_out(out, images.shape[0] * self._split_bytes(split_idx), True)
        _check(_lib.hapi_prefix_forward(self._h, split_idx, C.c_void_p(images.data_ptr()), images.shape[0],
                                        C.c_void_p(out.data_ptr())))
        return out

    def forward_suffix(self, end_idx: int, acts, out):
        """acts: CUDA tensor holding layer start_idx's output (NCHW, act dtype); out: CUDA
        tensor with room for layer end_idx's output."""
        import torch
        _need(isinstance(acts, torch.Tensor) and acts.is_cuda and acts.device.index == self.device,
              f"acts must be a tensor on cuda:{self.device}")
        _need(acts.is_contiguous() and acts.dtype == (torch.float32 if self.act == "f32" else torch.bfloat16),
              "acts must be contiguous, in the model's act dtype")
        n = acts.shape[0]
        _need(acts.numel() * acts.element_size() == n * self._split_bytes(self.start_idx),
              f"acts must hold {n} layer-{self.start_idx} outputs")
        self._check_out(out, n * self._split_bytes(end_idx), True)
        _check(_lib.hapi_suffix_forward(self._h, end_idx, C.c_void_p(acts.data_ptr()), acts.shape[0],
                                        C.c_void_p(out.data_ptr())))
        return out

    def forward_host(self, split_idx: int, images, out):
        """HOST buffers (CPU torch tensors, ideally pinned); synchronous end-to-end call.
        Needs a model created with host_chunk != 0."""
        self._check_images(images, False)
        self._check_out(out, images.shape[0] * self._split_bytes(split_idx), False)
        ip, op = images.data_ptr(), out.data_ptr()
        _check(_lib.hapi_prefix_forward_host(self._h, split_idx, C.c_void_p(ip), images.shape[0], C.c_void_p(op)))
        return out

    def forward_host_async(self, split_idx: int, images, out):
        """Enqueue a host-buffer call without waiting (hapi_prefix_forward_host_async): keep
        `images` and `out` alive and untouched until host_sync()."""
        self._check_images(images, False)
        self._check_out(out, images.shape[0] * self._split_bytes(split_idx), False)
        _check(_lib.hapi_prefix_forward_host_async(self._h, split_idx, C.c_void_p(images.data_ptr()), images.shape[0],
                                                   C.c_void_p(out.data_ptr())))
        return out

    def host_sync(self):
        _check(_lib.hapi_host_sync(self._h))

    # u8 ingest: uint8 NCHW images, x = scale[c] * u + shift[c] applied by the input pack kernel
    def set_u8_norm(self, scale, shift):
        """Per-channel affine of the u8 calls (3 finite floats each; default 1/255, 0)."""
        sc = [float(v) for v in scale]
        sh = [float(v) for v in shift]
        _need(len(sc) == 3 and len(sh) == 3, "scale and shift take 3 values (one per channel)")
        _check(_lib.hapi_model_set_u8_norm(self._h, (C.c_float * 3)(*sc), (C.c_float * 3)(*sh)))

    def forward_u8(self, split_idx: int, images, out):
        """images: CUDA uint8 [batch,3,H,W] contiguous tensor; otherwise as forward()."""
        self._check_images(images, True, u8=True)
        self._check_out(out, images.shape[0] * self._split_bytes(split_idx), True)
        _check(_lib.hapi_prefix_forward_u8(self._h, split_idx, C.c_void_p(images.data_ptr()), images.shape[0],
                                           C.c_void_p(out.data_ptr())))
        return out

    def forward_host_u8(self, split_idx: int, images, out):
        """Host uint8 images (ideally pinned); synchronous, as forward_host()."""
        self._check_images(images, False, u8=True)
        self._check_out(out, images.shape[0] * self._split_bytes(split_idx), False)
        _check(_lib.hapi_prefix_forward_host_u8(self._h, split_idx, C.c_void_p(images.data_ptr()), images.shape[0],
                                                C.c_void_p(out.data_ptr())))
        return out

    def forward_host_async_u8(self, split_idx: int, images, out):
        """Host uint8 images, enqueued without waiting, as forward_host_async()."""
        self._check_images(images, False, u8=True)
        self._check_out(out, images.shape[0] * self._split_bytes(split_idx), False)
        _check(_lib.hapi_prefix_forward_host_async_u8(self._h, split_idx, C.c_void_p(images.data_ptr()),
                                                      images.shape[0], C.c_void_p(out.data_ptr())))
        return out

    def forward_timed(self, split_idx: int, images, out) -> List[float]:
        self._check_images(images, True)
        self._check_out(out, images.shape[0] * self._split_bytes(split_idx), True)
        n = self.plan_info(split_idx)["n"]
        ms = (C.c_float * n)()
        _check(_lib.hapi_prefix_forward_timed(self._h, split_idx, C.c_void_p(images.data_ptr()), images.shape[0],
                                              C.c_void_p(out.data_ptr()), ms, n))
        return list(ms)

    def device_bytes(self):
        w, a = _lib.u64(), _lib.u64()
        _check(_lib.hapi_model_device_bytes(self._h, C.byref(w), C.byref(a)))
        return w.value, a.value

    def plan_info(self, split_idx: int):
        n = _lib.u32()
        _check(_lib.hapi_plan_info(self._h, split_idx, C.byref(n), None, None, None, 0))
        k = (_lib.u32 * n.value)()
        fl = (C.c_double * n.value)()
        by = (C.c_double * n.value)()
        _check(_lib.hapi_plan_info(self._h, split_idx, C.byref(n), k, fl, by, n.value))
        buf = C.create_string_buffer(256)
        desc = []
        for i in range(n.value):
            _check(_lib.hapi_plan_describe(self._h, split_idx, i, buf, 256))
            desc.append(buf.value.decode())
        return dict(n=n.value, kind=list(k), flops=list(fl), bytes=list(by), desc=desc)


KERNEL_CLASSES = {0: "conv_tc", 1: "conv_simt", 2: "pool", 3: "pack", 4: "eltwise"}
