"""Thin ctypes binding of include/hapi.h.  Argument marshalling only: every step of
the hot path runs inside libhapi.so.  There is no CPU fallback -- if the library is
missing this module raises at import time."""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HAPI_LIB") or os.path.join(_PKG, "libhapi.so")  # HAPI_LIB: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python paper_2210_08650_b200/build.py` "
                      "(there is no CPU fallback for the HAPI prefix forward)")
lib = C.CDLL(LIB_PATH)

u32, u64, i32, i64 = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64
P_u64, P_u32, P_dbl, P_f32 = C.POINTER(u64), C.POINTER(u32), C.POINTER(C.c_double), C.POINTER(C.c_float)


class SplitQuery(C.Structure):
    _fields_ = [("arch", C.c_int), ("in_h", u32), ("in_w", u32), ("act", C.c_int), ("freeze_idx", u32),
                ("training_batch", u64), ("link_bytes_per_s", u64), ("threshold_ms", u32),
                ("hbm_budget_bytes", u64), ("b_min", u32), ("b_max", u32)]


class SplitResult(C.Structure):
    _fields_ = [("split_idx", u32), ("cos_batch", u32), ("bytes_per_iteration", u64), ("est_bytes", u64),
                ("n_candidates", u32)]


class AdaptRequest(C.Structure):
    _fields_ = [("arrival_seq", u64), ("model_bytes", u64), ("data_bytes", u64), ("b_min", u32), ("b_max", u32)]


class ModelDesc(C.Structure):
    _fields_ = [("arch", C.c_int), ("act", C.c_int), ("in_h", u32), ("in_w", u32), ("min_split", u32),
                ("max_split", u32), ("max_batch", u32), ("device", C.c_int), ("host_chunk", u32)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


hapi_num_layers = _sig("hapi_num_layers", i32, C.c_int)
hapi_freeze_index = _sig("hapi_freeze_index", i32, C.c_int)
hapi_layer_sizes = _sig("hapi_layer_sizes", C.c_int, C.c_int, u32, u32, C.c_int, P_u64, P_u64, P_u64, P_u64, u32)
hapi_choose_split = _sig("hapi_choose_split", C.c_int, C.POINTER(SplitQuery), C.POINTER(SplitResult), P_u32)
hapi_adapt_batches = _sig("hapi_adapt_batches", C.c_int, C.POINTER(AdaptRequest), u32, u64, u32, P_u32, P_u64)
hapi_partition_requests = _sig("hapi_partition_requests", C.c_int, u32, u32, P_u32)
hapi_num_params = _sig("hapi_num_params", i32, C.c_int)
hapi_param_info = _sig("hapi_param_info", C.c_int, C.c_int, u32, C.c_char_p, u32, C.POINTER(i64), P_u32)
hapi_model_create = _sig("hapi_model_create", C.c_int, C.POINTER(ModelDesc), C.POINTER(C.c_void_p), u32,
                         C.POINTER(C.c_void_p))
hapi_model_create_suffix = _sig("hapi_model_create_suffix", C.c_int, C.POINTER(ModelDesc), u32, C.POINTER(C.c_void_p),
                                u32, C.POINTER(C.c_void_p))
hapi_suffix_forward = _sig("hapi_suffix_forward", C.c_int, C.c_void_p, u32, C.c_void_p, u64, C.c_void_p)
hapi_model_create_shared = _sig("hapi_model_create_shared", C.c_int, C.c_void_p, u32, u32, C.POINTER(C.c_void_p))
hapi_model_set_stream = _sig("hapi_model_set_stream", C.c_int, C.c_void_p, C.c_void_p)
hapi_prefix_forward = _sig("hapi_prefix_forward", C.c_int, C.c_void_p, u32, C.c_void_p, u64, C.c_void_p)
hapi_prefix_forward_host = _sig("hapi_prefix_forward_host", C.c_int, C.c_void_p, u32, C.c_void_p, u64, C.c_void_p)
hapi_prefix_forward_host_async = _sig("hapi_prefix_forward_host_async", C.c_int, C.c_void_p, u32, C.c_void_p, u64,
                                      C.c_void_p)
hapi_host_sync = _sig("hapi_host_sync", C.c_int, C.c_void_p)
P_f32 = C.POINTER(C.c_float)
hapi_model_set_u8_norm = _sig("hapi_model_set_u8_norm", C.c_int, C.c_void_p, P_f32, P_f32)
hapi_prefix_forward_u8 = _sig("hapi_prefix_forward_u8", C.c_int, C.c_void_p, u32, C.c_void_p, u64, C.c_void_p)
hapi_prefix_forward_host_u8 = _sig("hapi_prefix_forward_host_u8", C.c_int, C.c_void_p, u32, C.c_void_p, u64, C.c_void_p)
hapi_prefix_forward_host_async_u8 = _sig("hapi_prefix_forward_host_async_u8", C.c_int, C.c_void_p, u32, C.c_void_p, u64,
                                         C.c_void_p)
hapi_model_device_bytes = _sig("hapi_model_device_bytes", C.c_int, C.c_void_p, P_u64, P_u64)
hapi_plan_info = _sig("hapi_plan_info", C.c_int, C.c_void_p, u32, P_u32, P_u32, P_dbl, P_dbl, u32)
hapi_prefix_forward_timed = _sig("hapi_prefix_forward_timed", C.c_int, C.c_void_p, u32, C.c_void_p, u64, C.c_void_p,
                                 P_f32, u32)
hapi_plan_describe = _sig("hapi_plan_describe", C.c_int, C.c_void_p, u32, u32, C.c_char_p, u32)
hapi_model_destroy = _sig("hapi_model_destroy", None, C.c_void_p)
class SchedulerConfig(C.Structure):
    _fields_ = [("total_bytes", u64), ("occupied_bytes", u64), ("max_concurrency", u32), ("wait_us", u64)]


hapi_scheduler_create = _sig("hapi_scheduler_create", C.c_int, C.POINTER(SchedulerConfig), C.POINTER(C.c_void_p))
hapi_scheduler_submit = _sig("hapi_scheduler_submit", C.c_int, C.c_void_p, u64, C.POINTER(AdaptRequest), P_u64)
hapi_scheduler_poll = _sig("hapi_scheduler_poll", C.c_int, C.c_void_p, u64, P_u64, P_u32, u32, P_u32)
hapi_scheduler_finish = _sig("hapi_scheduler_finish", C.c_int, C.c_void_p, u64)
hapi_scheduler_query = _sig("hapi_scheduler_query", C.c_int, C.c_void_p, u64, P_u32, P_u32, P_u64)
hapi_scheduler_destroy = _sig("hapi_scheduler_destroy", None, C.c_void_p)
class ServerConfig(C.Structure):
    _fields_ = [("sched", SchedulerConfig), ("device", C.c_int), ("b_min", u32)]


hapi_server_create = _sig("hapi_server_create", C.c_int, C.POINTER(ServerConfig), C.POINTER(C.c_void_p))
hapi_server_add_model = _sig("hapi_server_add_model", C.c_int, C.c_void_p, C.POINTER(ModelDesc), C.POINTER(C.c_void_p),
                             u32, P_u32)
hapi_server_submit = _sig("hapi_server_submit", C.c_int, C.c_void_p, u64, u32, u32, u32, C.c_void_p, u64, C.c_void_p,
                          P_u64)
hapi_server_step = _sig("hapi_server_step", C.c_int, C.c_void_p, u64, P_u32)
hapi_server_query = _sig("hapi_server_query", C.c_int, C.c_void_p, u64, P_u32, P_u32, P_u64)
hapi_server_destroy = _sig("hapi_server_destroy", None, C.c_void_p)
hapi_last_error = _sig("hapi_last_error", C.c_char_p)
hapi_build_info = _sig("hapi_build_info", C.c_char_p)

EXPORTED = ["hapi_num_layers", "hapi_freeze_index", "hapi_layer_sizes", "hapi_choose_split", "hapi_adapt_batches",
            "hapi_partition_requests", "hapi_model_create_suffix", "hapi_suffix_forward", "hapi_num_params",
            "hapi_param_info", "hapi_model_create", "hapi_model_set_stream", "hapi_prefix_forward",
            "hapi_prefix_forward_host", "hapi_model_device_bytes", "hapi_plan_info", "hapi_plan_describe", "hapi_prefix_forward_timed",
            "hapi_model_destroy", "hapi_last_error", "hapi_build_info", "hapi_scheduler_create",
            "hapi_scheduler_submit", "hapi_scheduler_poll", "hapi_scheduler_finish", "hapi_scheduler_query",
            "hapi_scheduler_destroy", "hapi_model_create_shared", "hapi_server_create", "hapi_server_add_model",
            "hapi_server_submit", "hapi_server_step", "hapi_server_query", "hapi_server_destroy",
            "hapi_prefix_forward_host_async", "hapi_host_sync", "hapi_model_set_u8_norm", "hapi_prefix_forward_u8",
            "hapi_prefix_forward_host_u8", "hapi_prefix_forward_host_async_u8"]
