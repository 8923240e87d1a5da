"""ctypes binding of libmoe_eamc.so (include/moe_eamc.h).

The library is built in-tree (paper_2401_14361_b200/libmoe_eamc.so) for
sm_100a.  There is no Python or CPU fallback: if the shared library is
missing this module raises ImportError, and on a machine without an sm_100
GPU every compute entry point returns MOE_ERR_CUDA, surfaced as CudaError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MOE_LIB") or os.path.join(HERE, "libmoe_eamc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        " (or `make -C paper_2401_14361_b200/csrc`). There is no CPU fallback.")

lib = C.CDLL(LIB_PATH)

MOE_OK = 0
MOE_ERR_INVALID_ARGUMENT = 1
MOE_ERR_OUT_OF_RANGE = 2
MOE_ERR_SNAPSHOT = 3
MOE_ERR_LOGIC = 4
MOE_ERR_CUDA = 5
MOE_ERR_NCCL = 6
MOE_ERR_OOM = 7
MOE_ERR_OVERFLOW = 8
MOE_ERR_TRACE = 9

NONE = 0xFFFFFFFFFFFFFFFF


class moe_shape(C.Structure):
    _fields_ = [("n_layers", C.c_uint32), ("n_experts_per_layer", C.c_uint32),
                ("top_k", C.c_uint32)]


class moe_match(C.Structure):
    _fields_ = [("index", C.c_uint64), ("seq", C.c_uint64), ("distance", C.c_double)]


MATCH_DTYPE = np.dtype([("index", np.uint64), ("seq", np.uint64), ("distance", np.float64)])


class moe_candidate(C.Structure):
    _fields_ = [("layer_idx", C.c_uint32), ("expert_idx", C.c_uint32), ("priority", C.c_double)]


CAND_DTYPE = np.dtype([("layer_idx", np.uint32), ("expert_idx", np.uint32),
                       ("priority", np.float64)])

SLOT_DTYPE = np.dtype([("slot", np.uint64), ("layer_idx", np.uint32), ("expert_idx", np.uint32),
                       ("prefetch_protected", np.uint8), ("pinned", np.uint8),
                       ("pad_", np.uint8, 6)])
assert SLOT_DTYPE.itemsize == 24

vp = C.c_void_p
u64 = C.c_uint64
P = C.POINTER


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("moe_abi_version", C.c_int)
_sig("moe_host_threads", C.c_int)
_sig("moe_device_warmup", C.c_int, C.c_int)
_sig("moe_last_error", C.c_char_p)
_sig("moe_device_info", C.c_int, C.c_int, P(C.c_int), P(C.c_int), P(C.c_int), P(C.c_size_t))
_sig("moe_eamc_create", C.c_int, P(moe_shape), C.c_int, u64, C.c_int, C.c_int, P(vp))
_sig("moe_eamc_destroy", C.c_int, vp)
_sig("moe_eamc_create_sharded", C.c_int, P(moe_shape), C.c_int, u64, C.c_int, C.c_int,
     P(C.c_int), P(vp))
_sig("moe_eamc_shard_layout", C.c_int, vp, P(C.c_int), P(C.c_int))
_sig("moe_eamc_save_binary", C.c_int, vp, C.c_char_p)
_sig("moe_eamc_set_decision_server", C.c_int, vp, C.c_int)


class moe_expert_cache_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "transfers_started", "transfers_completed", "transfers_cancelled", "preemptions",
        "evictions", "hits", "misses", "bytes_moved", "queued", "in_flight")]


_sig("moe_expert_cache_create", C.c_int, P(moe_shape), u64, C.c_uint32, u64, vp, C.c_int, P(vp))
_sig("moe_expert_cache_destroy", C.c_int, vp)
_sig("moe_expert_cache_set_request_eam", C.c_int, vp, vp)
_sig("moe_expert_cache_submit", C.c_int, vp, vp, u64)
_sig("moe_expert_cache_progress", C.c_int, vp, C.c_int)
_sig("moe_expert_cache_acquire", C.c_int, vp, C.c_uint32, C.c_uint32, P(vp), P(C.c_int))
_sig("moe_expert_cache_release", C.c_int, vp, C.c_uint32, C.c_uint32)
_sig("moe_expert_cache_slot", C.c_int, vp, C.c_uint32, P(C.c_int64), P(C.c_int), P(C.c_int),
     P(C.c_double))
_sig("moe_expert_cache_stats_get", C.c_int, vp, P(moe_expert_cache_stats))
_sig("moe_expert_cache_read_slot", C.c_int, vp, C.c_uint32, vp)
_sig("moe_eamc_build_clustered", C.c_int, vp, vp, u64, C.c_uint32, vp, vp, P(C.c_uint32))
_sig("moe_eamc_load_sharded", C.c_int, C.c_char_p, P(moe_shape), C.c_int, P(C.c_int), P(vp))
_sig("moe_eamc_info", C.c_int, vp, P(moe_shape), P(C.c_int), P(u64), P(u64), P(u64),
     P(C.c_int))
_sig("moe_eamc_clone", C.c_int, vp, P(vp))
_sig("moe_eamc_entry", C.c_int, vp, u64, vp, P(u64))
_sig("moe_eamc_insert", C.c_int, vp, vp, C.c_int, C.c_int, P(C.c_int64), vp)
_sig("moe_eamc_build", C.c_int, vp, vp, u64, vp)
_sig("moe_eamc_append", C.c_int, vp, vp, vp, u64)
_sig("moe_eamc_append_packed", C.c_int, vp, vp, C.c_int, vp, u64)
_sig("moe_eamc_match", C.c_int, vp, vp, u64, vp, vp)
_sig("moe_eamc_match_device", C.c_int, vp, vp, C.c_int, u64, vp, vp)
_sig("moe_eamc_match_packed", C.c_int, vp, vp, C.c_int, u64, vp, vp)
_sig("moe_eamc_match_within", C.c_int, vp, vp, C.c_double, vp, u64, P(u64))
_sig("moe_match_merge", C.c_int, vp, u64, u64, vp)
_sig("moe_match_merge_device", C.c_int, vp, u64, u64, vp, vp)
_sig("moe_eamc_set_index_base", C.c_int, vp, u64)
_sig("moe_eamc_set_profiling", C.c_int, vp, C.c_int)
_sig("moe_eamc_kernel_times", C.c_int, vp, vp, vp)
_sig("moe_eam_distance", C.c_int, P(moe_shape), vp, vp, P(C.c_double))
_sig("moe_prefetch_priorities", C.c_int, vp, vp, C.c_uint32, C.c_int, vp, u64, P(u64))
_sig("moe_decide", C.c_int, vp, vp, C.c_uint32, vp, vp, u64, vp, u64, P(u64), P(C.c_int64))
_sig("moe_eamc_window_min_device", C.c_int, vp, vp, vp, vp)
_sig("moe_eamc_window_aggregate_device", C.c_int, vp, C.c_uint32, C.c_double, vp, vp, vp)
_sig("moe_eamc_prefetch_order_device", C.c_int, vp, vp, C.c_uint32, C.c_int, vp, vp, vp)
_sig("moe_cache_priority", C.c_int, P(moe_shape), vp, C.c_uint32, C.c_uint32, P(C.c_double))
_sig("moe_select_eviction_victim", C.c_int, P(moe_shape), vp, vp, u64, P(C.c_int64))
_sig("moe_eam_trace", C.c_int, P(moe_shape), vp, C.c_int, u64, vp, u64, vp)
_sig("moe_eam_trace_device", C.c_int, P(moe_shape), vp, C.c_int, u64, vp, u64, vp, vp, vp)
_sig("moe_traces_request_eams", C.c_int, C.c_char_p, P(moe_shape), C.c_int, vp, u64, P(u64))
_sig("moe_eamc_build_from_traces", C.c_int, vp, C.c_char_p, P(u64))
_sig("moe_eamc_capacity_bound", C.c_int, P(moe_shape), C.c_double, P(u64))
_sig("moe_eamc_save", C.c_int, vp, C.c_char_p)
_sig("moe_eamc_load", C.c_int, C.c_char_p, P(moe_shape), C.c_int, P(vp))
_sig("moe_gen_bench_family", C.c_int, u64, C.c_uint32, C.c_uint32, u64, u64, C.c_int, vp)

# every symbol include/moe_eamc.h declares
EXPORTS = [
    "moe_abi_version", "moe_host_threads", "moe_last_error", "moe_device_info", "moe_device_warmup", "moe_eamc_create",
    "moe_eamc_create_sharded", "moe_eamc_shard_layout", "moe_eamc_load_sharded",
    "moe_eamc_save_binary", "moe_eamc_build_clustered", "moe_eamc_set_decision_server",
    "moe_expert_cache_create", "moe_expert_cache_destroy", "moe_expert_cache_set_request_eam",
    "moe_expert_cache_submit", "moe_expert_cache_progress", "moe_expert_cache_acquire",
    "moe_expert_cache_release", "moe_expert_cache_slot", "moe_expert_cache_stats_get",
    "moe_expert_cache_read_slot",
    "moe_eamc_destroy", "moe_eamc_info", "moe_eamc_clone", "moe_eamc_entry", "moe_eamc_insert", "moe_eamc_build",
    "moe_eamc_append", "moe_eamc_append_packed", "moe_eamc_match", "moe_eamc_match_device",
    "moe_eamc_match_packed",
    "moe_eamc_match_within", "moe_match_merge", "moe_match_merge_device",
    "moe_eamc_set_index_base", "moe_eamc_set_profiling", "moe_eamc_kernel_times",
    "moe_eam_distance",
    "moe_prefetch_priorities", "moe_decide", "moe_cache_priority",
    "moe_eamc_window_min_device", "moe_eamc_window_aggregate_device",
    "moe_eamc_prefetch_order_device",
    "moe_select_eviction_victim", "moe_eam_trace", "moe_eam_trace_device",
    "moe_eamc_capacity_bound", "moe_traces_request_eams", "moe_eamc_build_from_traces",
    "moe_eamc_save", "moe_eamc_load", "moe_gen_bench_family",
]


class EamcSnapshotError(RuntimeError):
    """eam.hpp:63-65"""


class CudaError(RuntimeError):
    """MOE_ERR_CUDA / MOE_ERR_OOM / MOE_ERR_NCCL: no usable sm_100 device or a kernel failure."""


class TraceIngestError(RuntimeError):
    """MOE_ERR_TRACE: workload.hpp:55-59 -- a bad trace line ("line N: ...")."""


class CountOverflowError(OverflowError):
    """A count outside the range the device path represents exactly."""


def check(status: int) -> None:
    if status == MOE_OK:
        return
    msg = (lib.moe_last_error() or b"").decode(errors="replace")
    if status == MOE_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)            # std::invalid_argument
    if status == MOE_ERR_OUT_OF_RANGE:
        raise IndexError(msg)            # std::out_of_range
    if status == MOE_ERR_SNAPSHOT:
        raise EamcSnapshotError(msg)
    if status == MOE_ERR_LOGIC:
        raise RuntimeError(msg)          # std::logic_error
    if status == MOE_ERR_TRACE:
        raise TraceIngestError(msg)
    if status == MOE_ERR_OVERFLOW:
        raise CountOverflowError(msg)
    raise CudaError(f"status {status}: {msg}")


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def gen_bench_family(seed: int, L: int, E: int, n: int, skip: int = 0,
                     dtype=np.uint64) -> np.ndarray:
    """The reference bench stream (bench.cpp:44-54): EAMs skip..skip+n-1."""
    dt = np.dtype(dtype)
    out = np.zeros((n, L, E), dt)
    check(lib.moe_gen_bench_family(seed, L, E, skip, n, dt.itemsize, ptr(out)))
    return out
