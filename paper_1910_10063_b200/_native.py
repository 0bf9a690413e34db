"""ctypes binding of libskx.so (include/skx.h).

There is no CPU fallback: if the library or a B200 is missing, loading fails
loudly (NativeUnavailable).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DomainViolation, Error, InvalidArgument, NativeUnavailable

PKG = os.path.dirname(os.path.abspath(__file__))
LIBSKX = os.path.join(PKG, "libskx.so")
# A/B runs of library variants point SKX_LIBSKX at the variant instead of
# overwriting the in-tree build (tools/ab.sh).
LIBSKX_PATH = os.environ.get("SKX_LIBSKX") or LIBSKX

OK, INVALID_ARGUMENT, DOMAIN_VIOLATION, CUDA_ERROR, NCCL_ERROR, ERROR = 0, 1, 2, 3, 4, 5
DT_U32, DT_I32, DT_U64, DT_I64, DT_F64 = 0, 1, 2, 3, 4
OP_SUM, OP_MIN, OP_MAX = 0, 1, 2


class ErrorInfo(C.Structure):
    _fields_ = [("status", C.c_int32), ("row", C.c_uint64), ("value", C.c_uint32),
                ("domain", C.c_uint64), ("message", C.c_char * 256)]


_vp, _u64, _u32, _i32, _int, _dbl = (C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32, C.c_int,
                                     C.c_double)

# name -> (restype, argtypes); mirrors include/skx.h
SIGNATURES = {
    "skx_version": (_int, []),
    "skx_device_count": (_int, [C.POINTER(_int)]),
    "skx_ctx_create": (_int, [_int, C.POINTER(_vp)]),
    "skx_ctx_destroy": (_int, [_vp]),
    "skx_sync": (_int, [_vp, _vp]),
    "skx_last_error": (_int, [_vp, C.POINTER(ErrorInfo)]),
    "skx_launch_count": (_u64, [_vp]),
    "skx_reserve": (_int, [_vp, _int, _u64, _vp]),
    "skx_scratch_bytes": (_int, [_vp, _vp, _vp]),
    "skx_gather_u16": (_int, [_vp, _vp, _u64, _vp, _u64, _vp, _vp]),
    "skx_gather_u32": (_int, [_vp, _vp, _u64, _vp, _u64, _vp, _vp]),
    "skx_gather_u64": (_int, [_vp, _vp, _u64, _vp, _u64, _vp, _vp]),
    "skx_gather_split_u32": (_int, [_vp, _vp, _u64, _vp, _u64, _u32, _vp, _vp]),
    "skx_gather_split_u64": (_int, [_vp, _vp, _u64, _vp, _u64, _u32, _vp, _vp]),
    "skx_count_frequencies": (_int, [_vp, _vp, _u64, _u32, _vp, _vp]),
    "skx_histogram_u32": (_int, [_vp, _vp, _u64, _u32, _vp, _int, _vp]),
    "skx_build_index": (_int, [_vp, _vp, _u32, _u64, _vp, _vp, _vp]),
    "skx_build_index_u32": (_int, [_vp, _vp, _u32, _u64, _vp, _vp, _vp]),
    "skx_rebuild": (_int, [_vp, _vp, _u64, _u32, _vp, _vp, _vp]),
    "skx_recode_fact": (_int, [_vp, _vp, _u64, _vp, _u32, _vp, _vp]),
    "skx_permute_dimension_u16": (_int, [_vp, _vp, _u64, _vp, _u32, _vp, _vp]),
    "skx_permute_dimension_u32": (_int, [_vp, _vp, _u64, _vp, _u32, _vp, _vp]),
    "skx_permute_dimension_u64": (_int, [_vp, _vp, _u64, _vp, _u32, _vp, _vp]),
    "skx_aggregate": (_int, [_vp, _vp, _vp, _int, _u64, _u32, _u32, _vp, _vp, _vp]),
    "skx_select_offsets": (_int, [_vp, _vp, _u64, _vp, _u64, _u32, _vp, _vp, _vp]),
    "skx_permute_bitmap": (_int, [_vp, _vp, _u64, _vp, _u32, _vp, _vp]),
    "skx_build_bitmap_lt_i32": (_int, [_vp, _vp, _u64, _i32, _vp, _vp]),
    "skx_select_gather_sum": (_int, [_vp, _vp, _u64, _vp, _u32, _vp, _vp, _vp, _vp, _u32, _u32, _u64,
                                     _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "skx_heavy_hitter_count": (_int, [_vp, _vp, _u64, _u32, _u32, _vp, _vp]),
    "skx_zipf_cdf_host": (_int, [_u32, _dbl, _vp]),
    "skx_random_bijection_host": (_int, [_u32, _u64, _vp]),
    "skx_line_frequencies": (_int, [_vp, _vp, _u32, _vp, _u32, _vp, _vp]),
    "skx_estimate_hit_rate": (_int, [_vp, _vp, _u64, _u64, _vp, _vp]),
    "skx_trace_from_column": (_int, [_vp, _vp, _u64, _u32, _vp, _vp]),
    "skx_simulate_lru_host": (_int, [_vp, _u64, _u64, _vp]),
    "skx_generate_zipf": (_int, [_vp, _vp, _u32, _vp, _u64, _u64, _u64, _vp, _vp]),
    "skx_materialize_host": (_int, [_vp, _int, _vp, _u64, _vp, _u64, _vp]),
    "skx_aggregate_host": (_int, [_vp, _vp, _vp, _int, _u64, _u32, _u32, _vp, _vp]),
    "skx_set_gather_policy": (_int, [_vp, _int]),
    "skx_gather_last_plan": (_int, [_vp, _vp, _vp]),
    "skx_set_l2_fetch_granularity": (_int, [_vp, _int]),
    "skx_device_info": (_int, [_vp, _vp, _int]),
    "skx_reset_persisting_l2": (_int, [_vp]),
    "skx_set_histogram_mode": (_int, [_vp, _int]),
    "skx_set_aggregate_mode": (_int, [_vp, _int]),
    "skx_set_gather_tiers": (_int, [_vp, _u64, _u64, _dbl]),
    "skx_device_alloc": (_int, [_vp, _u64, C.POINTER(_vp)]),
    "skx_device_free": (_int, [_vp, _vp]),
    "skx_copy_to_device": (_int, [_vp, _vp, _vp, _u64]),
    "skx_copy_to_host": (_int, [_vp, _vp, _vp, _u64]),
    "skx_pinned_alloc": (_int, [_vp, _u64, C.POINTER(_vp)]),
    "skx_pinned_free": (_int, [_vp, _vp]),
    "skx_ctx_stream": (_vp, [_vp, _int]),
    "skx_copy_to_device_async": (_int, [_vp, _vp, _vp, _u64, _vp]),
    "skx_copy_to_host_async": (_int, [_vp, _vp, _vp, _u64, _vp]),
    "skx_find_domain_violation": (_int, [_vp, _vp, _u64, _u64, C.POINTER(_u64)]),
    "skx_fill_column": (_int, [_vp, _int, _int, _u64, _u64, _dbl, _dbl, _vp, _vp]),
    "skx_select_sum_partials": (_int, [_vp, _u32, _vp, _vp]),
    "skx_select_sums_from_partials": (_int, [_vp, _vp, _u32, _u32, _vp, _vp]),
    "skx_groupby_pack": (_int, [_vp, _vp, _vp, _u32, _u32, _vp, _vp, _vp]),
    "skx_groupby_unpack": (_int, [_vp, _vp, _u32, _u32, _vp, _vp, _vp]),
    "skx_groupby_packed_ok": (_int, [_vp]),
    "skx_comm_init_all": (_int, [_int, _vp, C.POINTER(_vp)]),
    "skx_comm_unique_id": (_int, [_vp]),
    "skx_comm_init_rank": (_int, [_int, _int, _int, _vp, C.POINTER(_vp)]),
    "skx_comm_destroy": (_int, [_vp]),
    "skx_comm_info": (_int, [_vp, C.POINTER(_int), C.POINTER(_int), C.POINTER(_int)]),
    "skx_comm_ctx": (_vp, [_vp, _int]),
    "skx_comm_stream": (_vp, [_vp, _int]),
    "skx_comm_error": (C.c_char_p, [_vp]),
    "skx_comm_sync": (_int, [_vp]),
    "skx_allreduce": (_int, [_vp, _vp, _u64, _int, _int, _vp]),
    "skx_reduce": (_int, [_vp, _vp, _u64, _int, _int, _int, _vp]),
    "skx_reduce_scatter": (_int, [_vp, _vp, _vp, _u64, _int, _int, _vp]),
    "skx_allgather": (_int, [_vp, _vp, _vp, _u64, _int, _vp]),
    "skx_broadcast": (_int, [_vp, _vp, _u64, _int, _int, _vp]),
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIBSKX_PATH) -> C.CDLL:
    """Load libskx.so once (building it first if only the sources exist)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            try:
                from .build import build_libskx
                build_libskx()
            except Exception as e:  # noqa: BLE001
                raise NativeUnavailable(f"libskx.so missing and build failed: {e}") from e
        try:
            lib = C.CDLL(path)
        except OSError as e:
            raise NativeUnavailable(f"cannot load {path}: {e}") from e
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def raise_for(status: int, info: ErrorInfo | None = None) -> None:
    if status == OK:
        return
    msg = info.message.decode(errors="replace") if info is not None else f"status {status}"
    if status == DOMAIN_VIOLATION:
        raise DomainViolation(info.row, info.value, info.domain)
    if status == INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == CUDA_ERROR:
        raise Error("CUDA error: " + msg)
    if status == NCCL_ERROR:
        raise Error("NCCL error: " + msg)
    raise Error(msg)
