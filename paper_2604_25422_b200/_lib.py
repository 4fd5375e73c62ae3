"""ctypes binding of the C ABI in include/ks_dwconv1d.h.

Loads the in-tree ``libks_dwconv1d.so`` (built by ``make``, see
``__graft_entry__.build``).  There is no fallback: if the library is missing
this raises, and every compute entry point returns ``KS_ERR_NO_DEVICE`` when
no CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# KS_LIB: an alternate build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("KS_LIB") or os.path.join(HERE, "libks_dwconv1d.so")

# enums (include/ks_dwconv1d.h)
KS_OK = 0
STATUS_NAMES = {
    0: "KS_OK", 1: "KS_ERR_DIM_B", 2: "KS_ERR_DIM_H", 3: "KS_ERR_DIM_L", 4: "KS_ERR_DIM_K",
    5: "KS_ERR_BAD_CHUNK", 6: "KS_ERR_BAD_MODE", 7: "KS_ERR_BAD_SCHEME", 8: "KS_ERR_NULL",
    9: "KS_ERR_WORKSPACE", 10: "KS_ERR_NO_DEVICE", 11: "KS_ERR_CUDA", 12: "KS_ERR_NCCL",
    13: "KS_ERR_SHARD", 14: "KS_ERR_BAD_OPTION", 15: "KS_ERR_TIMEOUT",
}
KS_OPTION_DEFAULT = -(1 << 63)
SEPARATE, FUSED = 0, 1
SEQUENTIAL, PAIRWISE, CHUNKED, HIERARCHICAL = 0, 1, 2, 3

# Every extern "C" symbol declared in include/ks_dwconv1d.h.
EXPORTED = [
    "ks_status_string", "ks_last_error_string", "ks_abi_version",
    "ks_dwconv1d_fwd_f32", "ks_dwconv1d_fwd_f64", "ks_dwconv1d_dx_f32", "ks_dwconv1d_dx_f64",
    "ks_dwconv1d_dw_workspace_bytes", "ks_dwconv1d_dw_f32", "ks_dwconv1d_dw_f64",
    "ks_dwconv1d_bwd_f32", "ks_fill_pm1_f32", "ks_launch_count", "ks_dwconv1d_plan", "ks_set_option", "ks_get_option",
    "ks_probe_fp32_tflops",
    "ks_dwconv1d_fwd_f32_host", "ks_dwconv1d_dx_f32_host", "ks_dwconv1d_dw_f32_host",
    "ks_dwconv1d_fwd_f64_host", "ks_dwconv1d_dx_f64_host", "ks_dwconv1d_dw_f64_host",
    "ks_dwconv1d_step_f32_host",
    "ks_dwconv1d_variant_workspace_bytes", "ks_dwconv1d_variant_f32",
    "ks_shard_rows", "ks_comm_unique_id", "ks_comm_init", "ks_comm_init_host", "ks_comm_destroy",
    "ks_comm_allgather_host",
    "ks_dwconv1d_dw_allreduce_f32", "ks_dwconv1d_dw_allgather_sum_f32", "ks_rank_tree_sum_f32",
    "ks_dwconv1d_dw_chunked_sharded_f32",
    "ks_peer_create", "ks_peer_destroy", "ks_dwconv1d_dw_f32_peer", "ks_peer_timed_out",
]

_i64, _u64, _p, _int, _sz = C.c_int64, C.c_uint64, C.c_void_p, C.c_int, C.c_size_t
# host all-gather callback of ks_comm_init_host: (send, recv, bytes, ctx) -> 0 on success
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
_SIGS = {
    "ks_status_string": ([_int], C.c_char_p),
    "ks_last_error_string": ([], C.c_char_p),
    "ks_abi_version": ([], _int),
    "ks_dwconv1d_fwd_f32": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int, _p], _int),
    "ks_dwconv1d_fwd_f64": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int, _p], _int),
    "ks_dwconv1d_dx_f32": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int, _p], _int),
    "ks_dwconv1d_dx_f64": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int, _p], _int),
    "ks_dwconv1d_dw_workspace_bytes": ([_i64, _i64, _i64, _i64, _int, _i64, _int, C.POINTER(_sz)], _int),
    "ks_dwconv1d_dw_f32": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int, _i64, _int, _p, _sz, _p], _int),
    "ks_dwconv1d_bwd_f32": ([_p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _int, _p, _sz, _p], _int),
    "ks_dwconv1d_dw_f64": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int, _i64, _int, _p, _sz, _p], _int),
    "ks_fill_pm1_f32": ([_u64, _u64, _p, _i64, _p], _int),
    "ks_probe_fp32_tflops": ([C.POINTER(C.c_double)], _int),
    "ks_launch_count": ([C.POINTER(_u64)], _int),
    "ks_dwconv1d_plan": ([_int, _i64, _i64, _i64, _i64, _int, _i64, _int, _p, _int, C.POINTER(_int)], _int),
    "ks_set_option": ([C.c_char_p, _i64], _int),
    "ks_get_option": ([C.c_char_p, C.POINTER(_i64)], _int),
    "ks_dwconv1d_fwd_f32_host": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int], _int),
    "ks_dwconv1d_dx_f32_host": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int], _int),
    "ks_dwconv1d_dw_f32_host": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int, _i64, _int], _int),
    "ks_dwconv1d_fwd_f64_host": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int], _int),
    "ks_dwconv1d_dx_f64_host": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int], _int),
    "ks_dwconv1d_dw_f64_host": ([_p, _p, _p, _i64, _i64, _i64, _i64, _int, _i64, _int], _int),
    "ks_dwconv1d_step_f32_host": ([_p] * 6 + [_i64, _i64, _i64, _i64, _int, _i64, _int], _int),
    "ks_dwconv1d_variant_workspace_bytes": ([_int, _int, _i64, _i64, C.POINTER(_sz)], _int),
    "ks_dwconv1d_variant_f32": ([_int, _int, _p, _p, _p, _i64, _i64, _i64, _i64, _int, _p, _sz, _p], _int),
    "ks_shard_rows": ([_i64, _int, _int, C.POINTER(_i64), C.POINTER(_i64)], _int),
    "ks_comm_unique_id": ([_p], _int),
    "ks_comm_init": ([C.POINTER(_p), _p, _int, _int], _int),
    "ks_comm_init_host": ([C.POINTER(_p), _int, _int, ALLGATHER_FN, _p], _int),
    "ks_rank_tree_sum_f32": ([_p, _p, _i64, _int, _p], _int),
    "ks_comm_allgather_host": ([_p, _p, _p, _sz], _int),
    "ks_comm_destroy": ([_p], _int),
    "ks_dwconv1d_dw_allreduce_f32": ([_p, _i64, _i64, _p, _p], _int),
    "ks_dwconv1d_dw_allgather_sum_f32": ([_p, _p, _i64, _i64, _p, _p], _int),
    "ks_dwconv1d_dw_chunked_sharded_f32": ([_p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _int, _p, _p],
                                           _int),
    "ks_peer_create": ([_p, _sz, C.POINTER(_p)], _int),
    "ks_peer_destroy": ([_p], _int),
    "ks_dwconv1d_dw_f32_peer": ([_p, _p, _p, _i64, _i64, _i64, _i64, _i64, _int, _p, _p], _int),
    "ks_peer_timed_out": ([_p, C.POINTER(_int)], _int),
}



class LaunchRec(C.Structure):
    """ks_launch_rec (include/ks_dwconv1d.h)."""
    _fields_ = [("kernel", C.c_char * 256), ("grid", C.c_uint32 * 3), ("block", C.c_uint32 * 3),
                ("smem_bytes", C.c_uint64), ("regs", C.c_int32), ("static_smem", C.c_int32), ("ctas_per_sm", C.c_int32)]


_lib = None


class KsError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        name = STATUS_NAMES.get(status, str(status))
        detail = ""
        if _lib is not None:
            detail = (_lib.ks_last_error_string() or b"").decode()
            text = (_lib.ks_status_string(status) or b"").decode()
        else:
            text = ""
        super().__init__(f"{what}: {name} ({text}){' ' + detail if detail else ''}")


def lib() -> C.CDLL:
    """The loaded library (raises if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                "there is no CPU fallback")
        l = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(l, name)
            f.argtypes = args
            f.restype = res
        _lib = l
    return _lib


def check(status: int, what: str) -> None:
    if status != KS_OK:
        raise KsError(status, what)
