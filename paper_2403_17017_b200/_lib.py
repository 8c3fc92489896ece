"""ctypes binding of libkpb200.so (the C-ABI in include/kernelpick_b200.h).

There is deliberately no CPU fallback: if the shared library is missing or no CUDA
device is present, every compute entry point raises ``BackendUnavailable``.
PyTorch is used only as the device-memory / stream allocator (plumbing).
"""

from __future__ import annotations

import ctypes
import os

from .errors import KernelPickError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkpb200.so")

# status codes (kernelpick_b200.h)
KP_OK, KP_EINVAL, KP_ECUDA, KP_ENOMEM, KP_EUNSUPPORTED, KP_ERANGE = 0, -1, -2, -3, -4, -5
KP_I32, KP_I64 = 0, 1
KP_F32, KP_F64 = 0, 1
KP_USE_KNOWN, KP_USE_GATHERED = 0, 1
KP_SELECT_STATIC, KP_SELECT_EMITTED, KP_SELECT_PARAM, KP_SELECT_TABLE = 0, 1, 2, 3

EXPORTS = (
    "kp_reduce_workspace_bytes", "kp_length_stats", "kp_wave_ceil_max_sum", "kp_gather_features",
    "kp_tree_predict", "kp_seer_select", "kp_prepare_bytes", "kp_prepare",
    "kp_spmv_workspace_bytes", "kp_spmv", "kp_seer_plan_bytes", "kp_seer_plan_create", "kp_seer_plan_launch",
    "kp_seer_plan_destroy", "kp_shard_partition", "kp_version", "kp_launch_count", "kp_debug_set_wave_warps",
    "kp_seer_select_partials", "kp_coo_workspace_bytes", "kp_csr_from_coo", "kp_spmv_bcast", "kp_spmv_bcast_acc",
    "kp_mm_header", "kp_mm_parse", "kp_watchdog_start", "kp_watchdog_heartbeat", "kp_watchdog_status",
    "kp_watchdog_stop", "kp_seer_plan_select_kind", "kp_seer_emitted_predict", "kp_seer_emitted_sha256",
    "kp_pack_bits", "kp_pack_cols_bytes", "kp_pack_cols", "kp_unpack_cols",
)


class BackendUnavailable(KernelPickError):
    """The sm_100a backend (libkpb200.so + a CUDA device) is not available."""


class KernelError(KernelPickError):
    """A C-ABI call returned a non-zero status."""


class kp_csr(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("off_type", ctypes.c_int32), ("val_type", ctypes.c_int32),
                ("row_offsets", ctypes.c_void_p), ("col_indices", ctypes.c_void_p),
                ("values", ctypes.c_void_p)]


class kp_outcome(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_int64), ("hi", ctypes.c_int64), ("s1", ctypes.c_int64),
                ("s2", ctypes.c_int64), ("max_d", ctypes.c_double), ("min_d", ctypes.c_double),
                ("mean_d", ctypes.c_double), ("var_d", ctypes.c_double), ("kernel", ctypes.c_int32),
                ("path", ctypes.c_int32), ("status", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class kp_prepared(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("group", ctypes.c_int32), ("n_units", ctypes.c_int64),
                ("ell_cap", ctypes.c_int64), ("buf", ctypes.c_void_p), ("bytes", ctypes.c_size_t)]


KP_MAX_PEERS = 8
KP_EPARSE = -6
KP_WD_OK, KP_WD_NCCL_ERROR, KP_WD_TIMEOUT = 0, 1, 2


class kp_mm_info(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64), ("n_entries", ctypes.c_int64),
                ("n_triples", ctypes.c_int64), ("field", ctypes.c_int32), ("symmetry", ctypes.c_int32),
                ("err_line", ctypes.c_int64), ("err", ctypes.c_char * 192)]


class kp_peers(ctypes.Structure):
    _fields_ = [("y", ctypes.c_void_p * KP_MAX_PEERS), ("n", ctypes.c_int32), ("self", ctypes.c_int32)]


OUTCOME_BYTES = ctypes.sizeof(kp_outcome)  # 96
_lib = None


def load(require: bool = True):
    """Load libkpb200.so (no CUDA context needed).  Raises BackendUnavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not require:
            return None
        raise BackendUnavailable(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or make -C paper_2403_17017_b200/csrc); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    i32, i64, p, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
    P = ctypes.POINTER
    sig = {
        "kp_reduce_workspace_bytes": (sz, []),
        "kp_length_stats": (ctypes.c_int, [p, i32, i64, p, p, p]),
        "kp_wave_ceil_max_sum": (ctypes.c_int, [p, i32, i64, i64, i64, p, p, p]),
        "kp_gather_features": (ctypes.c_int, [p, i32, i64, i64, p, p, p]),
        "kp_tree_predict": (ctypes.c_int, [p, p, i64, i32, p, p]),
        "kp_seer_select": (ctypes.c_int, [p, i32, i64, i64, i64, i64, p, p, p, p, p, p]),
        "kp_prepare_bytes": (ctypes.c_int, [i32, P(kp_csr), i64, P(sz)]),
        "kp_prepare": (ctypes.c_int, [i32, P(kp_csr), i64, p, sz, P(kp_prepared), p]),
        "kp_spmv_workspace_bytes": (ctypes.c_int, [i32, P(kp_csr), P(sz)]),
        "kp_spmv": (ctypes.c_int, [i32, P(kp_csr), P(kp_prepared), p, p, p, sz, p]),
        "kp_seer_plan_bytes": (ctypes.c_int, [P(kp_csr), i64, P(sz)]),
        "kp_seer_plan_create": (ctypes.c_int, [P(kp_csr), i64, i64, p, p, p, p, p, p, sz, p, p, P(p), p]),
        "kp_seer_plan_launch": (ctypes.c_int, [p, p]),
        "kp_seer_plan_destroy": (ctypes.c_int, [p]),
        "kp_shard_partition": (ctypes.c_int, [p, i32, i64, i32, p, p]),
        "kp_version": (ctypes.c_char_p, []),
        "kp_launch_count": (ctypes.c_uint64, []),
        "kp_debug_set_wave_warps": (ctypes.c_int64, [i64]),
        "kp_seer_select_partials": (ctypes.c_int, [p, i32, i64, i64, i64, i64, p, p, p, p, p]),
        "kp_coo_workspace_bytes": (ctypes.c_int, [i64, i64, i64, P(sz)]),
        "kp_csr_from_coo": (ctypes.c_int, [i64, i64, p, p, p, i64, p, p, p, p, p, sz, p]),
        "kp_spmv_bcast": (ctypes.c_int, [i32, P(kp_csr), P(kp_prepared), p, P(kp_peers), p, sz, p]),
        "kp_spmv_bcast_acc": (ctypes.c_int, [i32, P(kp_csr), P(kp_prepared), p, p, p, P(kp_peers), p, sz, p]),
        "kp_mm_header": (ctypes.c_int, [ctypes.c_char_p, sz, P(kp_mm_info)]),
        "kp_mm_parse": (ctypes.c_int, [ctypes.c_char_p, sz, p, p, p, i64, i32, P(kp_mm_info)]),
        "kp_watchdog_start": (ctypes.c_int, [p, i64, i64, P(p)]),
        "kp_watchdog_heartbeat": (ctypes.c_int, [p]),
        "kp_watchdog_status": (ctypes.c_int, [p, P(i32), ctypes.c_char_p, sz]),
        "kp_watchdog_stop": (ctypes.c_int, [p]),
        "kp_seer_plan_select_kind": (ctypes.c_int, [p]),
        "kp_seer_emitted_predict": (ctypes.c_int, [i32, p, i64, p, p]),
        "kp_seer_emitted_sha256": (ctypes.c_char_p, []),
        "kp_pack_bits": (i32, [i64]),
        "kp_pack_cols_bytes": (sz, [i64, i64]),
        "kp_pack_cols": (ctypes.c_int, [p, i64, i64, p, i32]),
        "kp_unpack_cols": (ctypes.c_int, [p, i64, i64, p, p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc == KP_OK:
        return
    if rc == KP_EINVAL:
        raise ValueError(f"{what}: invalid argument (KP_EINVAL)")
    if rc == KP_ERANGE:
        raise OverflowError(f"{what}: value outside the exactly representable range (KP_ERANGE)")
    if rc == KP_ENOMEM:
        raise MemoryError(f"{what}: workspace too small (KP_ENOMEM)")
    raise KernelError(f"{what}: status {rc}")


def require_cuda():
    """Import torch and check a CUDA device is present; returns the torch module."""
    import torch
    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device: the kernelpick-b200 backend runs only on sm_100a GPUs "
                                 "(there is no CPU fallback)")
    load()
    return torch


def stream_handle(stream=None, device=None) -> int:
    """cudaStream_t of ``stream``, else of ``device``'s (default: the current device's)
    current torch stream."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)
