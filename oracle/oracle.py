"""CPU oracle for the Seer hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module.  The product package
(paper_2403_17017_b200) never imports it and has no CPU fallback.

Every function cites the reference file:line (or SPEC.md line) it restates:

* length_stats / wave_ceil_max_sum -- /root/reference/pkg/src/kernelpick/_kernels/_pure.py:11-38
  and _core.pyx:15-56 (bit-exact integer aggregates; pinned by tests/golden).
* features_epilogue / gather_features -- features.py:64-87 (pinned by tests/golden).
* spmv_csr -- y = A.x over SparseMatrixCSR (sparse.py:33-39), fp64 accumulation.
  PARITY UNPINNED: the reference ships no SpMV.
* tree_predict / infer / total_cost / fastest_kernel -- SPEC.md:296-301, 376-384,
  205-222.  PARITY UNPINNED: the reference ships no tree code.
* csr_from_coo -- sparse.py:87-103 (lexsort, np.add.reduceat, bincount + cumsum);
  pinned by tests/golden/reference_coo_golden.json (bit-exact values).

The C restatement (kp_oracle.c -> liboracle.so) carries the O(nnz) loops; the
numpy forms below are the small-case cross-checks.  ``ref_core()`` loads the
UNMODIFIED reference _core.pyx compiled by ``make -C oracle ref`` (oracle/_ref).
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    targets = ["all"]
    if os.path.exists("/root/reference/pkg/src/kernelpick/_kernels/_core.pyx"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        i64, p = ctypes.c_int64, ctypes.c_void_p
        L.orc_length_stats.argtypes = [p, i64, p]
        L.orc_wave_ceil_max_sum.argtypes = [p, i64, i64, i64, p]
        L.orc_features_epilogue.argtypes = [i64] * 6 + [p]
        L.orc_features_epilogue.restype = None
        for n in ("orc_spmv_csr_f32", "orc_spmv_csr_f64", "orc_spmv_csr32_f32", "orc_spmv_csr32_f64"):
            getattr(L, n).argtypes = [i64, p, p, p, p, p, p]
            getattr(L, n).restype = None
        for n in ("orc_spmv_native_f32", "orc_spmv_native_f64"):
            getattr(L, n).argtypes = [i64, p, p, p, p, p]
            getattr(L, n).restype = None
        L.orc_tree_predict.argtypes = [p] * 6
        L.orc_tree_predict.restype = ctypes.c_int
        L.orc_threads.restype = ctypes.c_int
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_set_threads.restype = None
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# --------------------------------------------------------------------- integer core
def length_stats_np(row_offsets) -> tuple[int, int, int, int]:
    """numpy restatement of _pure.py:11-21."""
    lengths = np.diff(np.asarray(row_offsets, dtype=np.int64))
    if lengths.size == 0:
        return 0, 0, 0, 0
    return (int(lengths.min()), int(lengths.max()), int(lengths.sum()),
            int(np.dot(lengths, lengths)))


def wave_ceil_max_sum_np(row_offsets, divisor: int, wave_rows: int) -> int:
    """numpy restatement of _pure.py:24-38."""
    lengths = np.diff(np.asarray(row_offsets, dtype=np.int64))
    n = lengths.size
    if n == 0:
        return 0
    units = -(-lengths // divisor)
    pad = (-n) % wave_rows
    if pad:
        units = np.concatenate([units, np.zeros(pad, dtype=units.dtype)])
    return int(units.reshape(-1, wave_rows).max(axis=1).sum())


def length_stats(row_offsets) -> tuple[int, int, int, int]:
    """C restatement of _core.pyx:15-33 (scalar loop, wrapping int64)."""
    off = np.ascontiguousarray(row_offsets, dtype=np.int64)
    out = np.zeros(4, dtype=np.int64)
    lib().orc_length_stats(_ptr(off), off.size, _ptr(out))
    return tuple(int(v) for v in out)


def wave_ceil_max_sum(row_offsets, divisor: int, wave_rows: int) -> int:
    """C restatement of _core.pyx:36-56."""
    off = np.ascontiguousarray(row_offsets, dtype=np.int64)
    out = np.zeros(1, dtype=np.int64)
    if lib().orc_wave_ceil_max_sum(_ptr(off), off.size, int(divisor), int(wave_rows), _ptr(out)):
        raise ValueError("divisor and wave_rows must be positive")
    return int(out[0])


def features_epilogue(lo: int, hi: int, s1: int, s2: int, n: int, c: int) -> tuple:
    """Python restatement of features.py:74-85 (the fp64 epilogue), returning
    (max, min, mean, var) in as_vector order (features.py:46-52)."""
    max_d = hi / c
    min_d = lo / c
    denom = float(n) * float(c)
    mean_d = s1 / denom
    if hi == lo:
        var_d = 0.0
    else:
        var_d = s2 / (denom * float(c)) - mean_d * mean_d
        if var_d < 0.0:
            var_d = 0.0
    return (max_d, min_d, mean_d, var_d)


def features_epilogue_c(lo, hi, s1, s2, n, c) -> tuple:
    out = np.zeros(4, dtype=np.float64)
    lib().orc_features_epilogue(lo, hi, s1, s2, n, c, _ptr(out))
    return tuple(float(v) for v in out)


def gather_features(row_offsets, n_rows: int, n_cols: int) -> tuple:
    """features.py:64-87 without the clock: returns as_vector() order."""
    if n_rows == 0:
        raise ValueError("cannot gather features of an empty matrix")
    if n_cols == 0:
        raise ValueError("cannot gather features of a zero-column matrix")
    lo, hi, s1, s2 = length_stats(row_offsets)
    return features_epilogue(lo, hi, s1, s2, n_rows, n_cols)


# --------------------------------------------------------------------------- SpMV
def spmv_csr(row_offsets, col_indices, values, x) -> tuple[np.ndarray, np.ndarray]:
    """(y, absy): fp64-accumulated y = A.x and sum_j |a_ij x_j| per row.

    Inputs are the DEVICE-precision arrays (fp32 values/x for an fp32 run) so the
    only difference left against the GPU is accumulation order."""
    off = np.ascontiguousarray(row_offsets)
    col = np.ascontiguousarray(col_indices, dtype=np.int32)
    val = np.ascontiguousarray(values)
    xx = np.ascontiguousarray(x, dtype=val.dtype)
    n = off.size - 1
    y = np.zeros(n, dtype=np.float64)
    a = np.zeros(n, dtype=np.float64)
    suffix = {np.dtype(np.float32): "f32", np.dtype(np.float64): "f64"}[val.dtype]
    if off.dtype == np.int64:
        fn = getattr(lib(), "orc_spmv_csr_" + suffix)
    else:
        off = off.astype(np.int32, copy=False)
        fn = getattr(lib(), "orc_spmv_csr32_" + suffix)
    fn(n, _ptr(off), _ptr(col), _ptr(val), _ptr(xx), _ptr(y), _ptr(a))
    return y, a


def spmv_native(row_offsets32, col32, val, x) -> np.ndarray:
    """Native-precision multithreaded CPU SpMV (the timed CPU baseline port)."""
    n = row_offsets32.size - 1
    y = np.empty(n, dtype=val.dtype)
    fn = lib().orc_spmv_native_f32 if val.dtype == np.float32 else lib().orc_spmv_native_f64
    fn(n, _ptr(row_offsets32), _ptr(col32), _ptr(val), _ptr(x), _ptr(y))
    return y


def spmv_check(y_dev, y_ref, absy, tol: float) -> tuple[bool, float]:
    """Normwise-robust relative check |y - y_ref|_i <= tol * sum_j |a_ij x_j|."""
    y_dev = np.asarray(y_dev, dtype=np.float64)
    err = np.abs(y_dev - y_ref)
    bound = tol * absy + np.finfo(np.float64).tiny
    ratio = float(np.max(err / bound)) if err.size else 0.0
    return bool(np.all(err <= bound)), ratio


# --------------------------------------------------------------------------- COO -> CSR
def csr_from_coo(n_rows: int, n_cols: int, rows, cols, vals):
    """sparse.py:87-103 restated: (row_offsets int64, col_indices int64, values f64)."""
    r = np.asarray(rows, dtype=np.int64)
    c = np.asarray(cols, dtype=np.int64)
    v = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((c, r))  # stable: duplicates keep input order (sparse.py:92)
    r, c, v = r[order], c[order], v[order]
    if r.size:
        first = np.empty(r.size, dtype=bool)
        first[0] = True
        first[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        starts = np.flatnonzero(first)
        v = np.add.reduceat(v, starts)  # per run: v0 + numpy pairwise sum of the rest
        r, c = r[starts], c[starts]
    off = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n_rows), out=off[1:])
    return off, c, v


def threads() -> int:
    return int(lib().orc_threads())


def use_all_cores() -> int:
    """Run the CPU baseline on every core this process may use (launchers like torchrun set
    OMP_NUM_THREADS=1 per rank; the CPU arm runs on one rank only).  Returns the count."""
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    lib().orc_set_threads(int(n))
    return threads()


# --------------------------------------------------------------------------- trees
def tree_predict(tree: dict, x) -> int:
    """descend from the root, x[f] <= threshold goes left."""
    i = 0
    feat, thr, left, right, cls = (tree["feature"], tree["threshold"], tree["left"],
                                   tree["right"], tree["value"])
    while feat[i] >= 0:
        i = left[i] if float(x[feat[i]]) <= thr[i] else right[i]
    return int(cls[i])


def total_cost(runtime, preprocess, k: int) -> float:
    """preprocess + k * runtime; missing -> +inf."""
    if runtime is None or preprocess is None:
        return float("inf")
    return float(preprocess) + k * float(runtime)


def fastest_kernel(timings: list, k: int) -> int:
    """argmin of total_cost, ties to the lowest index."""
    costs = [total_cost(r, p, k) for (r, p) in timings]
    if all(c == float("inf") for c in costs):
        raise ValueError("all kernels missing")
    best = 0
    for i, c in enumerate(costs):
        if c < costs[best]:
            best = i
    return best


def infer(model: dict, rows: int, cols: int, nnz: int, k: int, gathered=None) -> tuple[int, int]:
    """SPEC.md:376-384 control flow: selector on (rows, cols, nnz, k); path 0 =
    USE_KNOWN -> known tree; path 1 = USE_GATHERED -> gathered tree on known +
    (max, min, mean, var).  Returns (kernel index, path)."""
    known = (float(rows), float(cols), float(nnz), float(k))
    path = tree_predict(model["selector"], known)
    if path == 0:
        return tree_predict(model["known"], known), 0
    if gathered is None:
        raise ValueError("selector demands gathered features")
    return tree_predict(model["gathered"], known + tuple(gathered)), 1


# --------------------------------------------------------------- compiled reference
def ref_core():
    """The UNMODIFIED reference _core (Cython) built into oracle/_ref, or None."""
    hits = glob.glob(os.path.join(HERE, "_ref", "_core*.so"))
    if not hits:
        return None
    spec = importlib.util.spec_from_file_location("_core", hits[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
