"""Matrix Market ingest (sparse.py:106-196) through the native parallel parser
(kp_mm_parse in libkpb200.so) -- the wire format in front of csr_from_coo.

* ``parse_matrix_market(data)`` -- drop-in for the reference: same grammar, checks, error
  messages with 1-based line numbers (``ParseError``), returns the host SparseMatrixCSR.
* ``read_matrix_market_device(data)`` -- the same parse, canonicalised on the GPU
  (``device.csr_from_coo``) into a DeviceCSR.
* ``write_matrix_market(m)`` -- the reference writer with its numpy-2 defect fixed
  (values written as ``repr(float(v))`` so the round trip parses).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ParseError


def _bytes(data) -> bytes:
    if isinstance(data, str):
        return data.encode("utf-8")
    return bytes(data)


def parse_arrays(data, n_threads: int = 0):
    """(n_rows, n_cols, rows, cols, vals): 0-based int64 coordinates and f64 values in the
    reference's append order (entry, then its mirror for symmetric storage)."""
    buf = _bytes(data)
    L = _lib.load()
    info = _lib.kp_mm_info()
    rc = L.kp_mm_header(buf, len(buf), ctypes.byref(info))
    if rc == _lib.KP_EPARSE:
        raise ParseError(info.err.decode("utf-8", "replace"))
    _lib.check(rc, "kp_mm_header")
    cap = int(info.n_entries) * (2 if info.symmetry else 1)
    while True:
        rows = np.empty(max(cap, 1), dtype=np.int64)
        cols = np.empty(max(cap, 1), dtype=np.int64)
        vals = np.empty(max(cap, 1), dtype=np.float64)
        rc = L.kp_mm_parse(buf, len(buf), rows.ctypes.data, cols.ctypes.data, vals.ctypes.data, cap, int(n_threads),
                           ctypes.byref(info))
        if rc == _lib.KP_EPARSE:
            raise ParseError(info.err.decode("utf-8", "replace"))
        if rc == _lib.KP_ENOMEM and info.n_triples > cap:
            cap = int(info.n_triples)
            continue
        _lib.check(rc, "kp_mm_parse")
        n = int(info.n_triples)
        return int(info.n_rows), int(info.n_cols), rows[:n], cols[:n], vals[:n]


def parse_matrix_market(data, n_threads: int = 0):
    """sparse.parse_matrix_market (sparse.py:106-196) -> host SparseMatrixCSR."""
    from .sparse import csr_from_coo
    R, C, r, c, v = parse_arrays(data, n_threads)
    return csr_from_coo(R, C, r, c, v)


def read_matrix_market_device(data, dtype=None, n_threads: int = 0):
    """Parse natively, canonicalise on the GPU (kp_csr_from_coo) -> DeviceCSR."""
    from .device import csr_from_coo
    R, C, r, c, v = parse_arrays(data, n_threads)
    return csr_from_coo(R, C, r, c, v, dtype=dtype)


def write_matrix_market(m) -> str:
    """Coordinate/real/general text (sparse.py:199-207) with values as repr(float(v))."""
    out = ["%%MatrixMarket matrix coordinate real general", f"{m.n_rows} {m.n_cols} {m.nnz}"]
    lengths = np.diff(np.asarray(m.row_offsets))
    row_of = np.repeat(np.arange(m.n_rows), lengths)
    for i, j, v in zip(row_of.tolist(), np.asarray(m.col_indices).tolist(), np.asarray(m.values).tolist()):
        out.append(f"{i + 1} {j + 1} {float(v)!r}")
    return "\n".join(out) + "\n"
