"""Canonical host CSR type and the zero-cost known features.

Drop-in for the reference's data model (/root/reference/pkg/src/kernelpick/sparse.py):

* ``SparseMatrixCSR`` (sparse.py:33-71): immutable, int64 offsets / int64 columns /
  float64 values, copied and frozen read-only on construction, validated canonical
  (offsets start at 0 and never decrease, columns in range and strictly increasing
  inside each row).
* ``KnownFeatures`` / ``known_features`` (sparse.py:24-30, 82-84): (rows, cols, nnz)
  read in O(1) without touching entries (SPEC.md:388 known-path purity).
* ``csr_from_coo`` (sparse.py:87-103): sort by (row, col), sum duplicates, build offsets.

The device-resident form used by the CUDA kernels is ``device.DeviceCSR``; this host
type is what the reference's callers already hold, so every public entry point
accepts it and uploads it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class KnownFeatures:
    """Structure metrics available at zero runtime cost."""

    rows: int
    cols: int
    nnz: int


def _frozen_copy(a, dtype) -> np.ndarray:
    out = np.array(a, dtype=dtype, copy=True)
    if out.ndim != 1:
        raise ValueError("expected a 1-D array")
    out.flags.writeable = False
    return out


@dataclass(frozen=True)
class SparseMatrixCSR:
    n_rows: int
    n_cols: int
    row_offsets: np.ndarray  # int64 [n_rows + 1]
    col_indices: np.ndarray  # int64 [nnz]
    values: np.ndarray       # float64 [nnz]

    def __post_init__(self):
        object.__setattr__(self, "row_offsets", _frozen_copy(self.row_offsets, np.int64))
        object.__setattr__(self, "col_indices", _frozen_copy(self.col_indices, np.int64))
        object.__setattr__(self, "values", _frozen_copy(self.values, np.float64))
        self._check_canonical()

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    def row_length(self, row: int) -> int:
        off = self.row_offsets
        return int(off[row + 1] - off[row])

    def _check_canonical(self) -> None:
        n, c = self.n_rows, self.n_cols
        off, col, val = self.row_offsets, self.col_indices, self.values
        if n < 0 or c < 0:
            raise ValueError("negative matrix dimensions")
        if off.size != n + 1:
            raise ValueError("row_offsets length must be n_rows + 1")
        lengths = off[1:] - off[:-1]
        if off[0] != 0 or (lengths < 0).any():
            raise ValueError("row_offsets must start at 0 and be non-decreasing")
        z = int(off[-1])
        if col.size != z or val.size != z:
            raise ValueError("col_indices/values length must equal row_offsets[-1]")
        if z == 0:
            return
        if col.min() < 0 or col.max() >= c:
            raise ValueError("column index out of range")
        # a step col[j] -> col[j+1] may only be non-increasing where j+1 starts a row
        row_start = np.zeros(z, dtype=bool)
        starts = off[:-1][lengths > 0]
        row_start[starts] = True
        bad = (col[1:] <= col[:-1]) & ~row_start[1:]
        if bad.any():
            raise ValueError("col_indices must be strictly increasing within a row")


def known_features(m) -> KnownFeatures:
    """O(1): reads n_rows, n_cols and the last offset only (never entries)."""
    return KnownFeatures(rows=int(m.n_rows), cols=int(m.n_cols), nnz=int(m.nnz))


def csr_from_coo(n_rows: int, n_cols: int, rows, cols, vals) -> SparseMatrixCSR:
    """Canonicalise coordinate triples: order by (row, col), sum duplicates, offsets."""
    r = np.asarray(rows, dtype=np.int64).ravel()
    c = np.asarray(cols, dtype=np.int64).ravel()
    v = np.asarray(vals, dtype=np.float64).ravel()
    if not (r.size == c.size == v.size):
        raise ValueError("rows, cols and vals must have the same length")
    if r.size:
        key_order = np.lexsort((c, r))
        r, c, v = r[key_order], c[key_order], v[key_order]
        new = np.ones(r.size, dtype=bool)
        new[1:] = (np.diff(r) != 0) | (np.diff(c) != 0)
        seg = np.flatnonzero(new)
        v = np.add.reduceat(v, seg)
        r, c = r[seg], c[seg]
    counts = np.bincount(r, minlength=n_rows) if r.size else np.zeros(n_rows, dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return SparseMatrixCSR(n_rows, n_cols, off, c, v)
