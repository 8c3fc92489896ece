"""Golden vectors for csr_from_coo from the UNMODIFIED reference (run in the build container).

    python tests/golden/make_golden_coo.py    # writes tests/golden/reference_coo_golden.json

Inputs are regenerated from `coo_case(spec)` (numpy PCG64, deterministic on every
platform); the JSON stores the reference's output (offsets, cols, values as float.hex) of
``kernelpick.sparse.csr_from_coo`` (sparse.py:87-103), imported read-only from
/root/reference/pkg/src.  Cases stress the parts parity depends on: stable order of
duplicates, numpy's pairwise summation inside np.add.reduceat (runs of 1..600 duplicates,
i.e. the < 8, <= 128 and recursive branches), cancellation, signed zeros, empty rows at
both ends.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_coo_golden.json")

SPECS = [
    {"name": "empty", "n_rows": 5, "n_cols": 3, "n": 0, "seed": 1, "kind": "uniform"},
    {"name": "single", "n_rows": 1, "n_cols": 1, "n": 1, "seed": 2, "kind": "uniform"},
    {"name": "dup_run_600", "n_rows": 3, "n_cols": 4, "n": 600, "seed": 3, "kind": "one_key"},
    {"name": "dups_dense_50x50", "n_rows": 50, "n_cols": 50, "n": 6000, "seed": 4, "kind": "uniform"},
    {"name": "dups_mixed_mag", "n_rows": 40, "n_cols": 7, "n": 3000, "seed": 5, "kind": "mixed"},
    {"name": "signed_zeros", "n_rows": 6, "n_cols": 6, "n": 200, "seed": 6, "kind": "zeros"},
    {"name": "sparse_edges", "n_rows": 1000, "n_cols": 900, "n": 2500, "seed": 7, "kind": "edges"},
    {"name": "runs_1_to_200", "n_rows": 64, "n_cols": 64, "n": 4000, "seed": 8, "kind": "runs"},
]


def coo_case(spec):
    rng = np.random.default_rng(spec["seed"])
    n, R, C = spec["n"], spec["n_rows"], spec["n_cols"]
    k = spec["kind"]
    if k == "one_key":
        rows = np.full(n, 1, dtype=np.int64)
        cols = np.full(n, 2, dtype=np.int64)
    elif k == "edges":
        rows = rng.integers(R // 4, R - R // 4, n)  # empty leading / trailing rows
        cols = rng.integers(0, C, n)
    elif k == "runs":
        keys = np.repeat(rng.integers(0, R * C, 60), rng.integers(1, 200, 60))[:n]
        rng.shuffle(keys)
        rows, cols = keys // C, keys % C
    else:
        rows = rng.integers(0, R, n)
        cols = rng.integers(0, C, n)
    if k == "mixed":
        vals = rng.normal(size=n) * 10.0 ** rng.integers(-12, 12, n)
    elif k == "zeros":
        vals = rng.choice([0.0, -0.0, 1.0, -1.0, 1e-300, -1e-300], n)
    else:
        vals = rng.uniform(-1, 1, n)
    return R, C, rows.astype(np.int64), cols.astype(np.int64), vals.astype(np.float64)


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    os.environ["KERNELPICK_PURE_KERNELS"] = "1"
    from kernelpick import sparse
    cases = []
    for spec in SPECS:
        R, C, rows, cols, vals = coo_case(spec)
        m = sparse.csr_from_coo(R, C, rows, cols, vals)
        cases.append({"spec": spec, "row_offsets": [int(v) for v in m.row_offsets],
                      "col_indices": [int(v) for v in m.col_indices],
                      "values": [float(v).hex() for v in m.values]})
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_golden_coo.py",
                   "reference": "kernelpick.sparse.csr_from_coo (/root/reference/pkg/src/kernelpick/sparse.py:87-103)",
                   "cases": cases}, f)
    print(f"wrote {len(cases)} cases to {OUT}")


if __name__ == "__main__":
    main()
