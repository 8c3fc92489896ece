"""Generate golden vectors from the UNMODIFIED reference (run in the build container).

    python tests/golden/make_golden.py            # writes tests/golden/reference_golden.json

Imports the reference package read-only from /root/reference/pkg/src and records:

* ``_kernels.length_stats`` / ``wave_ceil_max_sum`` outputs with the numpy backend
  (KERNELPICK_PURE_KERNELS=1, _kernels/__init__.py:13) AND the compiled Cython
  backend (oracle/_ref, built from the reference _core.pyx by ``make -C oracle ref``)
  on writable copies -- asserting the two reference backends agree first;
* ``features.gather_features`` on real ``SparseMatrixCSR`` objects (SPEC.md:118-120
  examples plus seeded random matrices) with a FixedClock, floats stored as
  ``float.hex`` so parity is bit-exact.

The GPU box never runs this (no /root/reference there); it only reads the JSON.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")


def _import_reference():
    os.environ["KERNELPICK_PURE_KERNELS"] = "1"
    sys.path.insert(0, REF_SRC)
    from kernelpick import _kernels, clock, features, sparse  # noqa: E402
    assert _kernels.BACKEND == "pure"
    return _kernels, clock, features, sparse


def _offset_cases(rng) -> list[np.ndarray]:
    cases = [
        np.array([], dtype=np.int64),
        np.array([0], dtype=np.int64),
        np.array([0, 0], dtype=np.int64),
        np.array([0, 7], dtype=np.int64),
        np.array([0, 4, 4, 9, 10], dtype=np.int64),          # SURVEY 8c probe KAT
        np.array([0, 4, 4], dtype=np.int64),                  # SPEC.md:118 rows [4,0]
        np.array([0, 1, 3, 6], dtype=np.int64),               # SPEC.md:120 rows [1,2,3]
        np.array([0, 2**32], dtype=np.int64),                 # len^2 == 2**64 wraps to 0
        np.array([0, 3037000500, 3037000500 * 2], dtype=np.int64),  # s2 wraps negative
    ]
    for n in (1, 2, 3, 31, 32, 33, 63, 64, 65, 127, 255, 256, 257, 1000, 4097, 10000):
        for dist in ("uniform", "poisson", "powerlaw", "empty-heavy", "const"):
            if dist == "uniform":
                ln = rng.integers(0, 50, n)
            elif dist == "poisson":
                ln = rng.poisson(8, n)
            elif dist == "powerlaw":
                ln = np.minimum((rng.pareto(1.2, n) * 3).astype(np.int64), 10**6)
            elif dist == "empty-heavy":
                ln = rng.integers(0, 3, n) * (rng.random(n) < 0.3)
            else:
                ln = np.full(n, 27)
            off = np.zeros(n + 1, dtype=np.int64)
            np.cumsum(ln, out=off[1:])
            cases.append(off)
    # offsets that do not start at 0 (the backend only differences them)
    cases.append(np.array([5, 9, 9, 30], dtype=np.int64))
    return cases


def _wave_params():
    return [(1, 1), (1, 64), (2, 3), (8, 8), (3, 5), (32, 2), (1000, 7), (7, 1000)]


def _matrix_cases(rng, sparse):
    mats = []
    # 2x4, rows nnz [4, 0]
    mats.append(("spec118", sparse.csr_from_coo(2, 4, [0, 0, 0, 0], [0, 1, 2, 3], [1.0] * 4)))
    # any 1-row matrix
    mats.append(("spec119", sparse.csr_from_coo(1, 5, [0, 0], [1, 3], [2.0, 3.0])))
    # 3x10, rows nnz [1, 2, 3]
    mats.append(("spec120", sparse.csr_from_coo(3, 10, [0, 1, 1, 2, 2, 2], [0, 0, 1, 0, 1, 2],
                                                [1.0] * 6)))
    for i, (n, c, z) in enumerate([(10, 10, 30), (100, 37, 500), (1000, 1000, 5000),
                                   (3000, 200, 40000), (257, 10**6, 3000), (5000, 5000, 1),
                                   (2000, 50, 2000)]):
        r = rng.integers(0, n, z)
        cc = rng.integers(0, c, z)
        v = rng.uniform(-1, 1, z)
        mats.append((f"rand{i}", sparse.csr_from_coo(n, c, r, cc, v)))
    # skewed: a few dense rows over a Poisson background
    n, c = 4000, 3000
    ln = rng.poisson(3, n)
    ln[[7, 1999, 3998]] = [3000, 2500, 2999]
    rows = np.repeat(np.arange(n), ln)
    cols = np.concatenate([rng.choice(c, size=l, replace=False) for l in ln])
    mats.append(("skew", sparse.csr_from_coo(n, c, rows, cols, np.ones(rows.size))))
    return mats


def main() -> None:
    _kernels, clock, features, sparse = _import_reference()
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
    from oracle import oracle as orc
    core = orc.ref_core()
    if core is None:
        orc.build()
        core = orc.ref_core()
    rng = np.random.default_rng(20240317)

    stats = []
    for off in _offset_cases(rng):
        pure = _kernels.length_stats(off)
        if core is not None:
            comp = core.length_stats(off.copy())  # writable copy
            assert tuple(comp) == tuple(pure), (off[:8], comp, pure)
        waves = []
        for d, w in _wave_params():
            wp = _kernels.wave_ceil_max_sum(off, d, w)
            if core is not None:
                assert core.wave_ceil_max_sum(off.copy(), d, w) == wp
            waves.append([d, w, int(wp)])
        stats.append({"offsets": off.tolist(), "length_stats": [int(v) for v in pure],
                      "wave": waves})

    feats = []
    for name, m in _matrix_cases(rng, sparse):
        g = features.gather_features(m, clock.FixedClock(tick=0.25))
        feats.append({
            "name": name, "n_rows": m.n_rows, "n_cols": m.n_cols,
            "row_offsets": m.row_offsets.tolist(),
            "length_stats": [int(v) for v in _kernels.length_stats(m.row_offsets)],
            "features_hex": [float(v).hex() for v in g.as_vector()],
            "collection_time": g.collection_time,
            "known": [sparse.known_features(m).rows, sparse.known_features(m).cols,
                      sparse.known_features(m).nnz],
        })

    # Epilogue-only vectors over random integer aggregates (A5-style), straight
    # through the reference gather_features with a duck-typed matrix whose
    # row_offsets reproduce the aggregates exactly.
    epi = []
    for _ in range(3000):
        n = int(rng.integers(1, 5000))
        c = int(rng.integers(1, 10**7))
        ln = rng.integers(0, min(c, 10**5) + 1, n) if rng.random() < 0.5 else \
            np.minimum(rng.poisson(rng.uniform(0.1, 50), n), c)
        off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(ln, out=off[1:])

        class _M:  # gather_features duck-types n_rows / n_cols / row_offsets (features.py:67-74)
            pass
        m = _M()
        m.n_rows, m.n_cols, m.row_offsets = n, c, off
        g = features.gather_features(m, clock.FixedClock())
        epi.append({"n": n, "c": c, "agg": [int(v) for v in _kernels.length_stats(off)],
                    "features_hex": [float(v).hex() for v in g.as_vector()]})

    doc = {
        "generator": "tests/golden/make_golden.py",
        "reference": "/root/reference/pkg/src/kernelpick (KERNELPICK_PURE_KERNELS=1; "
                     "compiled _core cross-checked: %s)" % (core is not None),
        "length_stats": stats,
        "gather_features": feats,
        "epilogue": epi,
    }
    with open(OUT, "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print(f"wrote {OUT}: {len(stats)} offset cases, {len(feats)} matrices, {len(epi)} epilogue vectors")


if __name__ == "__main__":
    main()
