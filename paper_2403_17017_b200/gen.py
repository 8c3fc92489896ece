"""Seeded synthetic matrices of the BASELINE.json config shapes (C1-C5) and the
training-corpus families.  Test / benchmark infrastructure, not the hot path.

Everything is drawn from a counter-based hash (splitmix64 of (seed, counter)) in
torch int64 arithmetic, so a generator produces bit-identical matrices on the CPU
(tests, oracle) and on the GPU (bench), and any row subset can be regenerated.
Duplicates are removed by sorting the (row, col) key, which leaves each row's
columns strictly increasing (canonical form, sparse.py:33-71); the value of an
entry is a hash of its coordinates, so it does not depend on generation order.
"""

from __future__ import annotations

import math

import numpy as np
import torch

_M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    v &= _M64
    return v - (1 << 64) if v >= 1 << 63 else v


_G = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _srl(z: torch.Tensor, s: int) -> torch.Tensor:
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    z = x + _G
    z = (z ^ _srl(z, 30)) * _C1
    z = (z ^ _srl(z, 27)) * _C2
    return z ^ _srl(z, 31)


def hash2(seed: int, ctr: torch.Tensor) -> torch.Tensor:
    return splitmix64(ctr * _G + splitmix64(torch.full_like(ctr, _s64(seed))))


def uniform01(seed: int, ctr: torch.Tensor) -> torch.Tensor:
    """float64 in [0, 1) from the top 53 bits."""
    return _srl(hash2(seed, ctr), 11).to(torch.float64) * (2.0 ** -53)


def randint(seed: int, ctr: torch.Tensor, n: int) -> torch.Tensor:
    return (uniform01(seed, ctr) * n).to(torch.int64).clamp_(max=n - 1)


class Matrix:
    """Generated CSR on some torch device (int64 offsets/cols, float64 values)."""

    def __init__(self, name, n_rows, n_cols, row_offsets, col_indices, values, meta=None):
        self.name, self.n_rows, self.n_cols = name, int(n_rows), int(n_cols)
        self.row_offsets, self.col_indices, self.values = row_offsets, col_indices, values
        self.meta = dict(meta or {})

    @property
    def nnz(self) -> int:
        return int(self.col_indices.numel())

    def to_device_csr(self, dtype=torch.float32, index: str = "auto", device=None):
        from .device import DeviceCSR
        dev = device or torch.device("cuda", torch.cuda.current_device())
        use32 = index == "int32" or (index == "auto" and self.nnz < 2**31 - 1)
        off = self.row_offsets.to(dev).to(torch.int32 if use32 else torch.int64)
        return DeviceCSR(self.n_rows, self.n_cols, off, self.col_indices.to(dev).to(torch.int32),
                         self.values.to(dev).to(dtype))

    def to_sparse_csr(self):
        """Reference-layout host matrix (validates canonical form)."""
        from .sparse import SparseMatrixCSR
        return SparseMatrixCSR(self.n_rows, self.n_cols, self.row_offsets.cpu().numpy(),
                               self.col_indices.cpu().numpy(), self.values.cpu().numpy())

    def numpy(self):
        return (self.row_offsets.cpu().numpy(), self.col_indices.cpu().numpy(), self.values.cpu().numpy())


def _values_for(seed: int, rows: torch.Tensor, cols: torch.Tensor, n_cols: int, kind: str = "uniform"):
    key = rows * n_cols + cols
    if kind == "uniform":
        return uniform01(seed ^ 0x5EED, key) * 2.0 - 1.0
    raise ValueError(kind)


def from_coo(name, n_rows, n_cols, rows, cols, seed, values="uniform", meta=None) -> Matrix:
    """Dedupe (row, col) pairs by sorting the key, build offsets, hash values."""
    key = rows.to(torch.int64) * n_cols + cols.to(torch.int64)
    key = torch.unique(key, sorted=True)  # sorted unique: canonical row-major order
    r = torch.div(key, n_cols, rounding_mode="floor")
    c = key - r * n_cols
    counts = torch.bincount(r, minlength=n_rows)
    off = torch.zeros(n_rows + 1, dtype=torch.int64, device=key.device)
    torch.cumsum(counts, 0, out=off[1:])
    if values == "stochastic":  # row-stochastic 1/len (C5: iterates stay bounded)
        ln = counts.to(torch.float64)
        v = (1.0 / ln.clamp(min=1.0))[r]
    else:
        v = _values_for(seed, r, c, n_cols)
    return Matrix(name, n_rows, n_cols, off, c, v, meta)


# ---------------------------------------------------------------------------- families
def uniform_random(n_rows: int, n_cols: int, n_pairs: int, seed: int = 1, device="cpu") -> Matrix:
    """C1: n_pairs uniformly random (row, col) pairs, duplicates merged."""
    ctr = torch.arange(n_pairs, dtype=torch.int64, device=device)
    rows = randint(seed, 2 * ctr, n_rows)
    cols = randint(seed, 2 * ctr + 1, n_cols)
    return from_coo(f"uniform_{n_rows}x{n_cols}_{n_pairs}", n_rows, n_cols, rows, cols, seed)


def rmat(scale: int, edge_factor: int = 16, abc=(0.57, 0.19, 0.19), seed: int = 42, permute: bool = True,
         device="cpu", values="uniform", chunk: int = 1 << 26) -> Matrix:
    """C2 / C5: R-MAT (Chakrabarti et al.) with random row and column relabelling."""
    n = 1 << scale
    m = n * edge_factor
    a, b, c = abc
    ab, abc_ = a + b, a + b + c
    rows_all, cols_all = [], []
    for e0 in range(0, m, chunk):
        e = torch.arange(e0, min(m, e0 + chunk), dtype=torch.int64, device=device)
        r = torch.zeros_like(e)
        cc = torch.zeros_like(e)
        for lvl in range(scale):
            u = uniform01(seed, e * scale + lvl)
            bit = 1 << (scale - 1 - lvl)
            down = u >= ab                       # quadrants c, d: row bit set
            right = ((u >= a) & (u < ab)) | (u >= abc_)  # quadrants b, d: col bit set
            r += down.to(torch.int64) * bit
            cc += right.to(torch.int64) * bit
        rows_all.append(r)
        cols_all.append(cc)
    rows = torch.cat(rows_all)
    del rows_all
    cols = torch.cat(cols_all)
    del cols_all
    if permute:
        idx = torch.arange(n, dtype=torch.int64, device=device)
        prow = torch.argsort(hash2(seed + 1, idx))
        pcol = torch.argsort(hash2(seed + 2, idx))
        rows, cols = prow[rows], pcol[cols]
    return from_coo(f"rmat_s{scale}_ef{edge_factor}", n, n, rows, cols, seed, values,
                    {"scale": scale, "edge_factor": edge_factor, "abc": abc})


def stencil27(n: int, device="cpu") -> Matrix:
    """C3: 27-point stencil on an n^3 grid (row = linear grid index)."""
    N = n * n * n
    idx = torch.arange(N, dtype=torch.int64, device=device)
    z, rem = torch.div(idx, n * n, rounding_mode="floor"), idx % (n * n)
    y, x = torch.div(rem, n, rounding_mode="floor"), rem % n
    cols, rows = [], []
    for dz in (-1, 0, 1):          # lexicographic (dz, dy, dx) = increasing column index
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = (z + dz >= 0) & (z + dz < n) & (y + dy >= 0) & (y + dy < n) & (x + dx >= 0) & (x + dx < n)
                cols.append(torch.where(ok, idx + dz * n * n + dy * n + dx, torch.full_like(idx, -1)))
    C = torch.stack(cols, 1)  # [N, 27]
    valid = C >= 0
    counts = valid.sum(1)
    off = torch.zeros(N + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=off[1:])
    col = C[valid]
    row = idx.repeat_interleave(counts)
    val = _values_for(3, row, col, N)
    return Matrix(f"stencil27_{n}", N, N, off, col, val, {"grid": n})


def banded(n_rows: int, width: int, device="cpu", seed: int = 3) -> Matrix:
    """Exact band: row i holds columns i - w//2 .. i + w - w//2 - 1 clipped -> ELL-ideal."""
    idx = torch.arange(n_rows, dtype=torch.int64, device=device)
    offs = torch.arange(width, dtype=torch.int64, device=device) - width // 2
    C = idx[:, None] + offs[None, :]
    valid = (C >= 0) & (C < n_rows)
    counts = valid.sum(1)
    off = torch.zeros(n_rows + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=off[1:])
    col = C[valid]
    row = idx.repeat_interleave(counts)
    return Matrix(f"band_{n_rows}_w{width}", n_rows, n_rows, off, col, _values_for(seed, row, col, n_rows))


def _poisson_lengths(seed: int, n: int, lam: float, device) -> torch.Tensor:
    """Inverse-CDF Poisson(lam) from hashed uniforms (device independent)."""
    kmax = int(lam + 12 * math.sqrt(lam) + 20)
    pmf = np.array([math.exp(-lam + k * math.log(lam) - math.lgamma(k + 1)) for k in range(kmax)])
    cdf = torch.tensor(np.cumsum(pmf), dtype=torch.float64, device=device)
    u = uniform01(seed, torch.arange(n, dtype=torch.int64, device=device))
    return torch.searchsorted(cdf, u).clamp_(max=kmax - 1)


def skewed(n_rows: int = 2_000_000, lam: float = 8.0, n_dense: int = 4, dense_len: int = 1_000_000,
           seed: int = 7, device="cpu") -> Matrix:
    """C4: Poisson(lam) background rows with uniform columns + n_dense rows holding
    exactly dense_len distinct sorted columns (merge-path favourable)."""
    C = n_rows
    ln = _poisson_lengths(seed, n_rows, lam, device)
    rows = torch.arange(n_rows, dtype=torch.int64, device=device).repeat_interleave(ln)
    cols = randint(seed + 1, torch.arange(rows.numel(), dtype=torch.int64, device=device), C)
    dense_rows = randint(seed + 2, torch.arange(n_dense, dtype=torch.int64, device=device), n_rows)
    extra_r, extra_c = [rows], [cols]
    for i, dr in enumerate(dense_rows.tolist()):
        perm = torch.argsort(hash2(seed + 10 + i, torch.arange(C, dtype=torch.int64, device=device)))
        dc = perm[:dense_len]
        extra_r.append(torch.full((dense_len,), dr, dtype=torch.int64, device=device))
        extra_c.append(dc)
    rows = torch.cat(extra_r)
    cols = torch.cat(extra_c)
    m = from_coo(f"skewed_{n_rows}_{n_dense}x{dense_len}", n_rows, C, rows, cols, seed)
    # background duplicates may collide with a dense row: keep exactly dense_len there
    m.meta["dense_rows"] = sorted(set(dense_rows.tolist()))
    return m


def powerlaw_rows(n_rows: int, mean: float, alpha: float = 1.5, seed: int = 11, device="cpu",
                  n_cols: int | None = None) -> Matrix:
    """Corpus family: Pareto(alpha) row lengths scaled to ``mean``, uniform columns."""
    C = n_cols or n_rows
    u = uniform01(seed, torch.arange(n_rows, dtype=torch.int64, device=device))
    raw = (1.0 - u).pow(-1.0 / alpha)                  # Pareto >= 1, mean alpha/(alpha-1)
    ln = (raw * (mean * (alpha - 1) / alpha)).floor().to(torch.int64).clamp_(max=C)
    rows = torch.arange(n_rows, dtype=torch.int64, device=device).repeat_interleave(ln)
    cols = randint(seed + 1, torch.arange(rows.numel(), dtype=torch.int64, device=device), C)
    return from_coo(f"powerlaw_{n_rows}_m{mean}_a{alpha}", n_rows, C, rows, cols, seed)


def constant_rows(n_rows: int, length: int, seed: int = 5, device="cpu", n_cols: int | None = None) -> Matrix:
    """Corpus family: every row has ~``length`` uniformly random columns."""
    C = n_cols or n_rows
    rows = torch.arange(n_rows, dtype=torch.int64, device=device).repeat_interleave(length)
    cols = randint(seed, torch.arange(rows.numel(), dtype=torch.int64, device=device), C)
    return from_coo(f"const_{n_rows}_l{length}", n_rows, C, rows, cols, seed)


# ------------------------------------------------------ structured families (OOD checks)
# Held out of the frozen bundle's corpus families: finite-element meshes, circuit
# (modified-nodal-analysis) matrices and road networks -- the structures SuiteSparse adds on
# top of the synthetic generators (PAPER.md:330 evaluates on all of SuiteSparse).
def _sym_coo(name, n, rows, cols, seed, meta=None, diag=True) -> Matrix:
    dev = rows.device
    r = torch.cat([rows, cols] + ([torch.arange(n, dtype=torch.int64, device=dev)] if diag else []))
    c = torch.cat([cols, rows] + ([torch.arange(n, dtype=torch.int64, device=dev)] if diag else []))
    return from_coo(name, n, n, r, c, seed, meta=meta)


def fem_mesh(n: int, order: int = 1, tile: int = 64, seed: int = 21, device="cpu") -> Matrix:
    """2-D triangulated n x n vertex lattice (each square split along one diagonal): P1
    elements couple a vertex with its 6 lattice neighbours (7-point rows), P2 with every
    vertex of the adjacent triangles' edge midpoints as well (order 2: lattice distance
    <= 2 along the triangulation, ~19-point rows).  Vertices are renumbered inside tiles of
    `tile` consecutive indices (a mesh generator's local ordering): locality stays, exact
    bands do not.  Boundary rows are shorter."""
    N = n * n
    idx = torch.arange(N, dtype=torch.int64, device=device)
    i, j = torch.div(idx, n, rounding_mode="floor"), idx % n
    nb = [(0, 1), (1, 0), (1, -1)] if order == 1 else \
        [(0, 1), (1, 0), (1, -1), (0, 2), (2, 0), (2, -2), (1, 1), (2, -1), (1, -2)]
    rows, cols = [], []
    for di, dj in nb:
        ok = (i + di < n) & (j + dj >= 0) & (j + dj < n)
        rows.append(idx[ok])
        cols.append((idx + di * n + dj)[ok])
    rows, cols = torch.cat(rows), torch.cat(cols)
    # renumber within tiles: a hashed permutation of each tile's indices
    key = torch.div(idx, tile, rounding_mode="floor") * (1 << 40) + (hash2(seed, idx) >> 24)
    perm = torch.empty_like(idx)
    perm[torch.argsort(key)] = idx
    return _sym_coo(f"fem_p{order}_{n}", N, perm[rows], perm[cols], seed, {"grid": n, "order": order})


def circuit(n: int, n_rails: int = 8, rail_frac: float = 0.1, seed: int = 23, device="cpu") -> Matrix:
    """Modified-nodal-analysis-like pattern: every node couples to 1-4 nodes of a local
    window (a netlist's hierarchical locality, window 256), `n_rails` supply / ground nodes
    couple to a `rail_frac` fraction of all nodes (dense rows AND dense columns), symmetric
    with a diagonal."""
    ctr = torch.arange(n, dtype=torch.int64, device=device)
    deg = 1 + randint(seed, ctr, 4)
    src = ctr.repeat_interleave(deg)
    e = torch.arange(src.numel(), dtype=torch.int64, device=device)
    dst = (src + randint(seed + 1, e, 512) - 256).clamp_(0, n - 1)
    rails = randint(seed + 2, torch.arange(n_rails, dtype=torch.int64, device=device), n)
    m = int(n * rail_frac)
    rr = [src]
    cc = [dst]
    for k, r in enumerate(rails.tolist()):
        tgt = randint(seed + 10 + k, torch.arange(m, dtype=torch.int64, device=device), n)
        rr.append(torch.full((m,), r, dtype=torch.int64, device=device))
        cc.append(tgt)
    return _sym_coo(f"circuit_{n}_r{n_rails}_f{rail_frac}", n, torch.cat(rr), torch.cat(cc), seed,
                    {"rails": n_rails, "rail_frac": rail_frac})


def road(side: int, keep: float = 0.62, shortcut: float = 0.01, seed: int = 25, device="cpu") -> Matrix:
    """Road-network-like graph Laplacian pattern: a side x side grid with each lattice edge
    kept with probability `keep` (mean degree ~2.5), a `shortcut` fraction of vertices with
    one edge to a vertex within +-2 rows (ramps), row-major vertex order (spatial locality,
    no band structure beyond the grid width).  Symmetric with a diagonal."""
    N = side * side
    idx = torch.arange(N, dtype=torch.int64, device=device)
    i, j = torch.div(idx, side, rounding_mode="floor"), idx % side
    rows, cols = [], []
    for k, (di, dj) in enumerate(((0, 1), (1, 0))):
        ok = (i + di < side) & (j + dj < side) & (uniform01(seed + k, idx) < keep)
        rows.append(idx[ok])
        cols.append((idx + di * side + dj)[ok])
    sc = idx[uniform01(seed + 5, idx) < shortcut]
    if sc.numel():
        off = (randint(seed + 6, sc, 4 * side + 1) - 2 * side)
        rows.append(sc)
        cols.append((sc + off).clamp_(0, N - 1))
    return _sym_coo(f"road_{side}_k{keep}", N, torch.cat(rows), torch.cat(cols), seed, {"side": side})


# ---------------------------------------------------------------------------- configs
def config(name: str, device="cpu", small: bool = False) -> Matrix:
    """BASELINE.json configs by short name (C1..C5); small=True gives a reduced
    instance of the same family for CPU-side tests."""
    if name == "C1":
        return uniform_random(10_000, 10_000, 100_000, seed=1, device=device)
    if name == "C2":
        return rmat(12 if small else 20, 16, seed=42, device=device)
    if name == "C3":
        return stencil27(12 if small else 159, device=device)
    if name == "C4":
        return skewed(20_000, 8.0, 4, 10_000, seed=7, device=device) if small else skewed(device=device)
    if name == "C5":
        return rmat(12 if small else 26, 16, seed=42, device=device, values="stochastic")
    raise ValueError(name)
