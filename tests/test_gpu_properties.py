"""Property tests (hypothesis, SURVEY 4 / SPEC.md:140-142) on the device path:
* K1/K2 vs the oracle restatement of _pure.py / _core.pyx on generated offset arrays
  (lengths up to 2^40 so the int64 sum of squares wraps like the reference's);
* gather_features invariant under row permutation (bit-exact) and under duplicating
  every row (mean / var bit-exact);
* every SpMV kernel is linear: A(a x + b z) == a A x + b A z within the fp64 tolerance."""
import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from paper_2403_17017_b200 import _kernels, features, gen, kernels
from paper_2403_17017_b200.device import DeviceCSR

pytestmark = pytest.mark.gpu
SET = settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.too_slow])

lengths = st.lists(st.one_of(st.integers(0, 40), st.integers(0, 1 << 20), st.integers(0, 1 << 40)),
                   min_size=0, max_size=3000)


@SET
@given(ln=lengths, div=st.integers(1, 70), wave=st.integers(1, 5000))
def test_length_stats_and_waves_vs_oracle(ln, div, wave, orc):
    off = np.concatenate([[0], np.cumsum(np.asarray(ln, dtype=np.int64))]).astype(np.int64)
    assert _kernels.length_stats(off) == orc.length_stats_np(off)
    assert _kernels.wave_ceil_max_sum(off, div, wave) == orc.wave_ceil_max_sum_np(off, div, wave)


def _mat(R, C, rows, cols, seed=3):
    return gen.from_coo("h", R, C, torch.tensor(rows, dtype=torch.int64), torch.tensor(cols, dtype=torch.int64), seed)


coo = st.integers(1, 300).flatmap(lambda R: st.integers(1, 300).flatmap(
    lambda C: st.tuples(st.just(R), st.just(C), st.lists(st.tuples(st.integers(0, R - 1), st.integers(0, C - 1)),
                                                         min_size=1, max_size=4000))))


@SET
@given(case=coo, rnd=st.randoms(use_true_random=False))
def test_features_permutation_and_duplication_invariant(case, rnd):
    R, C, pairs = case
    rows, cols = zip(*pairs)
    m = _mat(R, C, rows, cols)
    off, col, _ = m.numpy()
    base = features.gather_features(m.to_device_csr(torch.float64))
    # row permutation: densities form a multiset
    perm = list(range(R))
    rnd.shuffle(perm)
    inv = np.argsort(perm)
    r2 = [int(inv[r]) for r in rows]
    p = features.gather_features(_mat(R, C, r2, cols).to_device_csr(torch.float64))
    assert p.as_vector() == base.as_vector()
    # duplicating every row keeps mean and var
    r3 = list(rows) + [r + R for r in rows]
    d = features.gather_features(_mat(2 * R, C, r3, list(cols) * 2).to_device_csr(torch.float64))
    assert (d.mean_row_density, d.var_row_density) == (base.mean_row_density, base.var_row_density)


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(case=coo, a=st.floats(-4, 4), b=st.floats(-4, 4))
def test_spmv_linearity_every_kernel(case, a, b):
    R, C, pairs = case
    rows, cols = zip(*pairs)
    A = _mat(R, C, rows, cols).to_device_csr(torch.float64)
    g = torch.Generator().manual_seed(R * 7 + C)
    x = torch.rand(C, generator=g, dtype=torch.float64).cuda()
    z = torch.rand(C, generator=g, dtype=torch.float64).cuda()
    absA = DeviceCSR(A.n_rows, A.n_cols, A.row_offsets, A.col_indices, A.values.abs())
    bound = kernels.spmv(absA, x.abs() + z.abs(), kernels.CSR_MP) * (abs(a) + abs(b) + 1)
    for k in range(len(kernels.KERNELS)):
        lhs = kernels.spmv(A, a * x + b * z, k)
        rhs = a * kernels.spmv(A, x, k) + b * kernels.spmv(A, z, k)
        assert torch.all((lhs - rhs).abs() <= 1e-12 * bound + 1e-300), kernels.KERNELS[k]
