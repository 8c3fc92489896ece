"""kp_csr_from_coo (device canonicalisation, sparse.py:87-103) vs the reference's own
outputs (golden) and the oracle restatement on larger inputs: offsets, columns and the
duplicate sums bit-exact (np.add.reduceat order and pairwise summation)."""
import json
import os
import sys

import numpy as np
import pytest
import torch

from paper_2403_17017_b200 import device, gen

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _host(A):
    off, col, val = A.to_host()
    return np.asarray(off, dtype=np.int64), np.asarray(col, dtype=np.int64), np.asarray(val, dtype=np.float64)


def _same(A, off, col, val):
    o, c, v = _host(A)
    assert np.array_equal(o, off)
    assert np.array_equal(c, col)
    assert [float(x).hex() for x in v] == [float(x).hex() for x in val]


def test_device_coo2csr_matches_reference_golden():
    sys.path.insert(0, HERE)
    from make_golden_coo import coo_case
    doc = json.load(open(os.path.join(HERE, "reference_coo_golden.json")))
    for case in doc["cases"]:
        R, C, rows, cols, vals = coo_case(case["spec"])
        A = device.csr_from_coo(R, C, rows, cols, vals)
        _same(A, np.array(case["row_offsets"]), np.array(case["col_indices"]),
              np.array([float.fromhex(h) for h in case["values"]]))


@pytest.mark.parametrize("shape,n,seed", [((1, 1), 5, 1), ((300, 70000), 200000, 2), ((2**20, 2**20), 3_000_000, 3),
                                          ((5, 2**31 - 1), 100000, 4), ((2**31 - 2, 3), 100000, 5)])
def test_device_coo2csr_matches_oracle(shape, n, seed, orc):
    R, C = shape
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, R, n)
    cols = rng.integers(0, C, n)
    if n > 1000:  # force duplicate runs
        k = n // 10
        rows[:k] = rows[k:2 * k]
        cols[:k] = cols[k:2 * k]
    vals = rng.normal(size=n) * 10.0 ** rng.integers(-8, 8, n)
    off, col, val = orc.csr_from_coo(R, C, rows, cols, vals)
    if R > 10_000_000:  # compare the non-trivial part (offsets are a long constant tail)
        A = device.csr_from_coo(R, C, rows, cols, vals)
        assert A.nnz == col.size
        assert np.array_equal(A.col_indices.cpu().numpy(), col)
        assert [float(x).hex() for x in A.values.cpu().numpy()] == [float(x).hex() for x in val]
        dev_off = A.row_offsets
        pick = torch.from_numpy(np.unique(np.concatenate([rows[:1000], [0, R - 1, R]]))).cuda()
        assert np.array_equal(dev_off[pick].cpu().numpy().astype(np.int64), off[pick.cpu().numpy()])
        return
    _same(device.csr_from_coo(R, C, rows, cols, vals), off, col, val)


def test_device_coo2csr_rmat_c2_scale(orc):
    """C2-sized R-MAT COO (16.8 M triples, ~4 % duplicates) from device tensors."""
    n = 1 << 20
    e = torch.arange(n * 16, dtype=torch.int64, device="cuda")
    rows = gen.randint(42, 2 * e, n)
    cols = gen.randint(42, 2 * e + 1, n)
    vals = gen.uniform01(43, e) * 2 - 1
    A = device.csr_from_coo(n, n, rows, cols, vals)
    off, col, val = orc.csr_from_coo(n, n, rows.cpu().numpy(), cols.cpu().numpy(), vals.cpu().numpy())
    _same(A, off, col, val)


def test_device_coo2csr_rejects_out_of_range():
    with pytest.raises(ValueError):
        device.csr_from_coo(4, 4, np.array([0, 4]), np.array([0, 0]), np.array([1.0, 2.0]))
    with pytest.raises(ValueError):
        device.csr_from_coo(4, 4, np.array([0, 1]), np.array([-1, 0]), np.array([1.0, 2.0]))
