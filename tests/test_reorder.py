"""Vertex reordering of a distributed matrix (dist.degree_order / permute_symmetric, CPU):
P A P^T is a permutation of A's entries, y' = A' x' equals P (A x) for x' = P x, and row
lengths (hence Seer's features) are only reordered."""
import numpy as np
import pytest
import torch

from paper_2403_17017_b200 import dist as kdist


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_permute_symmetric_is_p_a_pt(seed):
    rng = np.random.default_rng(seed)
    n = 257
    lens = rng.integers(0, 9, n)
    lens[::11] = 0
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    # skewed columns so the degree order is non-trivial
    cols = np.concatenate([np.sort(rng.choice(n, size=k, replace=False, p=None)) for k in lens])
    cols = (cols ** 2) % n
    vals = rng.normal(size=cols.size)
    order, newid = kdist.degree_order(torch.from_numpy(cols), n)
    assert torch.equal(newid[order], torch.arange(n))
    deg = np.bincount(cols, minlength=n)
    assert np.all(np.diff(deg[order.numpy()]) <= 0)              # hottest first
    o2, c2, v2 = kdist.permute_symmetric(torch.from_numpy(off), torch.from_numpy(cols),
                                         torch.from_numpy(vals), order, newid)
    o2, c2, v2 = o2.numpy(), c2.numpy(), v2.numpy()
    assert np.array_equal(np.sort(np.diff(o2)), np.sort(lens))    # row lengths only reordered
    x = rng.normal(size=n)
    y = np.array([vals[off[r]:off[r + 1]] @ x[cols[off[r]:off[r + 1]]] for r in range(n)])
    xp = np.empty(n)
    xp[newid.numpy()] = x                                         # x' = P x
    y2 = np.array([v2[o2[r]:o2[r + 1]] @ xp[c2[o2[r]:o2[r + 1]]] for r in range(n)])
    np.testing.assert_allclose(y2, y[order.numpy()], rtol=1e-12, atol=1e-12)   # y' = P y
    # entry order within a row is kept (same values, same sequence)
    r_new = 5
    r_old = int(order[r_new])
    assert np.array_equal(v2[o2[r_new]:o2[r_new + 1]], vals[off[r_old]:off[r_old + 1]])
