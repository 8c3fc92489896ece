"""Column blocking of a row shard (dist.split_columns / column_blocks, CPU part): the
slices partition the entries, keep each row's entry order, and their SpMVs sum to the
whole; the automatic slice count follows the L2 budget."""
import numpy as np
import pytest
import torch

from paper_2403_17017_b200 import dist as kdist


def test_auto_col_slices():
    l2 = 126 << 20
    budget = int(kdist.COL_SLICE_L2_FRACTION * l2)
    assert kdist.auto_col_slices(0, l2) == 1
    assert kdist.auto_col_slices(budget, l2) == 1
    assert kdist.auto_col_slices(budget + 1, l2) == 2
    assert kdist.auto_col_slices(64 << 22, l2) == 3            # C5 fp32: 268 MB x
    assert kdist.auto_col_slices(1 << 40, l2) == kdist.MAX_COL_SLICES


def test_col_slice_bounds():
    assert kdist.col_slice_bounds(10, 3) == [0, 3, 6, 10]
    assert kdist.col_slice_bounds(0, 2) == [0, 0, 0]
    with pytest.raises(ValueError):
        kdist.col_slice_bounds(10, 0)


@pytest.mark.parametrize("S", [1, 2, 3, 7])
def test_split_columns_partitions_and_sums(S):
    rng = np.random.default_rng(S)
    R, C = 300, 97
    lens = rng.integers(0, 12, R)
    lens[::17] = 0                                               # empty rows
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(C, size=n, replace=False)) for n in lens]).astype(np.int32)
    vals = rng.normal(size=cols.size)
    x = rng.normal(size=C)
    want = np.array([vals[off[r]:off[r + 1]] @ x[cols[off[r]:off[r + 1]]] for r in range(R)])
    b = kdist.col_slice_bounds(C, S)
    got = np.zeros(R)
    total = 0
    for s in range(S):
        o, c, v = kdist.split_columns(torch.from_numpy(off), torch.from_numpy(cols), torch.from_numpy(vals),
                                      b[s], b[s + 1])
        o, c, v = o.numpy(), c.numpy(), v.numpy()
        assert o[0] == 0 and np.all(np.diff(o) >= 0) and o[-1] == c.size == v.size
        assert np.all((c >= b[s]) & (c < b[s + 1]))
        total += c.size
        for r in range(R):
            cr = c[o[r]:o[r + 1]]
            keep = (cols[off[r]:off[r + 1]] >= b[s]) & (cols[off[r]:off[r + 1]] < b[s + 1])
            assert np.array_equal(cr, cols[off[r]:off[r + 1]][keep])   # same entries, same order
            got[r] += v[o[r]:o[r + 1]] @ x[cr]
    assert total == cols.size
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_compress_rows():
    off = torch.tensor([0, 0, 3, 3, 3, 5, 6, 6], dtype=torch.int64)
    o, rid = kdist.compress_rows(off)
    assert o.tolist() == [0, 3, 5, 6] and rid.tolist() == [1, 4, 5] and rid.dtype == torch.int32
    o, rid = kdist.compress_rows(torch.zeros(4, dtype=torch.int64))
    assert o.tolist() == [0] and rid.numel() == 0
