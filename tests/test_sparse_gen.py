import numpy as np
import pytest
import torch

from paper_2403_17017_b200 import gen, sparse


def test_known_features_examples():
    m = sparse.csr_from_coo(3, 4, [0, 0, 1, 2, 2], [0, 3, 1, 0, 2], [1, 2, 3, 4, 5])
    assert sparse.known_features(m) == sparse.KnownFeatures(3, 4, 5)
    assert sparse.known_features(sparse.SparseMatrixCSR(0, 0, [0], [], [])) == sparse.KnownFeatures(0, 0, 0)


def test_csr_from_coo_sums_duplicates_and_sorts():
    m = sparse.csr_from_coo(3, 3, [0, 0, 2, 1], [0, 0, 1, 2], [1.0, 2.0, 5.0, 7.0])
    assert m.row_offsets.tolist() == [0, 1, 2, 3]
    assert m.col_indices.tolist() == [0, 2, 1] and m.values.tolist() == [3.0, 7.0, 5.0]
    assert not m.row_offsets.flags.writeable


def test_validation():
    with pytest.raises(ValueError):
        sparse.SparseMatrixCSR(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        sparse.SparseMatrixCSR(1, 2, [0, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(ValueError):
        sparse.SparseMatrixCSR(1, 2, [0, 1], [2], [1.0])
    sparse.SparseMatrixCSR(2, 2, [0, 1, 2], [1, 0], [1.0, 1.0])  # decrease across rows is fine


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_generators_canonical_and_deterministic(name):
    a = gen.config(name, small=True)
    b = gen.config(name, small=True)
    assert torch.equal(a.row_offsets, b.row_offsets) and torch.equal(a.col_indices, b.col_indices)
    assert torch.equal(a.values, b.values)
    a.to_sparse_csr()  # validates canonical form


def test_stencil_nnz_formula():
    m = gen.stencil27(7)
    assert m.nnz == (3 * 7 - 2) ** 3
    assert int((m.row_offsets[1:] - m.row_offsets[:-1]).max()) == 27


def test_skewed_has_dense_rows():
    m = gen.config("C4", small=True)
    ln = (m.row_offsets[1:] - m.row_offsets[:-1])
    assert int(ln.max()) >= 10_000


def test_gpu_parity_fixtures_are_canonical():
    """The GPU parity matrices themselves must be valid CSR (caught an out-of-range fixture)."""
    import test_gpu_spmv as t
    assert len(t.mats()) >= 13


@pytest.mark.parametrize("make", [
    lambda: gen.fem_mesh(40, 1), lambda: gen.fem_mesh(30, 2), lambda: gen.circuit(3000, 4, 0.05),
    lambda: gen.road(50, 0.6)])
def test_structured_families_are_canonical_and_symmetric(make):
    """The OOD families (gen.fem_mesh / circuit / road): canonical CSR (sorted, unique, in
    range -- SparseMatrixCSR's checks), a symmetric pattern with a full diagonal, and the
    row-length shapes they stand for."""
    m = make()
    sp = m.to_sparse_csr()
    off, col = np.asarray(sp.row_offsets), np.asarray(sp.col_indices)
    n = m.n_rows
    rows = np.repeat(np.arange(n), np.diff(off))
    pairs = set(zip(rows.tolist(), col.tolist()))
    assert all((c, r) in pairs for r, c in pairs)
    assert all((i, i) in pairs for i in range(n))
    ln = np.diff(off)
    if m.name.startswith("fem_p1"):
        assert ln.max() == 7 and ln.min() >= 3
    elif m.name.startswith("fem_p2"):
        assert ln.max() == 19
    elif m.name.startswith("circuit"):
        assert ln.max() > 10 * np.median(ln)  # supply rails: dense rows (and columns)
    else:
        assert ln.max() <= 8 and 2.5 < ln.mean() < 4.5


def test_structured_families_are_seeded():
    a, b = gen.circuit(2000, 3, 0.1, seed=5), gen.circuit(2000, 3, 0.1, seed=5)
    assert np.array_equal(a.col_indices.numpy(), b.col_indices.numpy())
    c = gen.circuit(2000, 3, 0.1, seed=6)
    assert not (c.nnz == a.nnz and np.array_equal(a.col_indices.numpy(), c.col_indices.numpy()))
