"""Row-sharded path on ONE GPU (loopback over ranks): the device partition (K14), the
rank-padded column remap and the exact feature-partial combine, checked against the
single-matrix oracle.  Real NCCL needs >= 2 GPUs; the multi-process host logic is in
test_dist_gloo.py, and ShardedSeer at world 1 runs the same code as at world N minus
the all-gather."""
import numpy as np
import pytest
import torch

from paper_2403_17017_b200 import dist as kdist
from paper_2403_17017_b200 import gen, kernels, seer

pytestmark = pytest.mark.gpu


def _model():
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    return seer.SeerModel.load(os.path.join(root, "paper_2403_17017_b200", "models", "seer_b200.json"))


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_loopback_sharded_spmv_matches_oracle(world, orc):
    m = gen.config("C5", small=True, device="cuda")
    off, col, val = m.numpy()
    x = np.random.default_rng(7).uniform(0, 1, m.n_cols)
    yref, absy = orc.spmv_csr(off, col.astype(np.int32), val, x)
    y = np.zeros(m.n_rows)
    cuts_host = kdist.partition_cuts(off, world)
    for rank in range(world):
        A, plan, cuts = kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, rank, world,
                                           torch.float64)
        assert np.array_equal(cuts.cpu().numpy(), cuts_host)  # K14 == host lower_bound restatement
        xp = plan.pad(torch.from_numpy(x).cuda())
        for kern in (kernels.CSR_WO, kernels.COO_WM, kernels.CSR_WM):
            yr = kernels.spmv(A, xp, kern).cpu().numpy()
            y[plan.r0:plan.r1] = yr
            ok, r = orc.spmv_check(y[plan.r0:plan.r1], yref[plan.r0:plan.r1], absy[plan.r0:plan.r1], 1e-12)
            assert ok, (world, rank, kernels.KERNELS[kern], r)


@pytest.mark.parametrize("world", [2, 5])
def test_partials_select_equals_single_matrix_select(world):
    from paper_2403_17017_b200.features import decode_outcome
    model = _model()
    for name in ("C4", "C5", "C2"):
        m = gen.config(name, small=True, device="cuda")
        A_full = m.to_device_csr(torch.float32)
        parts = []
        for rank in range(world):
            A, plan, _ = kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, rank, world)
            parts.append(kdist._length_partials(A))
        allp = torch.cat(parts)
        for k in (1, 20, 100):
            from paper_2403_17017_b200 import _lib
            sel, kn, ga = model.device_trees(A_full.device)
            out = torch.empty(_lib.OUTCOME_BYTES, dtype=torch.uint8, device="cuda")
            _lib.check(_lib.load().kp_seer_select_partials(allp.data_ptr(), world, m.n_rows, m.n_cols, m.nnz, k,
                                                           sel.data_ptr(), kn.data_ptr(), ga.data_ptr(),
                                                           out.data_ptr(), _lib.stream_handle()), "partials")
            got = decode_outcome(out)
            want = decode_outcome(seer.select_async(model, A_full, k))
            assert (got.kernel, got.path) == (want.kernel, want.path)
            if want.path:  # gathered: features bit-identical to the single-matrix pass
                assert [got.max_d, got.min_d, got.mean_d, got.var_d] == [want.max_d, want.min_d, want.mean_d,
                                                                         want.var_d]
        # the exact integer combine itself, independent of the selector's path
        lo = min(int(p[0]) for p in parts)
        hi = max(int(p[1]) for p in parts)
        s1 = sum(int(p[2]) for p in parts)
        s2 = sum(int(p[3]) for p in parts)
        from oracle import oracle as orc
        assert (lo, hi, s1, s2) == tuple(orc.length_stats(m.row_offsets.cpu().numpy()))


def test_sharded_seer_world1_power_iteration(orc):
    m = gen.config("C5", small=True, device="cuda")
    A, plan, _ = kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, 0, 1, torch.float64)
    run = kdist.ShardedSeer(_model(), A, plan, 3, m.n_rows, m.n_cols, m.nnz)
    x0 = torch.full((m.n_rows,), 1.0 / m.n_rows, dtype=torch.float64, device="cuda")
    got = run.step(x0).cpu().numpy()
    off, col, val = m.numpy()
    ref = x0.cpu().numpy()
    for _ in range(3):
        ref, _ = orc.spmv_csr(off, col.astype(np.int32), val, ref)
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
