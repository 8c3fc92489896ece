"""Multi-rank host logic of the row-sharded path on CPU (gloo, world_size 2 and 3):
nnz-balanced cuts, rank-padded column remap, in-place all-gather; the per-rank SpMV is
the CPU oracle here (test infrastructure), the GPU path uses the same plan."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_17017_b200 import dist as kdist
from paper_2403_17017_b200 import gen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_cuts_balanced():
    m = gen.config("C2", small=True)
    off = m.row_offsets.numpy()
    for P in (1, 2, 3, 8):
        cuts = kdist.partition_cuts(off, P)
        assert cuts[0] == 0 and cuts[-1] == m.n_rows and np.all(np.diff(cuts) >= 0)
        for p in range(P):  # lower_bound(off, p*nnz/P)
            assert cuts[p] == np.searchsorted(off, p * m.nnz // P, side="left")


def test_remap_roundtrip():
    rng = np.random.default_rng(0)
    cuts = np.array([0, 3, 10, 11, 20])
    plan = kdist.ShardPlan(1, 4, cuts, 20)
    cols = rng.integers(0, 20, 200)
    rc = kdist.remap_columns(cols, cuts, plan.r_max)
    x = rng.normal(size=20)
    xp = plan.pad(x)
    assert np.array_equal(xp[rc], x[cols])
    assert np.array_equal(plan.unpad(xp), x)


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    m = gen.config("C5", small=True)  # row-stochastic R-MAT (iterates stay bounded)
    off, col, val = m.numpy()
    plan = kdist.ShardPlan(rank, world, kdist.partition_cuts(off, world), m.n_rows)
    loff, lc, lv = kdist.local_csr(off, col, val, plan)
    x = np.random.default_rng(5).uniform(0, 1, m.n_rows)
    buf = torch.from_numpy(plan.pad(x).astype(np.float64))
    for _ in range(3):
        y, _ = orc.spmv_csr(loff, lc, lv, buf.numpy())
        nxt = torch.full_like(buf, float("nan"))
        nxt[rank * plan.r_max: rank * plan.r_max + plan.local_rows] = torch.from_numpy(y)
        kdist.all_gather_slices(nxt, plan)  # the exchange ShardedSeer runs (gloo: host path)
        buf = nxt
    out = plan.unpad(buf.numpy())
    # exact integer feature partials combine to the global ones
    part = torch.tensor(orc.length_stats(off[plan.r0: plan.r1 + 1]), dtype=torch.int64)
    allp = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allp, part)
    if rank == 0:
        lo = min(int(p[0]) for p in allp if True)
        hi = max(int(p[1]) for p in allp)
        s1 = sum(int(p[2]) for p in allp)
        s2 = sum(int(p[3]) for p in allp)
        ref = x
        for _ in range(3):
            ref, _ = orc.spmv_csr(off, col.astype(np.int32), val, ref)
        result_q.put((np.abs(out - ref).max(), (lo, hi, s1, s2), orc.length_stats(off)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_power_iteration_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    err, combined, full = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-12
    assert combined == full
