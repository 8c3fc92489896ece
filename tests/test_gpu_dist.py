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


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("kern", [kernels.CSR_WO, kernels.CSR_MP])
def test_fused_exchange_loopback(world, kern, orc):
    """kp_spmv_bcast on one GPU with `world` simulated ranks: every rank's kernel stores its
    y slice into ALL ranks' next-x buffers (distinct local tensors standing in for the peer
    mappings); afterwards every buffer must hold the full next x (= the oracle's A.x)."""
    from paper_2403_17017_b200 import _lib
    L = _lib.load()
    prev = L.kp_debug_set_wave_warps(7)  # many units per warp: range-end carries -> fix-up broadcast
    try:
        m = gen.config("C5", small=True, device="cuda")
        off, col, val = m.numpy()
        x = np.random.default_rng(11).uniform(0, 1, m.n_cols)
        yref, absy = orc.spmv_csr(off, col.astype(np.int32), val, x)
        shards = [kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, r, world, torch.float64)
                  for r in range(world)]
        plan0 = shards[0][1]
        n = world * plan0.r_max
        nxt = [torch.full((n,), float("nan"), dtype=torch.float64, device="cuda") for _ in range(world)]
        for r, (A, plan, _) in enumerate(shards):
            xp = plan.pad(torch.from_numpy(x).cuda())
            dests = [nxt[q][r * plan.r_max: r * plan.r_max + plan.local_rows] for q in range(world)]
            kernels.spmv_bcast(A, xp, kern, dests, r)
        torch.cuda.synchronize()
        for q in range(world):
            got = plan0.unpad(nxt[q]).cpu().numpy()
            ok, ratio = orc.spmv_check(got, yref, absy, 1e-12)
            assert ok, (world, q, ratio)
    finally:
        L.kp_debug_set_wave_warps(prev)


def test_sharded_seer_fused_symmetric_memory_world1(orc):
    """ShardedSeer with exchange="fused" through torch symmetric memory at world size 1
    (the same code path as N ranks: symm-mem rendezvous, peer-mapped destinations,
    device barrier), vs the oracle power iteration."""
    import socket
    import torch.distributed as tdist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                             device_id=torch.device("cuda", 0))
    try:
        m = gen.config("C5", small=True, device="cuda")
        A, plan, _ = kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, 0, 1, torch.float64)
        model = _model()
        run = kdist.ShardedSeer(model, A, plan, 3, m.n_rows, m.n_cols, m.nnz, exchange="fused",
                                kernel=kernels.CSR_WO)
        assert run.exchange == "fused"
        x0 = torch.full((m.n_rows,), 1.0 / m.n_rows, dtype=torch.float64, device="cuda")
        got = run.step(x0).cpu().numpy()
        off, col, val = m.numpy()
        ref = x0.cpu().numpy()
        for _ in range(3):
            ref, _ = orc.spmv_csr(off, col.astype(np.int32), val, ref)
        assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
    finally:
        tdist.destroy_process_group()


def test_bench_gpus2_sharded_control_flow():
    """`python bench.py --gpus 2` without torchrun: two local ranks (gloo when the box has
    one GPU: ranks share it), row-sharded C5 family at a reduced scale, the host-staged y
    exchange, global selection from partials and the sampled-row parity check."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--scale", "16", "--steps", "2",
                        "--warmup", "1", "--iters", "3", "--watchdog-s", "120"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"].startswith("row-sharded x2")
    assert line["comm"]["nranks"] == 2 and line["parity"]["ok"]
    assert line["scaling"] == "strong" and line["value"] > 0


_WD_SCRIPT = r"""
import socket, sys, time, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
from paper_2403_17017_b200 import dist as kdist
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
wd = kdist.Watchdog.start(timeout_s=30.0)
assert wd is not None, "no NCCL communicator exposed"
t = torch.ones(8, device="cuda"); dist.all_reduce(t); torch.cuda.synchronize()
wd.heartbeat()
print("OK_STATE", wd.stop()["state"])
wd = kdist.Watchdog.start(timeout_s=0.2)
time.sleep(1.0)
try:
    wd.heartbeat()
    print("NO_TIMEOUT")
except RuntimeError as e:
    print("TIMEOUT_RAISED", e)
print("FINAL", wd.stop()["state"])
sys.stdout.flush()
import os; os._exit(0)  # the communicator was aborted: skip the process-group teardown
"""


def test_nccl_watchdog_heartbeat_and_timeout():
    """kp_watchdog on a real NCCL communicator (world 1): healthy with heartbeats; with no
    heartbeat inside the timeout it aborts the communicator and the next heartbeat raises."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", _WD_SCRIPT, root], capture_output=True, text=True, timeout=300)
    assert "OK_STATE ok" in p.stdout, (p.stdout, p.stderr[-2000:])
    assert "TIMEOUT_RAISED" in p.stdout and "FINAL timeout" in p.stdout, (p.stdout, p.stderr[-2000:])


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("kern", [kernels.CSR_WO, kernels.CSR_MP])
@pytest.mark.parametrize("mode", ["none", "separate", "alias"])
def test_bcast_acc_matches_oracle(dtype, kern, mode, orc):
    """kp_spmv_bcast_acc: every destination receives acc + A.x; acc may be the self
    destination itself (the in-place accumulation of the column blocks)."""
    from paper_2403_17017_b200 import _lib
    L = _lib.load()
    prev = L.kp_debug_set_wave_warps(7)  # range-end carries: the fix-up must not re-add acc
    try:
        m = gen.config("C5", small=True, device="cuda")
        A = m.to_device_csr(dtype)
        off, col, val = m.numpy()
        rng = np.random.default_rng(3)
        x = rng.uniform(0, 1, m.n_cols)
        a0 = rng.normal(size=m.n_rows)
        vv = val.astype(np.float32).astype(np.float64) if dtype == torch.float32 else val
        yref, absy = orc.spmv_csr(off, col.astype(np.int32), vv, x.astype(np.float32).astype(np.float64)
                                  if dtype == torch.float32 else x)
        xd = torch.from_numpy(x).to(dtype).cuda()
        dests = [torch.full((m.n_rows,), float("nan"), dtype=dtype, device="cuda") for _ in range(3)]
        acc = None
        if mode != "none":
            a0 = torch.from_numpy(a0).to(dtype).double().numpy()
            if mode == "alias":
                dests[1].copy_(torch.from_numpy(a0))
                acc = dests[1]
            else:
                acc = torch.from_numpy(a0).to(dtype).cuda()
            yref, absy = yref + a0, absy + np.abs(a0)
        kernels.spmv_bcast(A, xd, kern, dests, 1, acc=acc)
        torch.cuda.synchronize()
        tol = 1e-5 if dtype == torch.float32 else 1e-12
        for q, d in enumerate(dests):
            ok, r = orc.spmv_check(d.double().cpu().numpy(), yref, absy, tol)
            assert ok, (q, mode, r)
    finally:
        L.kp_debug_set_wave_warps(prev)


@pytest.mark.parametrize("compact", [True, False])
@pytest.mark.parametrize("world", [1, 3])
@pytest.mark.parametrize("S", [2, 3, 5])
def test_column_blocks_loopback_matches_oracle(world, S, compact, orc):
    """Column-blocked row shards (dist.column_blocks + accumulating stores, the last block's
    stores to every rank's next-x buffer), `world` simulated ranks on one GPU."""
    m = gen.config("C5", small=True, device="cuda")
    off, col, val = m.numpy()
    x = np.random.default_rng(13).uniform(0, 1, m.n_cols)
    yref, absy = orc.spmv_csr(off, col.astype(np.int32), val, x)
    shards = [kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, r, world, torch.float64)
              for r in range(world)]
    plan0 = shards[0][1]
    n = world * plan0.r_max
    nxt = [torch.full((n,), float("nan"), dtype=torch.float64, device="cuda") for _ in range(world)]
    for r, (A, plan, _) in enumerate(shards):
        blocks = kdist.column_blocks(A, S, compact=compact)
        assert sum(B.nnz for B, _ in blocks) == A.nnz
        assert (blocks[0][1] is not None) == compact and blocks[-1][1] is None
        xp = plan.pad(torch.from_numpy(x).cuda())
        acc = torch.empty(plan.local_rows, dtype=torch.float64, device="cuda")
        if compact:
            acc.zero_()
        for s, (B, rid) in enumerate(blocks[:-1]):
            if rid is not None:
                assert B.n_rows == rid.numel() <= plan.local_rows
                if B.n_rows:
                    kernels.spmv_bcast(B, xp, kernels.CSR_WO if s % 2 else kernels.CSR_MP, [acc], 0, acc=acc,
                                       rows=rid)
            else:
                kernels.spmv_bcast(B, xp, kernels.CSR_WO, [acc], 0, acc=acc if s else None)
        dests = [nxt[q][r * plan.r_max: r * plan.r_max + plan.local_rows] for q in range(world)]
        kernels.spmv_bcast(blocks[-1][0], xp, kernels.CSR_MP, dests, r, acc=acc)
    torch.cuda.synchronize()
    for q in range(world):
        ok, ratio = orc.spmv_check(plan0.unpad(nxt[q]).cpu().numpy(), yref, absy, 1e-12)
        assert ok, (world, S, q, ratio)


@pytest.mark.parametrize("compact", [True, False])
@pytest.mark.parametrize("S", [1, 3, 4])
@pytest.mark.parametrize("kern", [kernels.CSR_WO, kernels.CSR_MP])
def test_sharded_seer_column_blocked_power_iteration(S, kern, compact, orc):
    """ShardedSeer(col_slices=S) at world 1 (no process group: local exchange) == the
    oracle's power iteration; S = 1 is the unblocked path; compressed-row or full blocks."""
    m = gen.config("C5", small=True, device="cuda")
    A, plan, _ = kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, 0, 1, torch.float64)
    run = kdist.ShardedSeer(_model(), A, plan, 3, m.n_rows, m.n_cols, m.nnz, kernel=kern, col_slices=S,
                            compact_blocks=compact)
    assert run.col_slices == S and len(run.blocks) == S
    x0 = torch.full((m.n_rows,), 1.0 / m.n_rows, dtype=torch.float64, device="cuda")
    got = run.step(x0).cpu().numpy()
    off, col, val = m.numpy()
    ref = x0.cpu().numpy()
    for _ in range(3):
        ref, _ = orc.spmv_csr(off, col.astype(np.int32), val, ref)
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_sharded_seer_column_blocked_fused_world1(orc):
    """Column blocks + the fused symmetric-memory exchange (world 1), fp32 at 1e-5."""
    import socket
    import torch.distributed as tdist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                             device_id=torch.device("cuda", 0))
    try:
        m = gen.config("C5", small=True, device="cuda")
        A, plan, _ = kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, 0, 1, torch.float32)
        run = kdist.ShardedSeer(_model(), A, plan, 2, m.n_rows, m.n_cols, m.nnz, exchange="fused",
                                kernel=kernels.CSR_WO, col_slices=3)
        assert run.exchange == "fused" and run.col_slices == 3
        x0 = torch.rand(m.n_rows, dtype=torch.float32, device="cuda")
        got = run.step(x0).double().cpu().numpy()
        off, col, val = m.numpy()
        v32 = val.astype(np.float32).astype(np.float64)
        ref = x0.double().cpu().numpy()
        y1, _ = orc.spmv_csr(off, col.astype(np.int32), v32, ref)
        y1 = y1.astype(np.float32).astype(np.float64)
        y2, absy = orc.spmv_csr(off, col.astype(np.int32), v32, y1)
        ok, ratio = orc.spmv_check(got, y2, absy, 2e-5)
        assert ok, ratio
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("kern", [kernels.CSR_WO, kernels.CSR_MP])
def test_column_blocks_with_an_empty_block(kern, orc):
    """A block with no entries (every column in the first half): the accumulating store
    path must still deliver acc + 0 to the destinations (the nnz == 0 branch of
    kp_spmv_bcast_acc), and an empty first block zero-initialises the accumulator."""
    rng = np.random.default_rng(21)
    n = 5000
    lens = rng.integers(0, 9, n)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    for lo, hi in ((0, n // 2 - 1), (n // 2 + 1, n)):   # entries only in one half
        col = np.concatenate([np.sort(rng.choice(np.arange(lo, hi), size=k, replace=False)) for k in lens])
        val = rng.uniform(0, 1, col.size)
        from paper_2403_17017_b200.device import DeviceCSR
        A = DeviceCSR(n, n, torch.from_numpy(off).cuda(), torch.from_numpy(col.astype(np.int32)).cuda(),
                      torch.from_numpy(val).cuda())
        plan = kdist.ShardPlan(0, 1, np.array([0, n]), n)
        run = kdist.ShardedSeer(None, A, plan, 2, n, n, int(col.size), kernel=kern, col_slices=2)
        assert min(B.nnz for B in run.blocks) == 0
        x0 = torch.from_numpy(rng.uniform(0, 1, n)).cuda()
        got = run.step(x0).cpu().numpy()
        ref = x0.cpu().numpy()
        for _ in range(2):
            ref, _ = orc.spmv_csr(off, col.astype(np.int32), val, ref)
        assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("kern", [kernels.CSR_WO, kernels.CSR_MP])
def test_bcast_row_map_in_place(dtype, kern, orc):
    """kp_spmv_bcast_acc with a row map: dest[rows[r]] += (A x)[r] in place, every other
    row untouched -- with range-end carries through the fix-up (few resident warps)."""
    from paper_2403_17017_b200 import _lib
    L = _lib.load()
    prev = L.kp_debug_set_wave_warps(7)
    try:
        m = gen.config("C5", small=True, device="cuda")
        off, col, val = m.numpy()
        rng = np.random.default_rng(17)
        n_dest = m.n_rows * 3
        rows = np.sort(rng.choice(n_dest, size=m.n_rows, replace=False)).astype(np.int32)
        A = m.to_device_csr(dtype)
        x = rng.uniform(0, 1, m.n_cols)
        base = rng.normal(size=n_dest)
        d = torch.from_numpy(base).to(dtype).cuda()
        base = d.double().cpu().numpy()
        xd = torch.from_numpy(x).to(dtype).cuda()
        vv = val.astype(np.float32).astype(np.float64) if dtype == torch.float32 else val
        xx = x.astype(np.float32).astype(np.float64) if dtype == torch.float32 else x
        y, absy = orc.spmv_csr(off, col.astype(np.int32), vv, xx)
        kernels.spmv_bcast(A, xd, kern, [d], 0, acc=d, rows=torch.from_numpy(rows).cuda())
        got = d.double().cpu().numpy()
        want = base.copy()
        want[rows] += y
        bound = np.zeros(n_dest)
        bound[rows] = absy
        ok, r = orc.spmv_check(got, want, bound + np.abs(base), 1e-5 if dtype == torch.float32 else 1e-12)
        assert ok, r
        untouched = np.setdiff1d(np.arange(n_dest), rows)
        assert np.array_equal(got[untouched], base[untouched])
        with pytest.raises(ValueError):  # a row map scatters into exactly one destination
            kernels.spmv_bcast(A, xd, kern, [d, d], 0, acc=d, rows=torch.from_numpy(rows).cuda())
    finally:
        L.kp_debug_set_wave_warps(prev)


@pytest.mark.parametrize("world", [1, 3])
def test_reordered_shards_power_iteration(world, orc):
    """P A P^T distributed (dist.degree_order + permute_symmetric), `world` simulated ranks
    on one GPU with the fused-epilogue stores into every rank's buffer: after mapping back
    through newid, one iteration equals the oracle's A x on the ORIGINAL matrix."""
    m = gen.config("C5", small=True, device="cuda")
    off, col, val = m.numpy()
    n = m.n_rows
    order, newid = kdist.degree_order(m.col_indices, n)
    o2, c2, v2 = kdist.permute_symmetric(m.row_offsets, m.col_indices, m.values, order, newid)
    x = np.random.default_rng(29).uniform(0, 1, n)
    yref, absy = orc.spmv_csr(off, col.astype(np.int32), val, x)
    xp = np.empty(n)
    nid = newid.cpu().numpy()
    xp[nid] = x
    shards = [kdist.shard_device(o2, c2, v2, n, r, world, torch.float64) for r in range(world)]
    plan0 = shards[0][1]
    nxt = [torch.full((world * plan0.r_max,), float("nan"), dtype=torch.float64, device="cuda")
           for _ in range(world)]
    for r, (A, plan, _) in enumerate(shards):
        xpad = plan.pad(torch.from_numpy(xp).cuda())
        dests = [nxt[q][r * plan.r_max: r * plan.r_max + plan.local_rows] for q in range(world)]
        kernels.spmv_bcast(A, xpad, kernels.CSR_WO, dests, r)
    torch.cuda.synchronize()
    for q in range(world):
        got = plan0.unpad(nxt[q]).cpu().numpy()[nid]      # permuted ids -> original ids
        ok, ratio = orc.spmv_check(got, yref, absy, 1e-12)
        assert ok, (world, q, ratio)
