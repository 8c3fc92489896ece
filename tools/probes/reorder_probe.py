"""Probe (next-step evidence, not a product path): how much would a symmetric reordering of
C5 by column popularity (hottest vertices first, rows permuted the same way so x and y keep
one index space) help the row-sharded SpMV?  Times the unblocked CSR,WO SpMV and the
column-blocked ShardedSeer iteration (world 1) on the original and the reordered matrix.

    python tools/probes/reorder_probe.py
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import dist as kdist  # noqa: E402
from paper_2403_17017_b200 import gen, kernels  # noqa: E402


def timeit(fn, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def reorder(off, col, val, n):
    """P A P^T with P = columns by descending in-degree (ties by index)."""
    deg = torch.bincount(col.to(torch.int64), minlength=n)
    order = torch.argsort(-deg, stable=True)            # new position -> old id
    newid = torch.empty_like(order)
    newid[order] = torch.arange(n, device=order.device)  # old id -> new position
    ln = (off[1:] - off[:-1]).to(torch.int64)
    ln_new = ln[order]
    off_new = torch.zeros(n + 1, dtype=torch.int64, device=off.device)
    torch.cumsum(ln_new, 0, out=off_new[1:])
    # source index of every new entry: old row start + position inside the row
    row_of = torch.repeat_interleave(torch.arange(n, device=off.device), ln_new)
    pos = torch.arange(int(off_new[-1]), device=off.device) - off_new[row_of]
    src = off[order][row_of].to(torch.int64) + pos
    del row_of, pos
    c = newid[col[src].to(torch.int64)].to(torch.int32)
    v = val[src]
    del src
    # keep rows canonical (sorted columns) -- not needed by the kernels, kept for the oracle
    return off_new, c, v


def run(label, off, col, val, n):
    A, plan, _ = kdist.shard_device(off, col, val, n, 0, 1, torch.float32)
    x = torch.rand(n, device="cuda")
    y = torch.empty(n, device="cuda")
    t_un = timeit(lambda: kernels.spmv(A, x, kernels.CSR_WO, y=y))
    r = kdist.ShardedSeer(None, A, plan, 1, n, n, A.nnz, exchange="nccl", kernel=kernels.CSR_WO)
    Ps = r.prepare()
    t_bl = timeit(lambda: r.spmv_into(x, [y], 0, Ps))
    print(f"{label:10s} unblocked {t_un:7.3f} ms   column-blocked (S = {r.col_slices}) {t_bl:7.3f} ms", flush=True)
    del A, r, Ps
    torch.cuda.empty_cache()


def main():
    m = gen.config("C5", device="cuda")
    n = m.n_rows
    off, col, val = m.row_offsets, m.col_indices, m.values
    del m
    run("original", off, col, val, n)
    o2, c2, v2 = reorder(off, col, val, n)
    del off, col, val
    torch.cuda.empty_cache()
    run("reordered", o2, c2, v2, n)


if __name__ == "__main__":
    main()
