"""Strong-scaling projection of the row-sharded C5 SpMV on ONE GPU (this round has 1 GPU):
for P = 1, 2, 4, 8 the matrix is cut exactly as `dist.shard_device` cuts it for P ranks,
and every rank's local SpMV (the chosen kernel, rank-padded x) is timed in turn; the
step time of P GPUs is bounded below by the slowest rank.  Each rank's SpMV runs as
dist.ShardedSeer runs it (column blocks when its x exceeds the L2 budget; --col-slices
lists the settings to time, the last one is the headline).  Reports per-P max / mean rank
time, the compute-only speedup t(1) / max_p t_p(P), and the bytes each rank must push per
iteration in the y exchange (fused into the SpMV epilogue over NVLink, kp_spmv_bcast).

    python tools/shard_scaling.py [--kernel CSR,WO] [--parts 1,2,4,8] [--out profiles/shard_scaling_r01.json]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import dist as kdist  # noqa: E402
from paper_2403_17017_b200 import gen, kernels  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="CSR,WO")
    ap.add_argument("--parts", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--bcast", action="store_true", help="only measure the fused-exchange epilogue cost")
    ap.add_argument("--no-reorder", action="store_true", help="keep the generator's vertex numbering")
    ap.add_argument("--col-slices", default="1,auto",
                    help="column blocking of each rank's SpMV (dist.ShardedSeer col_slices), comma list")
    a = ap.parse_args()
    if a.bcast:
        bcast_overhead()
        return
    kern = kernels.kernel_index(a.kernel)
    m = gen.config("C5", device="cuda")
    R, C, Z = m.n_rows, m.n_cols, m.nnz
    if not a.no_reorder:  # as bench.py's C5 does at distribution time
        order, newid = kdist.degree_order(m.col_indices, C)
        m.row_offsets, m.col_indices, m.values = kdist.permute_symmetric(m.row_offsets, m.col_indices, m.values,
                                                                        order, newid)
        del order, newid
        torch.cuda.empty_cache()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    res = {"matrix": "C5 R-MAT s26 ef16", "rows": R, "nnz": Z, "kernel": a.kernel, "reordered": not a.no_reorder,
           "parts": {}}
    slices = a.col_slices.split(",")
    for P in [int(v) for v in a.parts.split(",")]:
        times = {S: [] for S in slices}
        nnzs, used = [], {}
        for rank in range(P):
            A, plan, _ = kdist.shard_device(m.row_offsets, m.col_indices, m.values, C, rank, P, torch.float32)
            x = torch.rand(P * plan.r_max, device="cuda", dtype=torch.float32)
            y = torch.empty(plan.local_rows, device="cuda", dtype=torch.float32)
            for S in slices:
                # the rank's local SpMV exactly as ShardedSeer runs it (column blocks and all)
                run = kdist.ShardedSeer(None, A, plan, 1, R, C, Z, exchange="nccl", kernel=kern, col_slices=S)
                used[S] = run.col_slices
                Ps = run.prepare()
                run.spmv_into(x, [y], 0, Ps)
                ts = []
                for _ in range(a.reps):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    run.spmv_into(x, [y], 0, Ps)
                    e1.record()
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e-3)
                times[S].append(statistics.median(ts))
                del run, Ps
            nnzs.append(A.nnz)
            del A, x, y
            torch.cuda.empty_cache()
        for S in slices:
            rec = {"col_slices": used[S], "max_rank_ms": max(times[S]) * 1e3,
                   "mean_rank_ms": statistics.mean(times[S]) * 1e3,
                   "rank_ms": [t * 1e3 for t in times[S]], "rank_nnz": nnzs,
                   "exchange_bytes_per_rank_per_iter": int(4 * (R // P) * (P - 1))}
            res["parts"][f"{P}" if S == slices[-1] else f"{P}/S={S}"] = rec
            print(P, S, json.dumps({k: v for k, v in rec.items() if k not in ("rank_ms", "rank_nnz")}), flush=True)
    t1 = res["parts"]["1"]["max_rank_ms"] if "1" in res["parts"] else None
    if t1:
        for P, rec in res["parts"].items():
            rec["compute_speedup_vs_1"] = t1 / rec["max_rank_ms"]
    print(json.dumps({P: round(r.get("compute_speedup_vs_1", 0), 2) for P, r in res["parts"].items()}))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)



def bcast_overhead(P: int = 8, reps: int = 5):
    """Cost of the fused exchange epilogue itself on one GPU: rank 0's shard at P ranks,
    kp_spmv vs kp_spmv_bcast writing its y slice into P distinct (local) next-x buffers."""
    m = gen.config("C5", device="cuda")
    A, plan, _ = kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, 0, P, torch.float32)
    del m
    torch.cuda.empty_cache()
    x = torch.rand(P * plan.r_max, device="cuda", dtype=torch.float32)
    nxt = [torch.empty(P * plan.r_max, device="cuda", dtype=torch.float32) for _ in range(P)]
    dests = [b[:plan.local_rows] for b in nxt]
    y = torch.empty(plan.local_rows, device="cuda", dtype=torch.float32)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    for name, fn in (("spmv", lambda: kernels.spmv(A, x, kernels.CSR_WO, y=y)),
                     (f"spmv_bcast_{P}_dests", lambda: kernels.spmv_bcast(A, x, kernels.CSR_WO, dests, 0))):
        fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name + "_ms"] = statistics.median(ts)
    print(json.dumps(out))
    return out


if __name__ == "__main__":
    main()
