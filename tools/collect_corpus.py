"""Measure every kernel on a synthetic B200 corpus -> Seer training data (GPU).

    python tools/collect_corpus.py --out DIR [--quick]

Writes the SPEC.md:246 artifact files into DIR:
  elapsed.csv     name + one column per kernel: seconds per SpMV iteration -- by default the
                  marginal cost of one more iteration inside a plan-like graph (--timing graph)
  preprocess.csv  name + one column per kernel: seconds of one-time cost -- preprocessing plus
                  the body's fixed launch cost (graph 1-iteration time minus one iteration)
  metadata.csv    name, max/min/mean/var density, collection_time = the realised overhead of
                  the gathered path in the Seer plan (forced-gathered plan minus the same body
                  as a plain graph: feature pass + tree + device SWITCH), or with --model ''
                  the bare kp_gather_features time
  known.csv       name, rows, cols, nnz
Times are CUDA-event device times on the launching stream (PAPER.md:331 uses 10 warm-ups +
mean of 10; we use 2 warm-ups + median of 5, enough for ranking).  A kernel slower than
--cap-ms on its first run is recorded from that run only.
"""

from __future__ import annotations

import argparse
import csv
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2403_17017_b200 import features, gen, kernels  # noqa: E402


STRUCTURED = ("fem", "circuit", "road")


def corpus(quick: bool, extra: int = 400, extra_structured: int = 60):
    C = []
    for R in (10_000, 100_000, 1_000_000, 4_000_000):
        for per in (2, 8, 32):
            if R * per <= 64_000_000:
                C.append(("uniform", dict(n_rows=R, n_cols=R, n_pairs=R * per, seed=R + per)))
    for R in (100_000, 1_000_000, 8_000_000):
        for ln in (1, 3, 8, 24, 64):
            if R * ln <= 128_000_000:
                C.append(("const", dict(n_rows=R, length=ln, seed=ln)))
    for R in (100_000, 1_000_000, 8_000_000):
        for w in (3, 7, 27, 100):
            if R * w <= 220_000_000:
                C.append(("band", dict(n_rows=R, width=w)))
    C += [("band", dict(n_rows=65_536, width=1024)), ("band", dict(n_rows=65_536, width=2048)),
          ("band", dict(n_rows=8_192, width=8_192))]
    for n in (20, 50, 100, 159):
        C.append(("stencil", dict(n=n)))
    for R in (100_000, 1_000_000, 4_000_000):
        for mean in (4.0, 16.0, 64.0):
            for alpha in (1.2, 1.5, 2.5):
                if R * mean <= 128_000_000:
                    C.append(("powerlaw", dict(n_rows=R, mean=mean, alpha=alpha, seed=int(mean * 10 + alpha * 100))))
    for scale in (12, 14, 16, 18, 20, 22):
        for ef in (4, 16):
            if (1 << scale) * ef <= 80_000_000:
                C.append(("rmat", dict(scale=scale, edge_factor=ef, seed=scale * 7 + ef)))
    for R in (200_000, 2_000_000):
        for nd in (1, 4, 16):
            for dl in (10_000, 100_000, 1_000_000):
                if dl <= R:
                    C.append(("skewed", dict(n_rows=R, n_dense=nd, dense_len=dl, seed=nd + dl % 97)))
    # seeded random draws per family (log-uniform sizes) for coverage between the grid points
    import numpy as np
    rng = np.random.default_rng(20240317)
    lu = lambda lo, hi: float(np.exp(rng.uniform(np.log(lo), np.log(hi))))  # noqa: E731
    for i in range(extra):
        fam = ["uniform", "const", "band", "powerlaw", "rmat", "skewed", "stencil"][i % 7]
        sd = 1000 + i
        if fam == "uniform":
            R = int(lu(5e3, 6e6)); per = lu(1, 64)
            if R * per > 1.2e8: per = 1.2e8 / R
            C.append(("uniform", dict(n_rows=R, n_cols=int(R * lu(0.2, 5)), n_pairs=int(R * per), seed=sd)))
        elif fam == "const":
            R = int(lu(5e3, 8e6)); ln = max(1, int(lu(1, 128)))
            if R * ln > 1.2e8: ln = max(1, int(1.2e8 / R))
            C.append(("const", dict(n_rows=R, length=ln, seed=sd)))
        elif fam == "band":
            R = int(lu(5e3, 8e6)); w = max(1, int(lu(1, 512)))
            if R * w > 1.5e8: w = max(1, int(1.5e8 / R))
            C.append(("band", dict(n_rows=R, width=w)))
        elif fam == "powerlaw":
            R = int(lu(5e3, 6e6)); mean = lu(2, 128); al = float(rng.uniform(1.1, 3.0))
            if R * mean > 1.2e8: mean = 1.2e8 / R
            C.append(("powerlaw", dict(n_rows=R, mean=round(mean, 2), alpha=round(al, 2), seed=sd)))
        elif fam == "rmat":
            sc = int(rng.integers(11, 22)); ef = int(rng.choice([2, 4, 8, 16, 32]))
            if (1 << sc) * ef > 8e7: ef = max(1, int(8e7 / (1 << sc)))
            C.append(("rmat", dict(scale=sc, edge_factor=ef, seed=sd)))
        elif fam == "skewed":
            R = int(lu(5e4, 4e6)); nd = int(rng.integers(1, 32)); dl = int(min(R, lu(1e3, 2e6)))
            C.append(("skewed", dict(n_rows=R, n_dense=nd, dense_len=dl, seed=sd)))
        else:
            C.append(("stencil", dict(n=int(lu(8, 170)))))
    C += large_tier()
    C += structured(extra_structured)
    if quick:
        C = C[::6]
    uniq, seen = [], set()  # random draws can repeat a grid point (e.g. a stencil size)
    for fam, p in C:
        key = (fam, tuple(sorted(p.items())))
        if key not in seen:
            seen.add(key)
            uniq.append((fam, p))
    return uniq


def structured(extra: int = 60):
    """FEM meshes, circuits and road networks (gen.py): absent from the round-1 corpus, so
    the frozen bundle meets them out of distribution.  A grid plus `extra` seeded draws per
    family (its own RNG: the original families' draws are unchanged)."""
    import numpy as np
    C = []
    for n in (100, 300, 1000, 2000, 2800):
        for order in (1, 2):
            C.append(("fem", dict(n=n, order=order, seed=n + order)))
    for n in (10_000, 100_000, 1_000_000, 4_000_000):
        for rails in (2, 16):
            for frac in (0.01, 0.2):
                C.append(("circuit", dict(n=n, n_rails=rails, rail_frac=frac, seed=n % 97 + rails)))
    for side in (100, 300, 1000, 3000, 6000):
        for keep in (0.5, 0.8):
            C.append(("road", dict(side=side, keep=keep, seed=side + int(keep * 10))))
    rng = np.random.default_rng(20261017)
    lu = lambda lo, hi: float(np.exp(rng.uniform(np.log(lo), np.log(hi))))  # noqa: E731
    for i in range(extra):
        for fam in STRUCTURED:
            sd = 5000 + 3 * i + STRUCTURED.index(fam)
            if fam == "fem":
                order = int(rng.integers(1, 3))
                C.append(("fem", dict(n=int(lu(60, 2800 if order == 2 else 4000)), order=order, seed=sd)))
            elif fam == "circuit":
                C.append(("circuit", dict(n=int(lu(5e3, 6e6)), n_rails=int(rng.integers(1, 33)),
                                          rail_frac=round(lu(0.002, 0.3), 4), seed=sd)))
            else:
                C.append(("road", dict(side=int(lu(80, 7000)), keep=round(float(rng.uniform(0.45, 0.9)), 3),
                                       seed=sd)))
    return C


def large_tier():
    """134M - 1.07B nnz (BASELINE C5 scale), so the trees do not extrapolate there."""
    C = [("rmat", dict(scale=sc, edge_factor=ef, seed=sc * 7 + ef))
         for sc, ef in ((23, 16), (24, 8), (24, 16), (25, 8), (25, 16), (26, 8), (26, 16))]
    C += [("uniform", dict(n_rows=32_000_000, n_cols=32_000_000, n_pairs=512_000_000, seed=77)),
          ("const", dict(n_rows=64_000_000, length=8, seed=78)),
          ("band", dict(n_rows=16_000_000, width=27)),
          ("band", dict(n_rows=64_000_000, width=7)),
          ("stencil", dict(n=280)),
          ("powerlaw", dict(n_rows=32_000_000, mean=16.0, alpha=1.5, seed=79)),
          ("skewed", dict(n_rows=16_000_000, n_dense=16, dense_len=4_000_000, seed=80))]
    return C


def build(fam, p, dev):
    if fam == "uniform":
        return gen.uniform_random(p["n_rows"], p["n_cols"], p["n_pairs"], p["seed"], device=dev)
    if fam == "const":
        return gen.constant_rows(p["n_rows"], p["length"], p["seed"], device=dev)
    if fam == "band":
        return gen.banded(p["n_rows"], p["width"], device=dev)
    if fam == "stencil":
        return gen.stencil27(p["n"], device=dev)
    if fam == "powerlaw":
        return gen.powerlaw_rows(p["n_rows"], p["mean"], p["alpha"], p["seed"], device=dev)
    if fam == "rmat":
        return gen.rmat(p["scale"], p["edge_factor"], seed=p["seed"], device=dev)
    if fam == "skewed":
        return gen.skewed(p["n_rows"], 8.0, p["n_dense"], p["dense_len"], p["seed"], device=dev)
    if fam == "fem":
        return gen.fem_mesh(p["n"], p["order"], seed=p["seed"], device=dev)
    if fam == "circuit":
        return gen.circuit(p["n"], p["n_rails"], p["rail_frac"], seed=p["seed"], device=dev)
    if fam == "road":
        return gen.road(p["side"], p["keep"], seed=p["seed"], device=dev)
    raise ValueError(fam)


def _plan_overhead(model, A, x, y, flush, ev, reps: int = 5):
    """Realised cost of the gathered path inside the Seer plan: time of a plan forced onto
    the gathered path (K1 feature pass + gathered tree + device SWITCH) minus the time of
    the same chosen body (prep + 1 SpMV) as a plain graph.  This, not the bare feature
    kernel, is what the selector must weigh against the known path."""
    from paper_2403_17017_b200 import seer
    plan = seer.SeerPlan(model, A, x, y, 1, force_gathered=True)
    plan.launch()
    torch.cuda.synchronize()
    kern = int(plan.outcome().kernel)

    def med(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = ev(), ev()
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        return statistics.median(ts)

    t_plan = med(plan.launch)
    plan.close()
    # the same body as a constant-model plan: same graph construction and launch
    body = seer.SeerPlan(seer.fixed_model(kern), A, x, y, 1)
    t_body = med(body.launch)
    body.close()
    return max(t_plan - t_body, 1e-6)


def _eager_costs(A, x, y, k, flush, ev, reps, cap_ms):
    """(runtime, preprocess) from single eager launches: one L2-flushed SpMV per sample."""
    P, tprep = None, 0.0
    if k in kernels.NEEDS_PREP:
        ts = []
        for _ in range(3):
            e0, e1 = ev(), ev()
            e0.record()
            P = kernels.prepare(A, k, cache=False)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        tprep = min(ts[1:])  # first call may include a cudaMalloc
    ts = []
    for r in range(reps + 1):
        flush.zero_()
        e0, e1 = ev(), ev()
        e0.record()
        kernels.spmv(A, x, k, y=y, prepared=P)
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) * 1e-3
        if r > 0 or t * 1e3 > cap_ms:
            ts.append(t)
        if t * 1e3 > cap_ms:
            break
    if not ts:  # reps = 0 and under the cap: the one run is the sample
        ts.append(t)
    return statistics.median(ts), tprep


def _graph_costs(A, x, y, k, flush, ev, reps, cap_ms):
    """(runtime, preprocess) as the Seer plan realises them: the kernel's prep + n SpMVs as
    ONE graph -- a constant-model kp_seer_plan, i.e. exactly the Seer plan's body --, L2
    flushed before each launch.  runtime = the marginal cost of one more
    iteration, (t_n - t_1) / (n - 1) -- later iterations find a matrix that fits in L2
    warm, as a real iterative run does; preprocess = t_1 - runtime, so prep + k x runtime
    reproduces the measured 1-iteration graph exactly and the n-iteration one by
    construction.  Kernels slower than cap_ms fall back to the eager figures."""
    def body(n):
        P = kernels.prepare(A, k, cache=False) if k in kernels.NEEDS_PREP else None
        for _ in range(n):
            kernels.spmv(A, x, k, y=y, prepared=P)

    body(1)  # first use: attributes, workspaces, allocations
    torch.cuda.synchronize()
    # the cap check on a WARM eager run (the first one pays allocations: a 64 M-row ELL
    # layout took > 40 ms cold and its eager preparation then landed in the corpus as 36 ms)
    t_warm = []
    for _ in range(2):
        e0, e1 = ev(), ev()
        flush.zero_()
        e0.record()
        body(1)
        e1.record()
        e1.synchronize()
        t_warm.append(e0.elapsed_time(e1))
    if min(t_warm) > cap_ms:
        return _eager_costs(A, x, y, k, flush, ev, 0, cap_ms)

    def graph_time(n):
        # prep + n SpMVs as a constant-model Seer plan: the graph the Seer plan's body is,
        # built and launched the same way (a torch-captured graph of the same calls runs
        # ~1-2 us slower per launch, tools/graph_launch_probe.py)
        from paper_2403_17017_b200 import seer
        plan = seer.SeerPlan(seer.fixed_model(k), A, x, y, n)
        plan.launch()
        torch.cuda.synchronize()
        ts = []
        nrep, i = reps, 0
        while i < nrep:
            flush.zero_()
            a0, a1 = ev(), ev()
            a0.record()
            plan.launch()
            a1.record()
            a1.synchronize()
            ts.append(a0.elapsed_time(a1) * 1e-3)
            if i == 0 and ts[0] < 1e-4:  # a few ~2 us timer ticks: mean of >= 2 ms of samples
                nrep = max(reps, min(100, int(2e-3 / max(ts[0], 1e-6))))
            i += 1
        plan.close()
        return statistics.mean(ts) if nrep > reps else statistics.median(ts)

    t1 = graph_time(1)
    n = 10 if t1 < 2e-3 else 3
    tn = graph_time(n)
    run = max((tn - t1) / (n - 1), 1e-7)
    return run, max(t1 - run, 0.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--extra", type=int, default=400, help="seeded random draws on top of the grid")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cap-ms", type=float, default=40.0)
    ap.add_argument("--timing", default="graph", choices=["graph", "eager"],
                    help="graph: marginal per-iteration cost inside a plan-like graph (default); "
                         "eager: one L2-flushed launch per SpMV")
    ap.add_argument("--only-large", action="store_true", help="only the large tier (append to a corpus)")
    ap.add_argument("--families", default=None, help="comma list: collect only these families")
    ap.add_argument("--shard", default="0/1", help="i/n: every n-th matrix from the i-th (split runs)")
    ap.add_argument("--extra-structured", type=int, default=60)
    ap.add_argument("--model", default=os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json"),
                    help="bundle whose gathered tree drives the plan-overhead measurement ('' = bare K1 time)")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    rows_el, rows_pp, rows_md, rows_kn = [], [], [], []
    model = None
    if a.model and os.path.exists(a.model):
        from paper_2403_17017_b200 import seer
        model = seer.SeerModel.load(a.model)
    t_start = time.time()
    todo = large_tier() if a.only_large else corpus(a.quick, a.extra, a.extra_structured)
    if a.families:
        todo = [(f, p) for f, p in todo if f in a.families.split(",")]
    si, sn = (int(v) for v in a.shard.split("/"))
    todo = todo[si::sn]
    print(f"{len(todo)} matrices", flush=True)
    for fam, p in todo:
        m = build(fam, p, dev)
        name = fam + "_" + "_".join(f"{k}{v}" for k, v in p.items())
        A = m.to_device_csr(torch.float32, device=dev)
        del m
        x = (torch.rand(A.n_cols, device=dev, dtype=torch.float64) * 2 - 1).float()
        y = torch.empty(A.n_rows, device=dev, dtype=torch.float32)
        # gathered features + device collection time
        for _ in range(2):
            buf = features.gather_outcome(A)
        cts = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = ev(), ev()
            e0.record()
            buf = features.gather_outcome(A, out=buf)
            e1.record()
            e1.synchronize()
            cts.append(e0.elapsed_time(e1) * 1e-3)
        o = features.decode_outcome(buf)
        coll = statistics.median(cts)
        if model is not None:
            coll = _plan_overhead(model, A, x, y, flush, ev) or coll
        rows_md.append([name, o.max_d, o.min_d, o.mean_d, o.var_d, coll])
        rows_kn.append([name, A.n_rows, A.n_cols, A.nnz])
        el, pp = [], []
        for k in range(len(kernels.KERNELS)):
            try:
                if a.timing == "graph":
                    tr, tp = _graph_costs(A, x, y, k, flush, ev, a.reps, a.cap_ms)
                else:
                    tr, tp = _eager_costs(A, x, y, k, flush, ev, a.reps, a.cap_ms)
                el.append(tr)
                pp.append(tp)
            except Exception as exc:  # record as missing (+inf cost)
                print(f"  {name} {kernels.KERNELS[k]} failed: {exc}", flush=True)
                el.append(None)
                pp.append(None)
        rows_el.append([name, *el])
        rows_pp.append([name, *pp])
        best = min(range(8), key=lambda i: el[i] if el[i] is not None else 1e9)
        print(f"{name:55s} R={A.n_rows:9d} nnz={A.nnz:11d} best={kernels.KERNELS[best]:13s} "
              f"{el[best] * 1e6:9.1f} us  coll={statistics.median(cts) * 1e6:6.1f} us  [{time.time() - t_start:5.0f}s]",
              flush=True)
        del A, x, y
        torch.cuda.empty_cache()

    def dump(fn, head, rows):
        with open(os.path.join(a.out, fn), "w", newline="") as f:
            w = csv.writer(f, lineterminator="\n")
            w.writerow(head)
            for r in rows:
                w.writerow(["" if v is None else (repr(float(v)) if isinstance(v, float) else v) for v in r])

    labels = list(kernels.KERNELS)
    dump("elapsed.csv", ["name", *labels], rows_el)
    dump("preprocess.csv", ["name", *labels], rows_pp)
    dump("metadata.csv", ["name", "max_density", "min_density", "mean_density", "var_density", "collection_time"],
         rows_md)
    dump("known.csv", ["name", "rows", "cols", "nnz"], rows_kn)
    print(f"wrote {len(rows_el)} matrices to {a.out}")


if __name__ == "__main__":
    main()
