"""Out-of-distribution check of the Seer trio: leave-one-FAMILY-out over the B200-measured
corpus (PAPER.md:330 evaluates on all of SuiteSparse; our corpus is 7 generator
families, so held-out families are the closest stand-in for unseen structure).  For each
family F: train with the frozen bundle's hyper-parameters on every other family, realise
the selector's cost on F and compare it with the best fixed kernel of F,
the oracle, and the frozen bundle (which saw 80 % of F) on the same rows.

    python tools/lofo_seer.py [--corpus DIR] [--out profiles/seer_lofo_r02.json]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from train_seer import ITERS, load  # noqa: E402

from paper_2403_17017_b200 import kernels, seer  # noqa: E402


def family(name: str) -> str:
    return name.split("_", 1)[0]


def realise(model, rows, k):
    nk = len(kernels.KERNELS)
    sel = [seer.realized_cost(model, r, k)[0] for r in rows]
    fixed = []
    for K in range(nk):
        tot = 0.0
        for r in rows:
            c = r.cost(K, k)
            if not math.isfinite(c):  # fixed-kernel totals only: worst present kernel
                c = max(r.cost(j, k) for j in range(nk) if math.isfinite(r.cost(j, k)))
            tot += c
        fixed.append(tot)
    bf = min(range(nk), key=lambda K: fixed[K])
    orc = sum(min(r.cost(j, k) for j in range(nk)) for r in rows)
    per = math.exp(sum(math.log(r.cost(bf, k) / c) for r, c in zip(rows, sel)) / len(rows))
    return {"selector_total_s": sum(sel), "best_fixed": kernels.KERNELS[bf], "best_fixed_total_s": fixed[bf],
            "aggregate_vs_best_fixed": fixed[bf] / sum(sel), "per_matrix_geomean_vs_best_fixed": per,
            "oracle_total_s": orc, "selector_over_oracle": sum(sel) / orc,
            "geomean_vs_all_fixed": math.exp(sum(math.log(f / sum(sel)) for f in fixed) / nk)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--corpus", default=os.path.join(ROOT, "paper_2403_17017_b200", "models", "corpus"))
    ap.add_argument("--bundle", default=os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json"))
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = load(a.corpus)
    frozen = seer.SeerModel.load(a.bundle)
    meta = frozen.meta
    fams = sorted({family(r.name) for r in rows})
    out = {"hyper_parameters": {k: meta.get(k) for k in ("max_depth", "gathered_depth", "min_samples_leaf", "weighting",
                                                         "selector_folds", "iterations")},
           "families": {}}
    for f in fams:
        held = [r for r in rows if family(r.name) == f]
        train = [r for r in rows if family(r.name) != f]
        m = seer.train_seer(train, ITERS, meta.get("max_depth", 5), meta.get("min_samples_leaf", 16),
                            kernels.KERNELS, weighting=meta.get("weighting", "cost-mix"),
                            selector_folds=meta.get("selector_folds", 0), gathered_depth=meta.get("gathered_depth"))
        res = {"n_held_out": len(held), "n_train": len(train), "k": {}}
        for k in ITERS:
            lofo, fr = realise(m, held, k), realise(frozen, held, k)
            res["k"][str(k)] = {"lofo": lofo, "frozen_bundle": fr}
            print(f"{f:9s} k={k:3d}  LOFO agg {lofo['aggregate_vs_best_fixed']:.3f} per {lofo['per_matrix_geomean_vs_best_fixed']:.3f}"
                  f" /oracle {lofo['selector_over_oracle']:.3f} (best fixed {lofo['best_fixed']}) | frozen agg "
                  f"{fr['aggregate_vs_best_fixed']:.3f} per {fr['per_matrix_geomean_vs_best_fixed']:.3f} "
                  f"/oracle {fr['selector_over_oracle']:.3f}", flush=True)
        out["families"][f] = res
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
