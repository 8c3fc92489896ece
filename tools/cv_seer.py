"""Hyper-parameter choice for the Seer trio by 5-fold cross-validation on the TRAINING split
only (the held-out test split is never looked at): for each (max_depth, min_samples_leaf,
selector_folds) train on 4 folds, realise the selector's cost on the 5th, and report per
iteration count the aggregate speed-up vs the best fixed kernel and the per-matrix geomean.

    python tools/cv_seer.py --corpus paper_2403_17017_b200/models/corpus
"""
import argparse
import itertools
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from train_seer import ITERS, load  # noqa: E402

from paper_2403_17017_b200 import dataset, kernels, seer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--corpus", required=True)
    ap.add_argument("--seed", type=int, default=2403)
    ap.add_argument("--folds", type=int, default=5)
    ap.add_argument("--depths", default="4,5,6")
    ap.add_argument("--leaves", default="1,4")
    ap.add_argument("--selector-folds", default="0,5")
    ap.add_argument("--gathered-depths", default="0", help="gathered-tree depths (0 = same as --depths)")
    a = ap.parse_args()
    rows = load(a.corpus)
    train, _ = dataset.split_train_test(rows, a.seed, 0.8)
    names = sorted(r.name for r in train)
    fold = {n: i % a.folds for i, n in enumerate(names)}
    nk = len(kernels.KERNELS)
    grid = itertools.product([int(v) for v in a.depths.split(",")], [int(v) for v in a.leaves.split(",")],
                             [int(v) for v in a.selector_folds.split(",")], [int(v) for v in a.gathered_depths.split(",")])
    for depth, leaf, sf, gdep in grid:
        sel = {k: 0.0 for k in ITERS}
        fixed = {k: [0.0] * nk for k in ITERS}
        real = {k: [] for k in ITERS}
        for f in range(a.folds):
            tr = [r for r in train if fold[r.name] != f]
            te = [r for r in train if fold[r.name] == f]
            m = seer.train_seer(tr, ITERS, depth, leaf, kernels.KERNELS, weighting="cost-mix", selector_folds=sf,
                                gathered_depth=gdep or None)
            for k in ITERS:
                for r in te:
                    c = seer.realized_cost(m, r, k)[0]
                    sel[k] += c
                    real[k].append((r, c))
                    for K in range(nk):
                        cc = r.cost(K, k)
                        if not math.isfinite(cc):
                            cc = max(r.cost(j, k) for j in range(nk) if math.isfinite(r.cost(j, k)))
                        fixed[k][K] += cc
        out = []
        for k in ITERS:
            bf = min(range(nk), key=lambda K: fixed[k][K])
            per = math.exp(sum(math.log(r.cost(bf, k) / c) for r, c in real[k]) / len(real[k]))
            out.append(f"k{k}: agg {fixed[k][bf] / sel[k]:.3f} per-matrix {per:.3f}")
        print(f"depth {depth} gathered_depth {gdep or depth} leaf {leaf} selector_folds {sf}  " + "  ".join(out), flush=True)


if __name__ == "__main__":
    main()
