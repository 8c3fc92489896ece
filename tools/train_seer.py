"""Train the Seer trio on the B200-measured corpus and freeze the bundle (host, offline).

    python tools/train_seer.py --corpus paper_2403_17017_b200/models/corpus \
        --out paper_2403_17017_b200/models/seer_b200.json [--report profiles/seer_eval_r01.json]

SPEC.md:358-362: labels = fastest_kernel(total_cost) per (matrix, iterations); known tree on
(rows, cols, nnz, k), gathered tree on that + (max, min, mean, var) density, selector on the
sub-models' own predictions.  Split 80/20 under a fixed seed; the report
has train/test accuracies and the realised-cost comparison of SPEC.md:482-496 (selector vs
oracle, vs every fixed kernel, geomean and best-fixed-aggregate speedups).
"""

from __future__ import annotations

import argparse
import csv
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2403_17017_b200 import dataset, kernels, seer  # noqa: E402

ITERS = (1, 3, 10, 30, 100)


def load(corpus):
    known = {r["name"]: (int(r["rows"]), int(r["cols"]), int(r["nnz"]))
             for r in csv.DictReader(open(os.path.join(corpus, "known.csv")))}
    rd = lambda f: open(os.path.join(corpus, f)).read()  # noqa: E731
    return dataset.read_tables(rd("elapsed.csv"), rd("preprocess.csv"), rd("metadata.csv"), known)


def accuracy(model, rows, k):
    acc = {"known": 0, "gathered": 0, "selector": 0}
    for r in rows:
        lab = dataset.fastest_kernel(r.timings(), k)
        kv = seer.known_vector(*r.known, k)
        acc["known"] += model.known_tree.predict(kv) == lab
        acc["gathered"] += model.gathered_tree.predict(kv + tuple(r.gathered)) == lab
        acc["selector"] += seer.realized_cost(model, r, k)[1] == lab
    return {n: v / len(rows) for n, v in acc.items()}


def evaluate(model, rows, iters):
    out = {}
    for k in iters:
        g = seer.geomean_speedup(rows, model, k)
        sel = g["selector_total"]
        always_known = sum(r.cost(model.known_tree.predict(seer.known_vector(*r.known, k)), k) for r in rows)
        always_gath = sum(r.cost(model.gathered_tree.predict(seer.known_vector(*r.known, k) + tuple(r.gathered)), k)
                          + r.collection_time for r in rows)
        # per-matrix geomean vs the best-overall fixed kernel (north star)
        best_fixed = min(range(len(model.kernels)), key=lambda K: g["fixed_totals"][K])
        per = [r.cost(best_fixed, k) / seer.realized_cost(model, r, k)[0] for r in rows]
        out[str(k)] = {
            "accuracy": accuracy(model, rows, k),
            "selector_total_s": sel, "oracle_total_s": g["oracle_total"],
            "always_known_total_s": always_known, "always_gathered_total_s": always_gath,
            "best_fixed_kernel": kernels.KERNELS[best_fixed],
            "aggregate_speedup_vs_best_fixed": g["vs_best_fixed"],
            "geomean_speedup_vs_all_fixed": g["geomean_vs_fixed"],
            "per_matrix_geomean_vs_best_fixed": math.exp(sum(math.log(v) for v in per) / len(per)),
            "selector_within_oracle": sel / g["oracle_total"],
        }
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--corpus", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--report", default=None)
    ap.add_argument("--max-depth", type=int, default=5)
    ap.add_argument("--gathered-depth", type=int, default=0, help="gathered-tree depth (0 = --max-depth)")
    ap.add_argument("--min-leaf", type=int, default=4,
                    help="min training examples per leaf (tools/cv_seer.py: 4 is robust, 1 overfits)")
    ap.add_argument("--seed", type=int, default=2403)
    ap.add_argument("--weighting", default="cost-mix", choices=["none", "regret", "cost-log", "cost-rel", "cost-mix"])
    ap.add_argument("--near-best", type=float, default=0.0, help="relabel within this fraction of the best")
    ap.add_argument("--plots", default=None, help="emit SPEC eval plot data (CSV + SVG, test split) here")
    ap.add_argument("--selector-folds", type=int, default=0,
                    help="out-of-fold sub-model predictions for the selector's labels (0 = in-sample)")
    a = ap.parse_args()
    rows = load(a.corpus)
    train, test = dataset.split_train_test(rows, a.seed, 0.8)
    model = seer.train_seer(train, ITERS, a.max_depth, a.min_leaf, kernels.KERNELS,
                            {"source": "B200-measured corpus (tools/collect_corpus.py)", "corpus": os.path.relpath(a.corpus, ROOT),
                             "iterations": list(ITERS), "max_depth": a.max_depth, "min_samples_leaf": a.min_leaf,
                             "split_seed": a.seed,
                             "n_train": len(train), "n_test": len(test), "near_best": a.near_best,
                             "selector_folds": a.selector_folds, "gathered_depth": a.gathered_depth or a.max_depth},
                            weighting=a.weighting, near_best=a.near_best, selector_folds=a.selector_folds,
                            gathered_depth=a.gathered_depth or None)
    model.save(a.out)
    plain = seer.train_seer(train, ITERS, a.max_depth, 1, kernels.KERNELS, weighting="none")
    rep = {"weighting": a.weighting, "n_train": len(train), "n_test": len(test),
           "spec_plain_cart_test": evaluate(plain, test, ITERS), "train": evaluate(model, train, ITERS),
           "test": evaluate(model, test, ITERS), "all": evaluate(model, rows, ITERS),
           "tree_nodes": {"known": model.known_tree.n_nodes, "gathered": model.gathered_tree.n_nodes,
                          "selector": model.selector_tree.n_nodes}}
    from paper_2403_17017_b200 import evaluate as ev
    rep["eval_report_test"] = {}
    for k in ITERS:
        er = ev.evaluate(model, test, k)
        rep["eval_report_test"][str(k)] = {
            name: {"total_realized_cost_s": p.total_realized_cost, "accuracy": p.accuracy,
                   "error_vs_oracle_s": p.error_vs_oracle} for name, p in er.predictors.items()}
        rep["eval_report_test"][str(k)]["geomean_speedup"] = ev.geomean_speedup(er)
        if a.plots:
            ev.emit_plot_data(er, a.plots, per_matrix=False)
    if a.report:
        with open(a.report, "w") as f:
            json.dump(rep, f, indent=1)
    for split in ("train", "test"):
        for k in ITERS:
            e = rep[split][str(k)]
            print(f"{split:5s} k={k:3d} acc known/gath/sel = {e['accuracy']['known']:.2f}/{e['accuracy']['gathered']:.2f}/"
                  f"{e['accuracy']['selector']:.2f}  agg vs best fixed ({e['best_fixed_kernel']}) "
                  f"{e['aggregate_speedup_vs_best_fixed']:.2f}x  geomean vs all fixed {e['geomean_speedup_vs_all_fixed']:.2f}x"
                  f"  per-matrix vs best fixed {e['per_matrix_geomean_vs_best_fixed']:.2f}x  sel/oracle {e['selector_within_oracle']:.3f}")


if __name__ == "__main__":
    main()
