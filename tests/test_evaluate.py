"""SPEC eval module: examples and invariants on hand-built and corpus rows."""
import os

import numpy as np
import pytest

from paper_2403_17017_b200 import dataset, evaluate, seer
from paper_2403_17017_b200.dtree import leaf_tree

K2 = ("A", "B")


def _model(known_kernel=0, gathered_kernel=1, path=seer.USE_KNOWN, kernels=K2):
    nk = len(kernels)
    return seer.SeerModel(leaf_tree(known_kernel, nk, 4), leaf_tree(gathered_kernel, nk, 8), leaf_tree(path, 2, 4),
                          kernels, {})


def _row(name, a, b, coll=0.0):
    return dataset.DatasetRow(name, (10, 10, 50), (0.1, 0.0, 0.05, 0.001), coll, [a, b], [0.0, 0.0])


def test_oracle_self_comparison():
    rows = [_row("m%d" % i, 1.0 + i, 2.0) for i in range(4)]
    rep = evaluate.evaluate(_model(), rows, 1)
    o = rep.predictors["oracle"]
    assert o.accuracy == 1.0 and o.error_vs_oracle == 0.0
    for name, p in rep.predictors.items():  # oracle dominance
        assert p.total_realized_cost >= o.total_realized_cost
        assert p.total_realized_cost == pytest.approx(sum(x[3] for x in p.rows), rel=0, abs=0)


def test_geomean_two_baselines_2x_8x():
    # selector total 1; fixed totals 2 and 8 -> sqrt(16) = 4
    rows = [_row("m", 2.0, 8.0, coll=0.0)]
    m = _model(known_kernel=0)
    rep = evaluate.evaluate(m, rows, 1)
    rep.predictors["selector"].total_realized_cost = 1.0
    assert evaluate.geomean_speedup(rep) == pytest.approx(4.0)


def test_accuracy_error_decoupling():
    """A predictor can be more accurate yet worse: 'A' wins 9 rows by 1 %
    and loses one by 100x; 'B' is 1 % off on those 9 and right on the last."""
    rows = [_row("w%d" % i, 1.0, 1.01) for i in range(9)] + [_row("loss", 100.0, 1.0)]
    rep = evaluate.evaluate(_model(), rows, 1)
    A, B = rep.predictors["A"], rep.predictors["B"]
    assert A.accuracy > B.accuracy
    assert A.error_vs_oracle > B.error_vs_oracle


def test_gathered_overhead_charged_and_plots(tmp_path):
    rows = [_row("m%d" % i, 1.0, 2.0, coll=0.25) for i in range(3)]
    rep = evaluate.evaluate(_model(path=seer.USE_GATHERED, gathered_kernel=0), rows, 1)
    assert rep.predictors["selector"].total_realized_cost == pytest.approx(3 * 1.25)
    assert rep.predictors["known"].rows[0][2] == 0.0  # known path: zero-height overhead
    files = evaluate.emit_plot_data(rep, str(tmp_path))
    agg = open(os.path.join(tmp_path, "single_iteration", "aggregate.csv")).read().splitlines()
    assert len(agg) == 1 + len(K2) + 4  # bars = |kernels| + 4 predictors
    # aggregate == column sums of the per-matrix files
    per = [open(os.path.join(tmp_path, "single_iteration", f"m{i}.csv")).read().splitlines()[1:] for i in range(3)]
    import csv
    aggr = list(csv.reader(agg))[1:]
    perr = [list(csv.reader(p)) for p in per]
    for j, (name, rt, ov) in enumerate(aggr):
        assert float(rt) == pytest.approx(sum(float(p[j][1]) for p in perr))
        assert float(ov) == pytest.approx(sum(float(p[j][2]) for p in perr))
    again = evaluate.emit_plot_data(rep, str(tmp_path / "b"))
    for f1, f2 in zip(files, again):  # deterministic bytes
        assert open(f1, "rb").read() == open(f2, "rb").read()


def test_corpus_report_runs():
    import csv
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2403_17017_b200",
                        "models")
    c = os.path.join(root, "corpus")
    known = {r["name"]: (int(r["rows"]), int(r["cols"]), int(r["nnz"])) for r in csv.DictReader(open(os.path.join(c, "known.csv")))}
    rd = lambda f: open(os.path.join(c, f)).read()  # noqa: E731
    rows = dataset.read_tables(rd("elapsed.csv"), rd("preprocess.csv"), rd("metadata.csv"), known)
    model = seer.SeerModel.load(os.path.join(root, "seer_b200.json"))
    _, test = dataset.split_train_test(rows, 2403, 0.8)
    for k in (1, 100):
        rep = evaluate.evaluate(model, test, k)
        assert rep.predictors["oracle"].accuracy == 1.0
        assert np.isfinite(evaluate.geomean_speedup(rep))
        assert rep.predictors["selector"].total_realized_cost >= rep.predictors["oracle"].total_realized_cost
