"""SPEC dataset / seer-core host semantics."""
import math

import numpy as np
import pytest

from paper_2403_17017_b200 import dataset, seer
from paper_2403_17017_b200.dataset import DatasetRow
from paper_2403_17017_b200.dtree import leaf_tree
from paper_2403_17017_b200.features import GatheredFeatures


def test_total_cost_examples():
    assert dataset.total_cost(5, 0, 1) == 5
    assert dataset.total_cost(3, 10, 1) == 13 and dataset.total_cost(3, 10, 19) == 67
    assert dataset.total_cost(None, 0, 1) == math.inf


def test_fastest_kernel_examples():
    t = [(5, 0), (3, 10)]
    assert dataset.fastest_kernel(t, 1) == 0 and dataset.fastest_kernel(t, 19) == 1
    assert dataset.fastest_kernel([(2, 0)], 1) == 0
    assert dataset.fastest_kernel([(2, 0), (2, 0)], 1) == 0
    assert dataset.fastest_kernel([(None, None), (2, 0)], 1) == 1


def test_crossover_at_most_n_minus_1_changes():
    rng = np.random.default_rng(0)
    for _ in range(50):
        t = [(float(rng.uniform(1, 10)), float(rng.uniform(0, 100))) for _ in range(5)]
        seq = [dataset.fastest_kernel(t, k) for k in range(1, 200)]
        assert sum(a != b for a, b in zip(seq, seq[1:])) <= 4


def _row(rt, pp, coll=0.0, known=(100, 100, 1000), g=(0.1, 0.0, 0.05, 0.001)):
    return DatasetRow("m", known, g, coll, list(rt), list(pp))


def test_selector_label_examples():
    r = _row([5, 3], [0, 0], coll=1.0)
    assert seer.selector_label(r, 0, 1, 1) == seer.USE_GATHERED
    assert seer.selector_label(r, 1, 1, 1) == seer.USE_KNOWN
    r2 = _row([5, 3], [0, 0], coll=2.0)
    assert seer.selector_label(r2, 0, 1, 1) == seer.USE_KNOWN


def _model(selector_cls):
    kt = leaf_tree(3, 8, 4)
    gt = leaf_tree(5, 8, 8)
    return seer.SeerModel(kt, gt, leaf_tree(selector_cls, 2, 4))


def test_infer_features_examples():
    m = _model(seer.USE_KNOWN)
    o = seer.infer_features(m, (10, 10, 30), 1)
    assert (o.chosen_kernel, o.path, o.charged_overhead) == (3, seer.USE_KNOWN, 0.0)
    m2 = _model(seer.USE_GATHERED)
    g = GatheredFeatures(0.5, 0.1, 0.2, 0.01, 0.5)
    o2 = seer.infer_features(m2, (10, 10, 30), 1, g)
    assert (o2.chosen_kernel, o2.path, o2.charged_overhead) == (5, seer.USE_GATHERED, 0.5)
    with pytest.raises(ValueError):
        seer.infer_features(m2, (10, 10, 30), 1, None)


def test_train_seer_known_separable_and_bundle_roundtrip():
    rows = []
    for i in range(40):
        nnz = 100 * (i + 1)
        lab = 0 if nnz <= 2000 else 1
        rt = [1.0, 2.0] if lab == 0 else [2.0, 1.0]
        rows.append(DatasetRow(f"m{i}", (100, 100, nnz), (0.1, 0.0, 0.05, 0.001), 10.0, rt + [None] * 6,
                               [0.0, 0.0] + [None] * 6))
    m = seer.train_seer(rows, iterations=(1,))
    for r in rows:
        assert m.known_tree.predict(seer.known_vector(*r.known, 1)) == dataset.fastest_kernel(r.timings(), 1)
        assert m.selector_tree.predict(seer.known_vector(*r.known, 1)) == seer.USE_KNOWN
    m2 = seer.SeerModel.from_json(m.to_json())
    assert m2.to_json() == m.to_json()
    rep = seer.geomean_speedup(rows, m, 1)
    assert rep["selector_total"] == rep["oracle_total"]


def test_csv_roundtrip():
    rows = [DatasetRow("a", (3, 4, 5), (0.5, 0.0, 0.25, 0.01), 0.001, [1e-3, None], [0.0, 2e-3]),
            DatasetRow("b", (6, 6, 9), (0.5, 0.1, 0.25, 0.02), 0.002, [2e-3, 1e-4], [None, 0.0])]
    e, p, md = dataset.write_tables(rows, ["CSR,TM", "ELL,TM"])
    back = dataset.read_tables(e, p, md, {"a": (3, 4, 5), "b": (6, 6, 9)})
    for r, b in zip(rows, back):
        assert (r.runtime, r.preprocess, r.gathered, r.collection_time) == \
               (b.runtime, b.preprocess, b.gathered, b.collection_time)


def test_split():
    tr, te = dataset.split_train_test(list(range(10)), 3)
    assert len(tr) == 8 and len(te) == 2 and sorted(tr + te) == list(range(10))
    assert dataset.split_train_test(list(range(10)), 3) == (tr, te)


@pytest.mark.parametrize("kern", [0, 3, 7])
def test_fixed_model_is_that_kernel_everywhere(kern):
    """The constant-model plan used as the Seer-vs-fixed baseline (bench.py, eval_seer.py)
    must take the known path and answer `kern` for any features, and its realised cost
    must be exactly that kernel's total cost."""
    m = seer.fixed_model(kern)
    assert m.meta["fixed_kernel"] == seer.KERNELS[kern]
    rng = np.random.default_rng(kern)
    for _ in range(50):
        r, c = int(10 ** rng.uniform(1, 8)), int(10 ** rng.uniform(1, 8))
        nnz, k = int(10 ** rng.uniform(1, 9)), int(rng.choice([1, 10, 100]))
        o = seer.infer_features(m, (r, c, nnz), k, (1.0, 0.5, 2.0, 0.01))
        assert (o.chosen_kernel, o.path) == (kern, seer.USE_KNOWN)
    row = DatasetRow("f", (100, 100, 500), (0.1, 0.0, 0.05, 0.001), 10.0,
                     [1e-3 * (i + 1) for i in range(8)], [1e-4 * i for i in range(8)])
    for k in (1, 10, 100):
        assert seer.realized_cost(m, row, k)[0] == pytest.approx(row.cost(kern, k))


def test_lofo_realise_on_corpus_subset():
    """tools/lofo_seer.py's realisation on a small slice of the committed corpus: the
    selector can never beat the per-matrix oracle, and the frozen bundle's per-family
    numbers are well formed."""
    import importlib.util
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tools = os.path.join(root, "tools")
    import sys
    sys.path.insert(0, tools)
    spec = importlib.util.spec_from_file_location("lofo_seer", os.path.join(tools, "lofo_seer.py"))
    lofo = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(lofo)
    rows = lofo.load(os.path.join(root, "paper_2403_17017_b200", "models", "corpus"))
    fams = {}
    for r in rows:
        fams.setdefault(lofo.family(r.name), []).append(r)
    assert len(fams) >= 5
    frozen = seer.SeerModel.load(os.path.join(root, "paper_2403_17017_b200", "models", "seer_b200.json"))
    held_f = sorted(fams)[0]
    held = fams[held_f][:40]
    train = [r for f, rs in fams.items() if f != held_f for r in rs[:40]]
    m = seer.train_seer(train, (1, 10), 3, 4, seer.KERNELS)
    for model in (m, frozen):
        for k in (1, 10):
            res = lofo.realise(model, held, k)
            assert res["selector_over_oracle"] >= 1.0 - 1e-12
            assert res["oracle_total_s"] <= res["best_fixed_total_s"] * (1 + 1e-12)
            assert res["best_fixed"] in seer.KERNELS and res["aggregate_vs_best_fixed"] > 0
