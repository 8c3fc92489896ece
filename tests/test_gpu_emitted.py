"""The bundle's trees compiled into libkpb200 (include/kp_seer_trees.h; SPEC.md:302-307,
402) on the device: kp_seer_emitted_predict == kp_tree_predict (the packed-tree
interpreter) on 1e5 vectors including every threshold hit, and Seer plans built from the
bundle select through the compiled trees ('emitted') with outcomes equal to seer.infer
and y equal to the oracle; any other model keeps the interpreter ('param')."""
import ctypes
import os

import numpy as np
import pytest
import torch

from paper_2403_17017_b200 import _lib, dtree, gen, seer
from test_emitted_trees import vectors
from test_gpu_plan import TOL, _bundle, _check_y, _run_plan, _x

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tree", [0, 1, 2])
def test_emitted_equals_interpreter(tree):
    m = _bundle()
    X = vectors(m, n=100_000, seed=11 + tree)
    nf = 8 if tree == 2 else 4
    xd = torch.from_numpy(np.ascontiguousarray(X[:, :nf])).cuda()
    L = _lib.load()
    a = torch.full((X.shape[0],), -9, dtype=torch.int32, device="cuda")
    b = torch.full((X.shape[0],), -9, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(L.kp_seer_emitted_predict(tree, xd.data_ptr(), X.shape[0], a.data_ptr(), s), "emitted")
    dev = m.device_trees("cuda:0")[tree]
    _lib.check(L.kp_tree_predict(dev.data_ptr(), xd.data_ptr(), X.shape[0], nf, b.data_ptr(), s), "predict")
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    t = (m.selector_tree, m.known_tree, m.gathered_tree)[tree]
    host = np.array([t.predict(tuple(v[:nf])) for v in X[-2000:]])
    assert np.array_equal(a[-2000:].cpu().numpy(), host)


def test_emitted_rejects_bad_tree():
    L = _lib.load()
    assert L.kp_seer_emitted_predict(3, None, 0, None, None) == _lib.KP_EINVAL


def _gathered_cases(model):
    """(matrix, k) pairs the bundle's own selector sends to USE_GATHERED (the smallest k
    per matrix), so the test follows a retrained bundle."""
    out = []
    for m in (gen.config("C1"), gen.config("C4", small=True), gen.stencil27(20)):
        for k in (1, 3, 10, 30, 100, 1000):
            if model.selector_tree.predict(seer.known_vector(m.n_rows, m.n_cols, m.nnz, k)) == seer.USE_GATHERED:
                out.append((m, k))
                break
    assert out, "the bundle never takes the gathered path on the test shapes"
    return out


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("index", ["int32", "int64"])
def test_bundle_plan_uses_emitted_trees(dtype, index, orc):
    """Shapes the bundle's selector sends to USE_GATHERED: the plan's selection kernel runs
    the compiled trees (feature pass -> seer_gathered -> SWITCH)."""
    model = _bundle()
    for m, k in _gathered_cases(model):
        A = m.to_device_csr(dtype, index=index)
        x = _x(A.n_cols, dtype)
        y = torch.full((A.n_rows,), float("nan"), dtype=dtype, device="cuda")
        plan = seer.SeerPlan(model, A, x, y, k)
        assert plan.select_kind() == "emitted", m.name
        plan.launch()
        plan.launch()
        torch.cuda.synchronize()
        o = plan.outcome()
        plan.close()
        ref = seer.infer(model, A, k)
        assert ref.path == seer.USE_GATHERED, m.name
        assert (o.kernel, o.path) == (ref.chosen_kernel, ref.path), m.name
        assert (o.max_d, o.min_d, o.mean_d, o.var_d) == ref.features
        ok, r = _check_y(A, x, y, orc)
        assert ok, (m.name, dtype, index, r)


def test_other_models_keep_the_interpreter():
    model = seer.SeerModel(dtree.leaf_tree(0, 8, 4), dtree.leaf_tree(2, 8, 8),
                           dtree.leaf_tree(seer.USE_GATHERED, 2, 4))
    A = gen.config("C1").to_device_csr(torch.float32)
    x = _x(A.n_cols, torch.float32)
    y = torch.empty(A.n_rows, dtype=torch.float32, device="cuda")
    plan = seer.SeerPlan(model, A, x, y, 1)
    assert plan.select_kind() == "param"
    plan.close()
    # the bundle on a known-path shape: resolved at creation, no selection kernel per launch
    plan = seer.SeerPlan(_bundle(), A, x, y, 1)
    assert plan.select_kind() == "static"
    plan.close()
