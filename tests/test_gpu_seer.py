"""Device tree evaluation and fused selection vs the host restatement (bit-exact indices)."""
import numpy as np
import pytest
import torch

from paper_2403_17017_b200 import _lib, dtree, gen, seer
from paper_2403_17017_b200.features import gather_features

pytestmark = pytest.mark.gpu


def _device_predict(t, X):
    L = _lib.load()
    tt = torch.from_numpy(np.frombuffer(t.pack(), dtype=np.uint8).copy()).cuda()
    xd = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float64)).cuda()
    out = torch.empty(X.shape[0], dtype=torch.int32, device="cuda")
    _lib.check(L.kp_tree_predict(tt.data_ptr(), xd.data_ptr(), X.shape[0], X.shape[1], out.data_ptr(),
                                 _lib.stream_handle()), "kp_tree_predict")
    return out.cpu().numpy()


def test_tree_predict_1e5_random_vectors():
    rng = np.random.default_rng(0)
    for depth in (0, 1, 3, 5, 8):
        X = rng.normal(size=(2000, 8)) * 10 ** rng.uniform(-4, 7, size=(1, 8))
        y = rng.integers(0, 8, 2000)
        t = dtree.train_tree(X, y, depth, 1, 8)
        Q = rng.normal(size=(100_000, 8)) * 10 ** rng.uniform(-4, 7, size=(1, 8))
        for j in range(min(t.n_nodes, 1000)):  # boundary values: x == threshold goes left
            if t.feature[j] >= 0:
                Q[j, t.feature[j]] = t.threshold[j]
        assert np.array_equal(_device_predict(t, Q), t.predict_many(Q))


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_seer_select_matches_host_infer(name):
    m = gen.config(name, small=name != "C1")
    A = m.to_device_csr(torch.float32)
    model = seer.bootstrap_model()
    for k in (1, 10, 100):
        o = seer.infer(model, A, k)
        g = gather_features(A)
        kern, path = model.predict_host(A.n_rows, A.n_cols, A.nnz, k, g.as_vector())
        assert (o.chosen_kernel, o.path) == (kern, path)
        assert o.features == g.as_vector()


def test_seer_known_path_does_not_read_matrix():
    """SPEC.md:388 purity: with a USE_KNOWN selector the select kernel never reads offsets
    -- pass a poisoned (NaN-free but garbage) offsets buffer and expect the known answer."""
    kt = dtree.leaf_tree(6, 8, 4)
    model = seer.SeerModel(kt, dtree.leaf_tree(1, 8, 8), dtree.leaf_tree(seer.USE_KNOWN, 2, 4))
    m = gen.config("C1")
    A = m.to_device_csr(torch.float32)
    A.row_offsets.fill_(-7)  # garbage: a gathered pass would produce nonsense features
    o = seer.infer(model, A, 1)
    assert (o.chosen_kernel, o.path, o.charged_overhead) == (6, seer.USE_KNOWN, 0.0)


def test_runner_end_to_end(orc):
    m = gen.config("C3", small=True)
    A = m.to_device_csr(torch.float32)
    x = (torch.rand(A.n_cols, device="cuda", dtype=torch.float64) * 2 - 1).float()
    y, o = seer.SeerRunner(seer.bootstrap_model()).run(A, x, k=3)
    off, col, val = A.to_host()
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    assert orc.spmv_check(y.cpu().numpy(), yref, absy, 1e-5)[0]


@pytest.mark.parametrize("name,k", [("C1", 1), ("C2", 1), ("C3", 3), ("C4", 2)])
def test_plan_graph_matches_host_dispatch(name, k, orc):
    """The one-graph pipeline (device-side SWITCH) selects the same kernel as the
    host-dispatched path and produces bit-identical y."""
    import os
    m = gen.config(name, small=name != "C1")
    A = m.to_device_csr(torch.float64 if name == "C4" else torch.float32)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    model = seer.SeerModel.load(os.path.join(root, "paper_2403_17017_b200", "models", "seer_b200.json"))
    x = (torch.rand(A.n_cols, device="cuda", dtype=torch.float64) * 2 - 1).to(A.values.dtype)
    y_plan = torch.full((A.n_rows,), float("nan"), device="cuda", dtype=A.values.dtype)
    plan = seer.SeerPlan(model, A, x, y_plan, k)
    for _ in range(3):
        plan.launch()
    torch.cuda.synchronize()
    o = plan.outcome()
    y_host, o2 = seer.SeerRunner(model).run(A, x, k=k)
    assert (o.kernel, o.path) == (o2.kernel, o2.path)
    assert torch.equal(y_plan, y_host)
    off, col, val = A.to_host()
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    tol = 1e-12 if name == "C4" else 1e-5
    assert orc.spmv_check(y_plan.cpu().numpy(), yref, absy, tol)[0]
    plan.close()
