"""The Seer plan's GATHERED branch on the device: the graph-flavour selection kernel
(k_seer_plan_select: trees by value, feature pass, gathered tree, cudaGraphSetConditional)
and every one of the 8 SWITCH bodies (prepare + k SpMVs), checked against the host
restatement of SPEC infer on the reference-pinned features and against
the fp64 CPU oracle for y (tol 1e-5 fp32 / 1e-12 fp64, normwise)."""
import os

import numpy as np
import pytest
import torch

from paper_2403_17017_b200 import dtree, gen, kernels, seer
from paper_2403_17017_b200.features import gather_features

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = {torch.float32: 1e-5, torch.float64: 1e-12}


def _bundle():
    return seer.SeerModel.load(os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json"))


def _gathered_leaf_model(cls):
    """Selector = USE_GATHERED leaf, gathered tree = leaf `cls`, known tree never consulted."""
    return seer.SeerModel(dtree.leaf_tree(0, 8, 4), dtree.leaf_tree(cls, 8, 8),
                          dtree.leaf_tree(seer.USE_GATHERED, 2, 4))


def _fixtures():
    return [gen.config("C1"), gen.config("C2", small=True), gen.config("C4", small=True),
            gen.stencil27(14), gen.powerlaw_rows(20_000, 9.0, 1.4, seed=8)]


def _x(n, dtype, seed=3):
    g = torch.Generator().manual_seed(seed)
    return (torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1).to(dtype).cuda()


def _run_plan(model, A, x, k, **kw):
    y = torch.full((A.n_rows,), float("nan"), dtype=A.values.dtype, device="cuda")
    plan = seer.SeerPlan(model, A, x, y, k, **kw)
    for _ in range(2):  # re-launch: the body and its prepared buffers are reused
        plan.launch()
    torch.cuda.synchronize()
    o = plan.outcome()
    plan.close()
    return y, o


def _check_y(A, x, y, orc):
    off, col, val = A.to_host()
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    ok, r = orc.spmv_check(y.cpu().numpy(), yref, absy, TOL[A.values.dtype])
    return ok, r


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("index", ["int32", "int64"])
@pytest.mark.parametrize("cls", range(8))
def test_gathered_switch_body(cls, dtype, index, orc):
    """SWITCH body `cls` reached through the device-side gathered path on every fixture:
    outcome == seer.infer (kernel, path, bit-exact features), y == oracle."""
    model = _gathered_leaf_model(cls)
    for m in _fixtures():
        A = m.to_device_csr(dtype, index=index)
        x = _x(A.n_cols, dtype)
        k = 3 if cls != kernels.CSR_TM or A.nnz < 1e6 else 1
        y, o = _run_plan(model, A, x, k)
        ref = seer.infer(model, A, k)
        assert (o.kernel, o.path) == (cls, seer.USE_GATHERED) == (ref.chosen_kernel, ref.path), m.name
        off64 = A.row_offsets.cpu().numpy().astype(np.int64)
        want = orc.gather_features(off64, A.n_rows, A.n_cols)
        assert (o.max_d, o.min_d, o.mean_d, o.var_d) == want == ref.features, m.name
        ok, r = _check_y(A, x, y, orc)
        assert ok, (m.name, kernels.KERNELS[cls], dtype, index, r)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_bundle_forced_gathered_matches_host(dtype, orc):
    """The frozen bundle's multi-level gathered tree walked from the kernel parameter space
    (force_gathered): the device pick equals the host predict on the device's features."""
    model = _bundle()
    for m in _fixtures() + [gen.banded(50_000, 27), gen.constant_rows(40_000, 3, seed=2)]:
        A = m.to_device_csr(dtype)
        x = _x(A.n_cols, dtype)
        for k in (1, 10):
            y, o = _run_plan(model, A, x, k, force_gathered=True)
            g = gather_features(A)
            kv = seer.known_vector(A.n_rows, A.n_cols, A.nnz, k)
            assert o.path == seer.USE_GATHERED
            assert o.kernel == model.gathered_tree.predict(kv + g.as_vector()), (m.name, k)
            assert (o.max_d, o.min_d, o.mean_d, o.var_d) == g.as_vector()
            ok, r = _check_y(A, x, y, orc)
            assert ok, (m.name, k, r)


def test_plan_selector_tree_mixed_paths(orc):
    """A selector that splits on nnz sends small matrices down the known path and large
    ones down the gathered path inside the same model; both plans agree with infer."""
    rng = np.random.default_rng(1)
    X = np.stack([10 ** rng.uniform(3, 7, 400), 10 ** rng.uniform(3, 7, 400), 10 ** rng.uniform(4, 8, 400),
                  rng.choice([1, 10, 100], 400)], 1)
    sel = dtree.train_tree(X, (X[:, 2] > 5e5).astype(int), 2, 1, 2)
    kn = dtree.train_tree(X, (X[:, 0] > 1e5).astype(int) * 3 + 2, 3, 1, 8)  # MP / COO
    Xg = np.concatenate([X, rng.uniform(0, 1e-3, (400, 4))], 1)
    gt = dtree.train_tree(Xg, (Xg[:, 6] > 5e-4).astype(int) * 4 + 3, 3, 1, 8)  # WM / ELL
    model = seer.SeerModel(kn, gt, sel)
    for m in (gen.config("C1"), gen.config("C2"), gen.stencil27(60)):
        A = m.to_device_csr(torch.float32)
        x = _x(A.n_cols, torch.float32)
        y, o = _run_plan(model, A, x, 2)
        ref = seer.infer(model, A, 2)
        assert (o.kernel, o.path) == (ref.chosen_kernel, ref.path)
        assert o.path == (1 if A.nnz > 5e5 else 0)
        ok, r = _check_y(A, x, y, orc)
        assert ok, (m.name, r)


def test_c3_full_size_plan_gathered_k100(orc):
    """BASELINE configs[2] at full size, k = 100: the bundle takes USE_GATHERED natively;
    the plan's pick equals the host restatement and y (= A.x after 100 iterations of the
    same SpMV) matches the oracle."""
    model = _bundle()
    A = gen.config("C3", device="cuda").to_device_csr(torch.float32)
    x = _x(A.n_cols, torch.float32)
    y, o = _run_plan(model, A, x, 100)
    g = gather_features(A)
    kern, path = model.predict_host(A.n_rows, A.n_cols, A.nnz, 100, g.as_vector())
    assert (o.kernel, o.path) == (kern, path)
    if path == seer.USE_GATHERED:
        assert (o.max_d, o.min_d, o.mean_d, o.var_d) == g.as_vector()
    ok, r = _check_y(A, x, y, orc)
    assert ok, r


def test_c3_full_size_every_kernel(orc):
    A = gen.config("C3", device="cuda").to_device_csr(torch.float32)
    x = _x(A.n_cols, torch.float32)
    off, col, val = A.to_host()
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    for k in range(8):
        y = torch.full((A.n_rows,), float("nan"), dtype=torch.float32, device="cuda")
        kernels.spmv(A, x, k, y=y, prepared=kernels.prepare(A, k, cache=False) if k in kernels.NEEDS_PREP else None)
        ok, r = orc.spmv_check(y.cpu().numpy(), yref, absy, 1e-5)
        assert ok, (kernels.KERNELS[k], r)


def test_c4_full_size_fp64_every_kernel(orc):
    """BASELINE configs[3] (four 1M-nnz rows, fp64) at 1e-12: the long rows are split over
    thousands of merge units / adaptive pieces and finished by k_carry_fixup."""
    A = gen.config("C4", device="cuda").to_device_csr(torch.float64)
    x = _x(A.n_cols, torch.float64)
    off, col, val = A.to_host()
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    for k in range(8):
        y = torch.full((A.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
        kernels.spmv(A, x, k, y=y, prepared=kernels.prepare(A, k, cache=False) if k in kernels.NEEDS_PREP else None)
        ok, r = orc.spmv_check(y.cpu().numpy(), yref, absy, 1e-12)
        assert ok, (kernels.KERNELS[k], r)
    # and through the bundle's plan
    y, o = _run_plan(_bundle(), A, x, 1)
    ok, r = orc.spmv_check(y.cpu().numpy(), yref, absy, 1e-12)
    assert ok, (kernels.KERNELS[o.kernel], r)


def test_c5_full_size_sampled_rows(orc):
    """BASELINE configs[4] at N = 1 (R-MAT s26, ~1.06 B nnz): the bundle's plan, checked on
    4096 sampled rows (their entries copied from the generated matrix) against the oracle."""
    m = gen.config("C5", device="cuda")
    A = m.to_device_csr(torch.float32)
    rng = np.random.default_rng(26)
    rows = np.sort(rng.choice(m.n_rows, 4096, replace=False))
    offh = m.row_offsets.cpu().numpy()
    samples = [(r, m.col_indices[offh[r]:offh[r + 1]].cpu().numpy(), m.values[offh[r]:offh[r + 1]].cpu().numpy())
               for r in rows]
    del m
    torch.cuda.empty_cache()
    x = _x(A.n_cols, torch.float32, seed=9)
    y, o = _run_plan(_bundle(), A, x, 1)
    xh = x.cpu().numpy().astype(np.float64)
    yh = y.cpu().numpy()
    for r, c, v in samples:
        vv = v.astype(np.float32).astype(np.float64)
        ref = float(np.dot(vv, xh[c]))
        assert abs(float(yh[r]) - ref) <= 1e-5 * float(np.abs(vv * xh[c]).sum()) + 1e-30, (r, kernels.KERNELS[o.kernel])
