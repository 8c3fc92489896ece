"""Seer runtime: the three-tree model and device-side inference.

* ``SeerModel`` -- known tree over (rows, cols, nnz, iterations), gathered tree over
  that + (max, min, mean, var) row density, selector tree over the known schema with
  classes {USE_KNOWN, USE_GATHERED}, plus the kernel vocabulary.
  Versioned JSON bundle.
* ``infer`` -- on a matrix, ONE fused kernel (``kp_seer_select``):
  every CTA evaluates the selector; USE_KNOWN answers from CTA 0 without touching
  the matrix (SPEC.md:388 purity); USE_GATHERED runs the feature pass and the last
  CTA evaluates the gathered tree on the bit-exact features.  The charged overhead
  is the measured collection time on the gathered path and 0 on the known path.
* ``train_seer`` / ``selector_label`` -- offline, host-side.
* ``SeerRunner.run`` -- select -> preprocess (cached) -> k SpMV iterations on the
  device: the end-to-end cost T_seer of SURVEY 8d.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .dataset import fastest_kernel
from .dtree import DecisionTree, leaf_tree, train_tree
from .kernels import KERNELS, NEEDS_PREP, prepare, spmv

SEER_FORMAT = "kernelpick-b200-seer/1"
KNOWN_SCHEMA = ("rows", "cols", "nnz", "iterations")
GATHERED_SCHEMA = KNOWN_SCHEMA + ("max_density", "min_density", "mean_density", "var_density")
USE_KNOWN, USE_GATHERED = 0, 1


@dataclass(frozen=True)
class InferenceOutcome:
    chosen_kernel: int
    path: int                    # USE_KNOWN / USE_GATHERED
    charged_overhead: float      # seconds; 0 on the known path
    predicted_total: float = float("nan")  # diagnostic only
    inference_time: float = 0.0  # the selection launch itself ("negligible but accounted")
    features: tuple | None = None


def known_vector(rows, cols, nnz, k) -> tuple:
    return (float(rows), float(cols), float(nnz), float(k))


class SeerModel:
    def __init__(self, known_tree: DecisionTree, gathered_tree: DecisionTree, selector_tree: DecisionTree,
                 kernels=KERNELS, meta: dict | None = None):
        self.known_tree, self.gathered_tree, self.selector_tree = known_tree, gathered_tree, selector_tree
        self.kernels = tuple(kernels)
        self.meta = dict(meta or {})
        if known_tree.n_classes != len(self.kernels) or gathered_tree.n_classes != len(self.kernels):
            raise ValueError("known/gathered trees must classify over the kernel vocabulary")
        if selector_tree.n_classes != 2:
            raise ValueError("selector tree must have 2 classes")
        if known_tree.n_features != 4 or selector_tree.n_features != 4 or gathered_tree.n_features != 8:
            raise ValueError("tree feature schemas must be known(4) / gathered(8) / selector(4)")
        self._dev: dict = {}

    # ------------------------------------------------------------------ bundle
    def to_json(self) -> str:
        return json.dumps({"format": SEER_FORMAT, "kernels": list(self.kernels), "meta": self.meta,
                           "known": self.known_tree.to_dict(), "gathered": self.gathered_tree.to_dict(),
                           "selector": self.selector_tree.to_dict()}, sort_keys=True, indent=1)

    @classmethod
    def from_json(cls, text: str) -> "SeerModel":
        from .errors import SchemaError
        d = json.loads(text)
        if not isinstance(d, dict) or d.get("format") != SEER_FORMAT:
            raise SchemaError("unsupported Seer bundle format")
        return cls(DecisionTree.from_dict(d["known"]), DecisionTree.from_dict(d["gathered"]),
                   DecisionTree.from_dict(d["selector"]), d["kernels"], d.get("meta"))

    @classmethod
    def load(cls, path: str) -> "SeerModel":
        with open(path) as f:
            return cls.from_json(f.read())

    def save(self, path: str) -> None:
        with open(path, "w") as f:
            f.write(self.to_json())

    def device_trees(self, device):
        """Packed (selector, known, gathered) trees resident on ``device``."""
        torch = _lib.require_cuda()
        key = str(device)
        if key not in self._dev:
            def up(t):
                raw = np.frombuffer(t.pack(), dtype=np.uint8).copy()
                return torch.from_numpy(raw).to(device)
            self._dev[key] = (up(self.selector_tree), up(self.known_tree), up(self.gathered_tree))
        return self._dev[key]

    # ------------------------------------------------------------------ host predict
    def predict_host(self, rows, cols, nnz, k, gathered=None) -> tuple[int, int]:
        """Host evaluation of the same trees (precomputed-features path / tests)."""
        kv = known_vector(rows, cols, nnz, k)
        path = self.selector_tree.predict(kv)
        if path == USE_KNOWN:
            return self.known_tree.predict(kv), USE_KNOWN
        if gathered is None:
            raise ValueError("selector demands gathered features but none were supplied")
        return self.gathered_tree.predict(kv + tuple(gathered)), USE_GATHERED

    # ------------------------------------------------------------------ emitted header
    def emit_header(self, source: str = "") -> str:
        """SPEC.md:402 ("one source header containing all three emitted functions plus a
        dispatch function mirroring infer's control flow") over SPEC.md:302-307 emit_source.
        One text for C hosts and CUDA device code (KP_SEER_HD).  The packed trees it was
        emitted from ride along, so a runtime can check a model it is handed against the
        compiled functions byte for byte before trusting them (kp_seer_plan_create does)."""
        import hashlib
        packed = [("selector", self.selector_tree), ("known", self.known_tree), ("gathered", self.gathered_tree)]
        sha = hashlib.sha256(b"".join(t.pack() for _, t in packed)).hexdigest()
        out = [f"/* kp_seer_trees.h -- GENERATED by tools/emit_trees.py{(' from ' + source) if source else ''};",
               " * do not edit.  Seer bundle " + SEER_FORMAT + ", kernels: " + ", ".join(
                   f"{i}={k}" for i, k in enumerate(self.kernels)) + ".",
               " * seer_selector / seer_known / seer_gathered: DecisionTree.emit_source (SPEC.md:302-307);",
               " * seer_dispatch: infer's control flow (SPEC.md:376-384).  Left iff x[f] <= threshold. */",
               "#ifndef KP_SEER_TREES_H", "#define KP_SEER_TREES_H", "",
               "#ifdef __CUDACC__", "#define KP_SEER_HD __host__ __device__", "#else",
               "#define KP_SEER_HD", "#endif", "",
               f'#define KP_SEER_TREES_SHA256 "{sha}"  /* sha256 of the three packed trees below */', ""]
        for name, t in packed:
            b = t.pack()
            out.append(f"/* dtree.pack() of the {name} tree ({len(b)} bytes): kp_tree_header + kp_tree_node[] */")
            out.append(f"static const unsigned char kp_seer_packed_{name}[{len(b)}] = {{")
            for i in range(0, len(b), 16):
                out.append("    " + ", ".join(f"0x{v:02x}" for v in b[i:i + 16]) + ",")
            out.append("};")
        out.append("")
        for name, t in packed:
            out.append(t.emit_source(f"seer_{name}", "hd"))
        out += ["/* infer (SPEC.md:376-384): the selector on the known features (rows, cols, nnz,",
                " * iterations); USE_KNOWN (0) -> the known tree, never reading `gathered`",
                " * (SPEC.md:388); USE_GATHERED (1) -> the gathered tree on known + (max, min, mean,",
                " * var) density, or -1 when `gathered` is NULL (the caller must collect features",
                " * first: seer_needs_gathered tells it so up front). */",
                "static inline KP_SEER_HD int seer_needs_gathered(double rows, double cols, double nnz, "
                "double iterations) {",
                "    const double xk[4] = {rows, cols, nnz, iterations};",
                "    return seer_selector(xk) != 0;",
                "}",
                "static inline KP_SEER_HD int seer_dispatch(double rows, double cols, double nnz, double iterations,",
                "                                           const double *gathered, int *path) {",
                "    const double xk[4] = {rows, cols, nnz, iterations};",
                "    if (seer_selector(xk) == 0) {",
                "        if (path) *path = 0;",
                "        return seer_known(xk);",
                "    }",
                "    if (path) *path = 1;",
                "    if (!gathered) return -1;",
                "    const double xg[8] = {rows, cols, nnz, iterations, gathered[0], gathered[1], gathered[2], gathered[3]};",
                "    return seer_gathered(xg);",
                "}", "", "#endif  /* KP_SEER_TREES_H */", ""]
        return "\n".join(out)


# ---------------------------------------------------------------------- inference
def select_async(model: SeerModel, A, k: int, out=None, stream=None):
    """Enqueue kp_seer_select for DeviceCSR ``A``; returns the 96-byte device outcome."""
    torch = _lib.require_cuda()
    from .device import reduce_workspace
    sel, kn, ga = model.device_trees(A.device)
    if out is None:
        out = torch.empty(_lib.OUTCOME_BYTES, dtype=torch.uint8, device=A.device)
    with torch.cuda.device(A.device):
        rc = _lib.load().kp_seer_select(A.row_offsets.data_ptr(), A.off_type, A.n_rows, A.n_cols, A.nnz, int(k),
                                        sel.data_ptr(), kn.data_ptr(), ga.data_ptr(), out.data_ptr(),
                                        reduce_workspace(A.device, stream).data_ptr(),
                                        _lib.stream_handle(stream, A.device))
    _lib.check(rc, "kp_seer_select")
    return out


def infer(model: SeerModel, m=None, k: int = 1, clock=None, features=None) -> InferenceOutcome:
    """SPEC.md:376-384.  ``m``: DeviceCSR or host SparseMatrixCSR (uploaded);
    ``features``: precomputed GatheredFeatures (host evaluation, overhead passed through)."""
    from .features import decode_outcome
    if m is None:
        if features is None:
            raise ValueError("infer needs a matrix or precomputed features")
        raise ValueError("precomputed-feature inference needs the known features: use infer_features")
    from .device import as_device
    A = as_device(m)
    clock = clock or time.perf_counter
    t0 = clock()
    buf = select_async(model, A, k)
    o = decode_outcome(buf)
    dt = clock() - t0
    if o.status == _lib.KP_ERANGE:
        raise OverflowError("feature epilogue outside the exactly representable range")
    gathered = o.path == USE_GATHERED
    feats = (o.max_d, o.min_d, o.mean_d, o.var_d) if gathered else None
    return InferenceOutcome(int(o.kernel), int(o.path), dt if gathered else 0.0, float("nan"), dt, feats)


def infer_features(model: SeerModel, known, k: int, gathered=None) -> InferenceOutcome:
    """Precomputed-features form of infer: ``known`` = (rows, cols, nnz);
    ``gathered`` = GatheredFeatures (its collection_time is the charged overhead)."""
    kv = known_vector(*known, k)
    path = model.selector_tree.predict(kv)
    if path == USE_KNOWN:
        return InferenceOutcome(model.known_tree.predict(kv), USE_KNOWN, 0.0)
    if gathered is None:
        raise ValueError("selector demands gathered features but neither matrix nor features were supplied")
    return InferenceOutcome(model.gathered_tree.predict(kv + tuple(gathered.as_vector())), USE_GATHERED,
                            float(gathered.collection_time), features=tuple(gathered.as_vector()))


class SeerRunner:
    """End-to-end Seer on one device matrix: select -> preprocess -> k SpMVs.

    The only host synchronisation is the 96-byte read of the selection outcome
    (the chosen kernel decides which kernel to launch next)."""

    def __init__(self, model: SeerModel):
        self.model = model

    def run(self, A, x, k: int = 1, y=None, stream=None, chain: bool = False):
        """Returns (y, outcome).  chain=False: y = A.x repeated k times (SPEC cost
        model k*runtime); chain=True: power iteration x <- A.x (square A)."""
        torch = _lib.require_cuda()
        from .features import decode_outcome
        buf = select_async(self.model, A, k, stream=stream)
        o = decode_outcome(buf, stream)  # ordered after the selection on `stream`
        kern = int(o.kernel)
        P = prepare(A, kern, stream=stream) if kern in NEEDS_PREP else None
        if y is None:
            y = torch.empty(A.n_rows, dtype=A.values.dtype, device=A.device)
        if chain:
            if A.n_rows != A.n_cols:
                raise ValueError("chain=True needs a square matrix")
            src, dst = x, y
            for _ in range(k):
                spmv(A, src, kern, y=dst, prepared=P, stream=stream)
                src, dst = dst, (x if dst is y else y)
            y = src
        else:
            for _ in range(k):
                spmv(A, x, kern, y=y, prepared=P, stream=stream)
        return y, o


class SeerPlan:
    """The whole pipeline (select -> chosen kernel's preprocessing -> k SpMVs) as one CUDA
    graph with device-side dispatch (``kp_seer_plan_*``): no host round trip per run.

    Binds ``A``, ``x`` and ``y`` (their device buffers; contents may change between
    launches).  ``launch()`` enqueues one graph launch on the current (or given) stream;
    ``outcome()`` reads the selection the last launch made."""

    def __init__(self, model: SeerModel, A, x, y, k: int = 1, ell_cap: int | None = None,
                 force_gathered: bool = False):
        """``force_gathered`` (measurement): replace the selector by a constant USE_GATHERED
        leaf, so every launch runs the feature pass + gathered tree + SWITCH -- the realised
        collection overhead the corpus charges to the gathered path."""
        import ctypes
        torch = _lib.require_cuda()
        from .device import as_device
        from .kernels import default_ell_cap
        from .kernels import check_vector
        self.A = as_device(A)
        # the graph binds raw pointers: x / y must stay valid, sized and on A's device
        check_vector(x, self.A, self.A.n_cols, "x")
        check_vector(y, self.A, self.A.n_rows, "y", out=True)
        if not x.is_contiguous():
            raise ValueError("x must be contiguous (the plan binds its pointer)")
        self.x, self.y, self.k = x, y, int(k)
        L = _lib.load()
        cap = int(ell_cap) if ell_cap else default_ell_cap(self.A)
        nbytes = ctypes.c_size_t(0)
        _lib.check(L.kp_seer_plan_bytes(ctypes.byref(self.A.struct), cap, ctypes.byref(nbytes)), "kp_seer_plan_bytes")
        dev = self.A.device
        self.buf = torch.empty(max(int(nbytes.value), 256), dtype=torch.uint8, device=dev)
        self.out = torch.zeros(_lib.OUTCOME_BYTES, dtype=torch.uint8, device=dev)
        self.red = torch.zeros(int(L.kp_reduce_workspace_bytes()), dtype=torch.uint8, device=dev)
        self.trees = model.device_trees(dev)
        sel, kn, ga = self.trees
        if force_gathered:
            import numpy as np
            from .dtree import leaf_tree
            raw = np.frombuffer(leaf_tree(USE_GATHERED, 2, 4).pack(), dtype=np.uint8).copy()
            sel = torch.from_numpy(raw).to(dev)
            self.trees = (sel, kn, ga)
        cap_stream = torch.cuda.Stream(device=dev)  # graph capture needs a created stream
        torch.cuda.synchronize(dev)
        handle = ctypes.c_void_p()
        with torch.cuda.device(dev):
            rc = L.kp_seer_plan_create(ctypes.byref(self.A.struct), self.k, cap, sel.data_ptr(), kn.data_ptr(),
                                       ga.data_ptr(), x.data_ptr(), y.data_ptr(), self.buf.data_ptr(), self.buf.numel(),
                                       self.red.data_ptr(), self.out.data_ptr(), ctypes.byref(handle),
                                       int(cap_stream.cuda_stream))
        _lib.check(rc, "kp_seer_plan_create")
        torch.cuda.synchronize(dev)
        self._handle = handle
        self._L = L

    def launch(self, stream=None) -> None:
        _lib.check(self._L.kp_seer_plan_launch(self._handle, _lib.stream_handle(stream, self.A.device)),
                   "kp_seer_plan_launch")

    def outcome(self):
        from .features import decode_outcome
        return decode_outcome(self.out)

    def select_kind(self) -> str:
        """How each launch selects: 'static' (known path resolved at creation), 'emitted'
        (the bundle compiled in from include/kp_seer_trees.h), 'param' (packed trees by
        value) or 'table' (trees in device memory)."""
        return ("static", "emitted", "param", "table")[self._L.kp_seer_plan_select_kind(self._handle)]

    def close(self) -> None:
        if getattr(self, "_handle", None) is not None and self._handle.value:
            self._L.kp_seer_plan_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------- training
def selector_label(row, known_pred: int, gathered_pred: int, k: int) -> int:
    """USE_GATHERED iff cost(gathered_pred) + collection < cost(known_pred);
    ties -> USE_KNOWN."""
    cg = row.cost(gathered_pred, k) + row.collection_time
    ck = row.cost(known_pred, k)
    return USE_GATHERED if cg < ck else USE_KNOWN


def train_seer(rows, iterations=(1,), max_depth: int = 5, min_samples_leaf: int = 1,
               kernels=KERNELS, meta: dict | None = None, weighting: str = "none",
               near_best: float = 0.0, selector_folds: int = 0, gathered_depth: int | None = None) -> SeerModel:
    """labels = fastest_kernel per (matrix, k); known tree on the known
    schema, gathered tree on the full schema, selector on labels from the two
    sub-models' own predictions on the training rows.

    weighting="none" is SPEC's plain CART.  weighting="regret" (extension) weights each
    example by what a wrong decision costs relative to the matrix's best time:
    kernel trees by log1p(mean relative regret over the other kernels), the selector by
    |log(realised gathered-path cost / realised known-path cost)| -- measured kernel
    families have 100-1000x outliers (thread-mapped schedules on 1M-nnz rows) that
    unweighted CART treats like a 1% miss.

    near_best > 0 (extension) relabels each example with the kernel that is most often
    within (1 + near_best) x the best time across the training set, among the kernels
    within that factor on this example: ties between near-equal kernels stop being label
    noise for CART (the realised cost changes by < near_best).

    gathered_depth (extension): a separate depth for the gathered tree, which sees 8
    features (and the iteration count) where the known and selector trees see 4."""
    nk = len(kernels)
    gd = max_depth if gathered_depth is None else int(gathered_depth)
    pref = np.zeros(nk)
    if near_best > 0:
        for r in rows:
            for k in iterations:
                c = [r.cost(j, k) for j in range(nk)]
                b = min(c)
                if np.isfinite(b):
                    for j in range(nk):
                        if c[j] <= b * (1 + near_best):
                            pref[j] += 1
    Xk, Xg, y, ex, wk = [], [], [], [], []
    for r in rows:
        if r.gathered is None:
            raise ValueError(f"row {r.name!r} has no gathered features")
        for k in iterations:
            try:
                lab = fastest_kernel(r.timings(), k)
            except Exception:
                continue
            if near_best > 0:
                b = r.cost(lab, k)
                cands = [j for j in range(nk) if r.cost(j, k) <= b * (1 + near_best)]
                lab = max(cands, key=lambda j: (pref[j], -j))
            kv = known_vector(*r.known, k)
            Xk.append(kv)
            Xg.append(kv + tuple(r.gathered))
            y.append(lab)
            ex.append((r, k))
            best = r.cost(lab, k)
            regrets = [(r.cost(j, k) - best) / best for j in range(nk)
                       if j != lab and np.isfinite(r.cost(j, k))]
            wk.append(float(np.log1p(np.mean(regrets))) if regrets else 0.0)
    if not y:
        raise ValueError("no labelled examples")
    if weighting in ("cost-log", "cost-rel", "cost-mix"):
        return _train_seer_cost(ex, Xk, Xg, max_depth, min_samples_leaf, kernels, meta, weighting, selector_folds, gd)
    if weighting not in ("none", "regret"):
        raise ValueError("weighting must be 'none', 'regret', 'cost-log', 'cost-rel' or 'cost-mix'")
    w = None if weighting == "none" else np.asarray(wk) + 1e-3
    kt = train_tree(Xk, y, max_depth, min_samples_leaf, nk, KNOWN_SCHEMA, w)
    gt = train_tree(Xg, y, gd, min_samples_leaf, nk, GATHERED_SCHEMA, w)
    ys, wsel = [], []
    for (r, k), xk, xg in zip(ex, Xk, Xg):
        kp, gp = kt.predict(xk), gt.predict(xg)
        ys.append(selector_label(r, kp, gp, k))
        ck, cg = r.cost(kp, k), r.cost(gp, k) + r.collection_time
        wsel.append(abs(float(np.log(cg / ck))) if np.isfinite(ck) and np.isfinite(cg) else 10.0)
    ws = None if weighting == "none" else np.asarray(wsel) + 1e-3
    st = train_tree(Xk, ys, max_depth, min_samples_leaf, 2, KNOWN_SCHEMA, ws)
    meta = dict(meta or {})
    meta.setdefault("weighting", weighting)
    return SeerModel(kt, gt, st, kernels, meta)


def _loss(costs, kind: str, cap: float = 1e3):
    """Per-example loss of predicting each class: cost-log = log(t / t_best) (per-matrix
    geomean objective), cost-rel = t / t_best - 1, cost-mix = log(t / t_best) + (t - t_best)
    / 1 ms (adds the aggregate-time objective, so large matrices are not out-voted by many
    small ones).  Missing kernels (inf) are capped at cap x t_best."""
    c = np.asarray(costs, dtype=np.float64)
    b = np.min(c[np.isfinite(c)])
    r = np.where(np.isfinite(c), c / b, cap)
    r = np.minimum(r, cap)
    if kind == "cost-log":
        return np.log(r)
    if kind == "cost-mix":
        return np.log(r) + (r - 1.0) * b / 1e-3
    return r - 1.0


def _train_seer_cost(ex, Xk, Xg, max_depth, min_samples_leaf, kernels, meta, kind,
                     selector_folds: int = 0, gathered_depth=None) -> SeerModel:
    """Cost-sensitive trio (extension): kernel trees minimise the summed loss of the
    realised per-iteration-count cost (log or relative regret vs the example's best
    kernel), the selector minimises the loss of the realised known vs gathered path
    (collection time charged, SPEC.md:367-375 costs).

    selector_folds > 1 (extension): the selector's known / gathered path costs come from
    OUT-OF-FOLD sub-model predictions (matrices split into that many folds; each fold
    predicted by trees trained on the others).  In-sample predictions make the known tree
    look right wherever it was fit, so the selector never learns where its blind spot
    (skew the known features cannot see) lies; out-of-fold costs expose it."""
    from .dtree import train_cost_tree
    nk = len(kernels)
    Ck = np.stack([_loss([r.cost(j, k) for j in range(nk)], kind) for r, k in ex])
    kt = train_cost_tree(Xk, Ck, max_depth, min_samples_leaf, KNOWN_SCHEMA)
    gd = max_depth if gathered_depth is None else gathered_depth
    gt = train_cost_tree(Xg, Ck, gd, min_samples_leaf, GATHERED_SCHEMA)
    kpred = [kt.predict(xk) for xk in Xk]
    gpred = [gt.predict(xg) for xg in Xg]
    if selector_folds > 1:
        names = sorted({r.name for r, _ in ex})
        fold_of = {n: i % selector_folds for i, n in enumerate(names)}
        fold = np.array([fold_of[r.name] for r, _ in ex])
        Xk_a, Xg_a = np.asarray(Xk, dtype=np.float64), np.asarray(Xg, dtype=np.float64)
        for f in range(selector_folds):
            tr, te = np.nonzero(fold != f)[0], np.nonzero(fold == f)[0]
            if len(te) == 0 or len(tr) == 0:
                continue
            kt_f = train_cost_tree(Xk_a[tr], Ck[tr], max_depth, min_samples_leaf, KNOWN_SCHEMA)
            gt_f = train_cost_tree(Xg_a[tr], Ck[tr], gd, min_samples_leaf, GATHERED_SCHEMA)
            for i in te:
                kpred[i] = kt_f.predict(Xk[i])
                gpred[i] = gt_f.predict(Xg[i])
    Cs = []
    for (r, k), kp, gp in zip(ex, kpred, gpred):
        ck = r.cost(kp, k)
        cg = r.cost(gp, k) + r.collection_time
        Cs.append(_loss([ck, cg], kind))
    st = train_cost_tree(Xk, np.stack(Cs), max_depth, min_samples_leaf, KNOWN_SCHEMA)
    meta = dict(meta or {})
    meta.setdefault("weighting", kind)
    return SeerModel(kt, gt, st, kernels, meta)


def realized_cost(model: SeerModel, row, k: int) -> tuple[float, int, int]:
    """(cost incl. charged collection, kernel, path) of the selector on a dataset row."""
    kv = known_vector(*row.known, k)
    path = model.selector_tree.predict(kv)
    if path == USE_KNOWN:
        kern = model.known_tree.predict(kv)
        return row.cost(kern, k), kern, path
    kern = model.gathered_tree.predict(kv + tuple(row.gathered))
    return row.cost(kern, k) + row.collection_time, kern, path


def geomean_speedup(rows, model: SeerModel, k: int) -> dict:
    """geomean over fixed kernels K of total(K) / total(selector), totals
    summed over ``rows``; also the best-fixed-kernel aggregate ratio.  Delegates to
    ``evaluate.evaluate`` so the missing-kernel rules are the eval module's: +inf for the
    selector's own choices, worst-present substitution only in the fixed-kernel totals."""
    from . import evaluate as ev
    rep = ev.evaluate(model, list(rows), k)
    sel = rep.predictors["selector"].total_realized_cost
    fixed = [rep.predictors[K].total_realized_cost for K in rep.kernels]
    return {"selector_total": sel, "fixed_totals": fixed,
            "geomean_vs_fixed": ev.geomean_speedup(rep),
            "vs_best_fixed": min(fixed) / sel,
            "oracle_total": rep.predictors["oracle"].total_realized_cost}


def fixed_model(kernel) -> SeerModel:
    """A constant model: the selector always takes the known path and both trees answer
    `kernel`.  A SeerPlan of it is that fixed kernel's prep + k SpMVs built and launched
    exactly like a Seer plan (same capture, same graph launch) -- the baseline the
    Seer-vs-fixed comparisons time."""
    k = kernel if isinstance(kernel, int) else KERNELS.index(kernel)
    return SeerModel(leaf_tree(k, len(KERNELS), 4), leaf_tree(k, len(KERNELS), 8), leaf_tree(USE_KNOWN, 2, 4),
                     KERNELS, {"fixed_kernel": KERNELS[k]})


def bootstrap_model() -> SeerModel:
    """A rule-derived placeholder used only until a B200-measured bundle exists
    (models/seer_b200.json).  Selector always gathers; gathered tree splits on
    mean/max density like the paper's Table III intuition."""
    rng = np.random.default_rng(0)
    X, y = [], []
    for _ in range(4000):
        rows = float(10 ** rng.uniform(3, 7.5))
        mean = float(10 ** rng.uniform(0, 2.5))
        cols = rows
        mx = mean * float(10 ** rng.uniform(0, 4))
        nnz = rows * mean
        k = float(rng.choice([1, 10, 100]))
        var = (mx - mean) ** 2 / 50
        if mx > 64 * mean:
            lab = 2 if k < 10 else 0          # skewed: MP / adaptive
        elif mean >= 24 and mx <= 2 * mean:
            lab = 7 if k >= 10 else 3         # regular: ELL when amortised
        elif mean > 12:
            lab = 3
        else:
            lab = 5
        X.append((rows, cols, nnz, k, mx / cols, 0.0, mean / cols, var / cols / cols))
        y.append(lab)
    gt = train_tree(X, y, 5, 1, 8, GATHERED_SCHEMA)
    kt = train_tree([x[:4] for x in X], y, 5, 1, 8, KNOWN_SCHEMA)
    st = leaf_tree(USE_GATHERED, 2, 4, KNOWN_SCHEMA)
    return SeerModel(kt, gt, st, KERNELS, {"source": "bootstrap rules (not B200-measured)"})

