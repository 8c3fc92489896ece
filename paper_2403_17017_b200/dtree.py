"""From-scratch CART decision trees (module ``dtree``).

The reference ships no tree code; this restates the SPEC contract:

* ``gini``, ``best_split``: thresholds at the
  midpoints of consecutive distinct values, go left iff ``x <= threshold``, ties to
  the lower feature index then the lower threshold;
* ``train_tree``: recursive CART, stops on a pure node, the depth
  limit, ``min_samples_leaf`` or no impurity-reducing split; leaf = majority label,
  ties to the lowest class (defaults depth 5, leaf 1: SPEC.md:323);
* ``predict``, ``emit_source`` (C/CUDA nested
  conditionals with exact hex-float thresholds), versioned serialisation
  (SPEC.md:308-312);
* ``pack`` -- the device layout (kp_tree_header + kp_tree_node[], kernelpick_b200.h)
  that ``kp_tree_predict`` / ``kp_seer_select`` evaluate on the GPU.

Training is host-side and offline (it produces the frozen bundle); prediction on the
runtime path happens on the device.
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field

import numpy as np

TREE_FORMAT = "kernelpick-b200-tree/1"


def gini(labels) -> float:
    """1 - sum_c p_c^2 over a non-empty label multiset."""
    y = np.asarray(labels)
    if y.size == 0:
        raise ValueError("gini of an empty label set")
    _, counts = np.unique(y, return_counts=True)
    p = counts / y.size
    return float(1.0 - np.sum(p * p))


def _midpoint(a: float, b: float) -> float:
    t = (a + b) / 2.0
    # adjacent doubles: the midpoint may round up to b, which would send b left
    return a if t >= b else t


def best_split(X, y, min_samples_leaf: int = 1, n_classes: int | None = None, sample_weight=None):
    """(feature, threshold, weighted impurity) minimising the children's weighted
    Gini, or None when no split reduces impurity.

    ``sample_weight`` (extension, default None = SPEC's plain CART): per-sample weights
    enter the class frequencies and the children's weighting; ``min_samples_leaf``
    still counts samples."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.int64)
    n = y.size
    if n < 2:
        return None
    k = int(n_classes if n_classes is not None else y.max() + 1)
    w = np.ones(n) if sample_weight is None else np.asarray(sample_weight, dtype=np.float64)
    W = float(w.sum())
    if W <= 0:
        return None
    tot = np.bincount(y, weights=w, minlength=k)
    parent = float(1.0 - np.sum((tot / W) ** 2))
    if np.count_nonzero(np.bincount(y, minlength=k)) <= 1:
        return None
    onehot = np.zeros((n, k), dtype=np.float64)
    onehot[np.arange(n), y] = w
    best = None  # (impurity, feature, threshold)
    for f in range(X.shape[1]):
        order = np.argsort(X[:, f], kind="stable")
        xs = X[order, f]
        cl = np.cumsum(onehot[order], axis=0)          # weighted class mass of the left prefix
        nl = np.arange(1, n + 1)
        # candidate split after position i (left = 0..i) where xs[i] < xs[i+1]
        pos = np.flatnonzero(xs[:-1] < xs[1:])
        if pos.size == 0:
            continue
        nL = nl[pos]
        nR = n - nL
        ok = (nL >= min_samples_leaf) & (nR >= min_samples_leaf)
        pos = pos[ok]
        if pos.size == 0:
            continue
        cL = cl[pos]
        cR = tot[None, :] - cL
        wL = cL.sum(1)
        wR = cR.sum(1)
        with np.errstate(invalid="ignore", divide="ignore"):
            gL = np.where(wL > 0, 1.0 - np.sum((cL / wL[:, None]) ** 2, axis=1), 0.0)
            gR = np.where(wR > 0, 1.0 - np.sum((cR / wR[:, None]) ** 2, axis=1), 0.0)
        imp = (wL * gL + wR * gR) / W
        i = int(np.argmin(imp))  # first minimum = lowest threshold for this feature
        cand = (float(imp[i]), f, _midpoint(float(xs[pos[i]]), float(xs[pos[i] + 1])))
        if best is None or cand[0] < best[0]:
            best = cand
    # SPEC.md:281 says "none when no split reduces impurity" but SPEC.md:295 requires XOR
    # (no single split reduces Gini) to reach 100% at depth 2.  We follow CART as in
    # scikit (impurity decrease >= 0 accepted) so both the XOR example and the
    # "splitting never increases impurity" invariant hold; pure nodes and
    # constant features still return None.
    if best is None or best[0] > parent + 1e-15:
        return None
    return best[1], best[2], best[0]


def _majority(y, n_classes: int, w=None) -> int:
    counts = np.bincount(np.asarray(y, dtype=np.int64), weights=w, minlength=n_classes)
    return int(np.argmax(counts))  # argmax returns the lowest index on ties


@dataclass
class DecisionTree:
    """Flat binary tree: node i is a leaf iff feature[i] < 0 (class value[i])."""

    feature: list = field(default_factory=list)
    threshold: list = field(default_factory=list)
    left: list = field(default_factory=list)
    right: list = field(default_factory=list)
    value: list = field(default_factory=list)
    n_classes: int = 1
    n_features: int = 0
    max_depth: int = 5
    feature_names: list = field(default_factory=list)

    @property
    def n_nodes(self) -> int:
        return len(self.feature)

    def depth(self) -> int:
        def d(i):
            return 0 if self.feature[i] < 0 else 1 + max(d(self.left[i]), d(self.right[i]))
        return d(0)

    def _add(self, f, thr, v) -> int:
        self.feature.append(int(f))
        self.threshold.append(float(thr))
        self.left.append(-1)
        self.right.append(-1)
        self.value.append(int(v))
        return len(self.feature) - 1

    # ------------------------------------------------------------------ predict
    def predict(self, x) -> int:
        """root-to-leaf descent, left iff x[f] <= threshold."""
        if len(x) != self.n_features:
            raise ValueError(f"feature vector has {len(x)} entries, tree expects {self.n_features}")
        i = 0
        while self.feature[i] >= 0:
            i = self.left[i] if float(x[self.feature[i]]) <= self.threshold[i] else self.right[i]
        return self.value[i]

    def predict_many(self, X) -> np.ndarray:
        return np.array([self.predict(row) for row in np.asarray(X, dtype=np.float64)], dtype=np.int64)

    # ------------------------------------------------------------------ (de)serialise
    def to_dict(self) -> dict:
        return {"format": TREE_FORMAT, "n_classes": self.n_classes, "n_features": self.n_features,
                "max_depth": self.max_depth, "feature_names": list(self.feature_names),
                "feature": list(self.feature), "threshold": [float(t) for t in self.threshold],
                "left": list(self.left), "right": list(self.right), "value": list(self.value)}

    @classmethod
    def from_dict(cls, d: dict) -> "DecisionTree":
        from .errors import SchemaError
        if not isinstance(d, dict) or d.get("format") != TREE_FORMAT:
            raise SchemaError(f"unsupported tree format {d.get('format') if isinstance(d, dict) else d!r}")
        try:
            t = cls([int(v) for v in d["feature"]], [float(v) for v in d["threshold"]],
                    [int(v) for v in d["left"]], [int(v) for v in d["right"]], [int(v) for v in d["value"]],
                    int(d["n_classes"]), int(d["n_features"]), int(d["max_depth"]), list(d["feature_names"]))
        except (KeyError, TypeError, ValueError) as e:
            raise SchemaError(f"malformed tree: {e}") from None
        t.validate()
        return t

    def serialize(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True, separators=(",", ":"))

    @classmethod
    def deserialize(cls, text: str) -> "DecisionTree":
        return cls.from_dict(json.loads(text))

    def validate(self) -> None:
        from .errors import SchemaError
        n = self.n_nodes
        if n == 0 or not (len(self.threshold) == len(self.left) == len(self.right) == len(self.value) == n):
            raise SchemaError("malformed node table")
        seen = [0] * n
        stack = [0]
        while stack:
            i = stack.pop()
            if not 0 <= i < n:
                raise SchemaError("child index out of range")
            seen[i] += 1
            if self.feature[i] >= 0:
                if self.feature[i] >= self.n_features:
                    raise SchemaError("split feature out of range")
                stack += [self.left[i], self.right[i]]
            elif not 0 <= self.value[i] < self.n_classes:
                raise SchemaError("leaf class out of range")
        if any(c != 1 for c in seen):
            raise SchemaError("tree is not a well-formed binary tree")

    # ------------------------------------------------------------------ device layout
    def pack(self) -> bytes:
        """kp_tree_header {n_nodes, n_features, n_classes, max_depth} + kp_tree_node[]
        {double threshold; int32 feature, left, right, value} (little endian, 24 B)."""
        out = [struct.pack("<iiii", self.n_nodes, self.n_features, self.n_classes, self.max_depth)]
        for i in range(self.n_nodes):
            out.append(struct.pack("<diiii", self.threshold[i], self.feature[i], self.left[i],
                                   self.right[i], self.value[i]))
        return b"".join(out)

    # ------------------------------------------------------------------ source emission
    def emit_source(self, name: str, dialect: str = "cuda") -> str:
        """Nested conditionals equivalent to ``predict``.
        dialect 'c', 'cuda' (adds __host__ __device__) or 'hd' (qualified by a KP_SEER_HD
        macro the including header defines, so one text compiles as C and as CUDA);
        thresholds as exact hex floats."""
        quals = {"c": "static inline int", "cuda": "static inline __host__ __device__ int",
                 "hd": "static inline KP_SEER_HD int"}
        if dialect not in quals:
            raise ValueError("dialect must be 'c', 'cuda' or 'hd'")
        qual = quals[dialect]
        names = self.feature_names or [f"f{i}" for i in range(self.n_features)]
        lines = [f"/* {name}: features {', '.join(names)}; left iff x[f] <= threshold */",
                 f"{qual} {name}(const double *x) {{"]

        def rec(i, ind):
            pad = "    " * ind
            if self.feature[i] < 0:
                lines.append(f"{pad}return {self.value[i]};")
                return
            f = self.feature[i]
            lines.append(f"{pad}if (x[{f}] <= {float(self.threshold[i]).hex()}) {{  /* {names[f]} */")
            rec(self.left[i], ind + 1)
            lines.append(f"{pad}}} else {{")
            rec(self.right[i], ind + 1)
            lines.append(f"{pad}}}")

        rec(0, 1)
        lines.append("}")
        return "\n".join(lines) + "\n"


def leaf_tree(cls: int, n_classes: int, n_features: int, feature_names=()) -> DecisionTree:
    t = DecisionTree(n_classes=n_classes, n_features=n_features, max_depth=0, feature_names=list(feature_names))
    t._add(-1, 0.0, cls)
    return t


def train_tree(X, y, max_depth: int = 5, min_samples_leaf: int = 1, n_classes: int | None = None,
               feature_names=(), sample_weight=None) -> DecisionTree:
    """Recursive CART with Gini; deterministic for fixed input order.
    ``sample_weight`` is an extension (None = SPEC's plain CART)."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.int64)
    if y.size == 0:
        raise ValueError("empty training set")
    if X.ndim != 2 or X.shape[0] != y.size:
        raise ValueError("X must be (n_samples, n_features) matching y")
    if max_depth < 0:
        raise ValueError("max_depth must be >= 0")
    k = int(n_classes if n_classes is not None else y.max() + 1)
    sw = None if sample_weight is None else np.asarray(sample_weight, dtype=np.float64)
    t = DecisionTree(n_classes=k, n_features=X.shape[1], max_depth=max_depth, feature_names=list(feature_names))

    def grow(idx: np.ndarray, depth: int) -> int:
        yy = y[idx]
        ww = None if sw is None else sw[idx]
        node = t._add(-1, 0.0, _majority(yy, k, ww))
        if depth >= max_depth or np.all(yy == yy[0]) or idx.size < 2 * min_samples_leaf:
            return node
        s = best_split(X[idx], yy, min_samples_leaf, k, ww)
        if s is None:
            return node
        f, thr, _ = s
        go_left = X[idx, f] <= thr
        t.feature[node] = f
        t.threshold[node] = thr
        t.value[node] = -1
        t.left[node] = grow(idx[go_left], depth + 1)
        t.right[node] = grow(idx[~go_left], depth + 1)
        return node

    grow(np.arange(y.size), 0)
    # leaves keep their class; split nodes carry value -1 -> normalise to 0 for packing
    t.value = [v if f < 0 else 0 for f, v in zip(t.feature, t.value)]
    return t


def train_cost_tree(X, C, max_depth: int = 5, min_samples_leaf: int = 1, feature_names=()) -> DecisionTree:
    """Cost-sensitive CART (extension; same tree format and ``predict`` as SPEC's CART).

    ``C[i, j]`` is the loss of predicting class j for example i (e.g. log(t_j / t_best)).
    A leaf predicts argmin_j sum_i C[i, j] (lowest class on ties); a split minimises the
    children's summed leaf losses, thresholds at midpoints between distinct sorted values,
    ``x <= thr`` goes left, first (feature, threshold) wins ties -- deterministic like
    ``train_tree``.  Kernel families with 100-1000x outliers make the label-purity
    criterion (Gini) a poor proxy for the time a wrong pick costs; this optimises it."""
    X = np.asarray(X, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    if C.ndim != 2 or X.ndim != 2 or X.shape[0] != C.shape[0] or C.shape[0] == 0:
        raise ValueError("X (n, f) and C (n, classes) must be non-empty and aligned")
    if not np.all(np.isfinite(C)):
        raise ValueError("costs must be finite (cap missing kernels first)")
    k = C.shape[1]
    t = DecisionTree(n_classes=k, n_features=X.shape[1], max_depth=max_depth, feature_names=list(feature_names))

    def leaf(idx):
        s = C[idx].sum(axis=0)
        j = int(np.argmin(s))
        return j, float(s[j])

    def split(idx):
        best = None
        _, here = leaf(idx)
        for f in range(X.shape[1]):
            xs = X[idx, f]
            order = np.argsort(xs, kind="stable")
            xv = xs[order]
            cs = np.cumsum(C[idx][order], axis=0)
            tot = cs[-1]
            n = xv.size
            # candidate cut after position p (left = 0..p): distinct neighbours, leaf sizes
            p = np.arange(min_samples_leaf - 1, n - min_samples_leaf)
            p = p[xv[p] < xv[p + 1]]
            if p.size == 0:
                continue
            loss = cs[p].min(axis=1) + (tot - cs[p]).min(axis=1)
            q = int(np.argmin(loss))
            if best is None or loss[q] < best[2] - 1e-12:
                best = (f, _midpoint(float(xv[p[q]]), float(xv[p[q] + 1])), float(loss[q]))
        if best is None or best[2] >= here - 1e-12:
            return None  # no split lowers the loss
        return best

    def grow(idx: np.ndarray, depth: int) -> int:
        node = t._add(-1, 0.0, leaf(idx)[0])
        if depth >= max_depth or idx.size < 2 * min_samples_leaf:
            return node
        s = split(idx)
        if s is None:
            return node
        f, thr, _ = s
        go_left = X[idx, f] <= thr
        t.feature[node] = f
        t.threshold[node] = thr
        t.value[node] = -1
        t.left[node] = grow(idx[go_left], depth + 1)
        t.right[node] = grow(idx[~go_left], depth + 1)
        return node

    grow(np.arange(C.shape[0]), 0)
    t.value = [v if f < 0 else 0 for f, v in zip(t.feature, t.value)]
    return t
