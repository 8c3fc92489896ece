"""SPEC eval module (no reference code): oracle comparison, accuracy /
error / speedup per predictor, and Fig. 5 / Fig. 7-shaped plot data (CSV + a minimal,
dependency-free stacked-bar SVG).  Host-side reporting over DatasetRow timing tables --
the measured B200 corpus (tools/collect_corpus.py) or live runs (tools/eval_seer.py).

Predictors: known, gathered, selector (the Seer trio), oracle (fastest kernel, zero
overhead), and every fixed kernel (zero overhead).  Overhead = the gathered path's
collection time, never hidden from the speedup denominator.
"""

from __future__ import annotations

import io
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import dataset, seer
from .errors import EmptyInputError


@dataclass
class PredictorResult:
    total_realized_cost: float
    accuracy: float
    error_vs_oracle: float
    rows: list = field(default_factory=list)  # (matrix, chosen kernel, overhead, cost)
    substituted: int = 0  # fixed kernels only: missing entries replaced by the worst present one


@dataclass
class EvalReport:
    k: int
    kernels: tuple
    predictors: dict  # name -> PredictorResult

    def geomean_speedup(self) -> float:
        return geomean_speedup(self)


def oracle_choice(row, k: int) -> int:
    """fastest_kernel(row.timings, k), zero overhead."""
    return dataset.fastest_kernel(row.timings(), k)


def _cost(row, K, k, fixed: bool = False):
    """Realised cost of kernel K.  A missing kernel costs +inf, so a model
    that predicts it is maximally penalised; only FIXED-kernel baselines substitute the
    worst present kernel, so their totals (the geomean's numerators) stay
    finite.  Such substitutions are counted in ``PredictorResult.substituted``."""
    c = row.cost(K, k)
    if fixed and not np.isfinite(c):
        c = max(row.cost(j, k) for j in range(len(row.timings())) if np.isfinite(row.cost(j, k)))
    return c


def evaluate(model: seer.SeerModel, rows, k: int) -> EvalReport:
    """realised cost per predictor = total_cost(chosen, k) + charged
    overhead; accuracy = fraction choosing the oracle kernel; error = sum(realised - oracle)."""
    if not rows:
        raise EmptyInputError("evaluate needs at least one row")
    nk = len(model.kernels)
    preds = {}

    def run(name, choose, fixed=False):
        res = PredictorResult(0.0, 0.0, 0.0)
        hits = 0
        for r in rows:
            kern, over = choose(r)
            cost = _cost(r, kern, k, fixed) + over
            res.substituted += int(fixed and not np.isfinite(r.cost(kern, k)))
            orc = oracle_choice(r, k)
            res.rows.append((r.name, kern, over, cost))
            res.total_realized_cost += cost
            res.error_vs_oracle += cost - _cost(r, orc, k)
            hits += kern == orc
        res.accuracy = hits / len(rows)
        preds[name] = res

    run("oracle", lambda r: (oracle_choice(r, k), 0.0))
    run("known", lambda r: (model.known_tree.predict(seer.known_vector(*r.known, k)), 0.0))
    run("gathered", lambda r: (model.gathered_tree.predict(seer.known_vector(*r.known, k) + tuple(r.gathered)),
                               r.collection_time))

    def sel(r):
        cost, kern, path = seer.realized_cost(model, r, k)
        return kern, (r.collection_time if path == seer.USE_GATHERED else 0.0)
    run("selector", sel)
    for K in range(nk):
        run(model.kernels[K], lambda r, K=K: (K, 0.0), fixed=True)
    return EvalReport(k, tuple(model.kernels), preds)


def geomean_speedup(report: EvalReport) -> float:
    """geometric mean over fixed kernels of total(K) / total(selector)."""
    sel = report.predictors["selector"].total_realized_cost
    tots = [report.predictors[K].total_realized_cost for K in report.kernels]
    return float(math.exp(sum(math.log(t / sel) for t in tots) / len(tots)))


def _bars(report: EvalReport, rows_idx=None):
    """(label, runtime, overhead) per bar: |kernels| fixed + 4 predictors."""
    out = []
    for name in list(report.kernels) + ["known", "gathered", "selector", "oracle"]:
        p = report.predictors[name]
        sel = p.rows if rows_idx is None else [p.rows[rows_idx]]
        over = sum(x[2] for x in sel)
        cost = sum(x[3] for x in sel)
        out.append((name, cost - over, over))
    return out


def _csv(bars) -> str:
    import csv
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")  # kernel labels contain commas ("CSR,MP")
    w.writerow(["predictor", "runtime_s", "overhead_s"])
    for name, rt, ov in bars:
        w.writerow([name, repr(float(rt)), repr(float(ov))])
    return buf.getvalue()


def _svg(bars, title: str) -> str:
    """Stacked bars (runtime + lighter overhead segment), hand-written rects / labels."""
    W, H, pad, bw = 40 * len(bars) + 80, 320, 50, 28
    top = max((rt + ov) for _, rt, ov in bars) or 1.0
    s = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}" font-family="sans-serif" font-size="10">',
         f'<text x="{W / 2:.0f}" y="16" text-anchor="middle" font-size="12">{title}</text>']
    for i, (name, rt, ov) in enumerate(bars):
        x = pad + i * 40
        h1 = (H - 2 * pad) * rt / top
        h2 = (H - 2 * pad) * ov / top
        y1 = H - pad - h1
        s.append(f'<rect x="{x}" y="{y1:.2f}" width="{bw}" height="{h1:.2f}" fill="#3b6ea8"/>')
        if h2 > 0:
            s.append(f'<rect x="{x}" y="{y1 - h2:.2f}" width="{bw}" height="{h2:.2f}" fill="#9cc0e8"/>')
        s.append(f'<text x="{x + bw / 2:.1f}" y="{H - pad + 12}" text-anchor="end" '
                 f'transform="rotate(-45 {x + bw / 2:.1f} {H - pad + 12})">{name}</text>')
    s.append(f'<text x="8" y="{pad - 6}">{top * 1e3:.3g} ms</text></svg>')
    return "\n".join(s) + "\n"


def emit_plot_data(report: EvalReport, out_dir: str, per_matrix: bool = True) -> list[str]:
    """per-matrix and aggregate CSV + SVG, named like the artifact
    appendix (plots/single_iteration/<name>.svg, plots/multi_iteration/<name>_<k>iter.svg).
    Deterministic bytes for deterministic input."""
    sub = "single_iteration" if report.k == 1 else "multi_iteration"
    d = os.path.join(out_dir, sub)
    os.makedirs(d, exist_ok=True)
    suffix = "" if report.k == 1 else f"_{report.k}iter"
    written = []
    items = [("aggregate", None)]
    if per_matrix:
        items += [(name, i) for i, (name, *_rest) in enumerate(report.predictors["oracle"].rows)]
    for name, idx in items:
        bars = _bars(report, idx)
        base = os.path.join(d, f"{name}{suffix}")
        with open(base + ".csv", "w") as f:
            f.write(_csv(bars))
        with open(base + ".svg", "w") as f:
            f.write(_svg(bars, f"{name} (k = {report.k})"))
        written += [base + ".csv", base + ".svg"]
    return written
