"""Cost accounting and training labels (module ``dataset``).

On the hot path: ``total_cost`` and ``fastest_kernel``
 -- the amortised cost model Seer's labels and evaluation use.
Off the hot path but needed to store the B200 training corpus: the artifact CSV
schemas ``elapsed.csv`` / ``preprocess.csv`` (name + one column per
kernel, seconds, empty = missing) and ``metadata.csv``
(name, max/min/mean/var density, collection_time), plus the seeded 80/20 split.
"""

from __future__ import annotations

import csv
import io
import math
import random
from dataclasses import dataclass, field

from .errors import EmptyInputError, ParseError, SchemaError

INF = math.inf
METADATA_COLUMNS = ("name", "max_density", "min_density", "mean_density", "var_density", "collection_time")


def total_cost(runtime, preprocess, k: int) -> float:
    """preprocess + k * runtime; a missing kernel costs +inf (never a silent zero)."""
    if k < 1:
        raise ValueError("iterations must be >= 1")
    if runtime is None or preprocess is None:
        return INF
    return float(preprocess) + k * float(runtime)


def fastest_kernel(timings, k: int) -> int:
    """argmin over kernels of total_cost; ties go to the lowest vocabulary index.
    ``timings``: sequence of (runtime, preprocess) per kernel, None = missing."""
    costs = [total_cost(r, p, k) for r, p in timings]
    if not costs or all(c == INF for c in costs):
        raise EmptyInputError("all kernels missing")
    best = 0
    for i, c in enumerate(costs):
        if c < costs[best]:
            best = i
    return best


@dataclass
class DatasetRow:
    """One matrix: known features, gathered features (optional), per-kernel timings."""

    name: str
    known: tuple                      # (rows, cols, nnz)
    gathered: tuple | None = None     # (max, min, mean, var)
    collection_time: float = 0.0
    runtime: list = field(default_factory=list)     # per kernel, seconds per iteration (None = missing)
    preprocess: list = field(default_factory=list)  # per kernel, seconds one-time (None = missing)

    def timings(self):
        return list(zip(self.runtime, self.preprocess))

    def cost(self, kernel: int, k: int) -> float:
        return total_cost(self.runtime[kernel], self.preprocess[kernel], k)


def split_train_test(rows, seed: int, fraction: float = 0.8):
    """Deterministic shuffle under ``seed``; first ``fraction`` is train."""
    if not 0.0 < fraction < 1.0:
        raise ValueError("fraction must be in (0, 1)")
    if len(rows) < 2:
        raise EmptyInputError("need at least 2 rows to split")
    idx = list(range(len(rows)))
    random.Random(seed).shuffle(idx)
    cut = int(round(fraction * len(rows)))
    cut = min(max(cut, 1), len(rows) - 1)
    return [rows[i] for i in idx[:cut]], [rows[i] for i in idx[cut:]]


# ---------------------------------------------------------------------------- CSV
def _fmt(v) -> str:
    return "" if v is None else repr(float(v))


def write_tables(rows, kernels) -> tuple[str, str, str]:
    """(elapsed.csv, preprocess.csv, metadata.csv) texts for ``rows``."""
    el, pp, md = io.StringIO(), io.StringIO(), io.StringIO()
    we, wp, wm = csv.writer(el, lineterminator="\n"), csv.writer(pp, lineterminator="\n"), \
        csv.writer(md, lineterminator="\n")
    we.writerow(["name", *kernels])
    wp.writerow(["name", *kernels])
    wm.writerow(METADATA_COLUMNS)
    for r in rows:
        we.writerow([r.name, *(_fmt(v) for v in r.runtime)])
        wp.writerow([r.name, *(_fmt(v) for v in r.preprocess)])
        if r.gathered is not None:
            wm.writerow([r.name, *(_fmt(v) for v in r.gathered), _fmt(r.collection_time)])
    return el.getvalue(), pp.getvalue(), md.getvalue()


def _read_table(text: str, what: str):
    rd = list(csv.reader(io.StringIO(text)))
    if not rd or rd[0][:1] != ["name"]:
        raise SchemaError(f"{what}: header must start with 'name'")
    head, out = rd[0], {}
    for ln, row in enumerate(rd[1:], start=2):
        if not row:
            continue
        if len(row) != len(head):
            raise SchemaError(f"{what} line {ln}: {len(row)} fields, header has {len(head)}")
        if row[0] in out:
            raise SchemaError(f"{what} line {ln}: duplicate name {row[0]!r}")
        vals = []
        for cell in row[1:]:
            if cell == "":
                vals.append(None)
                continue
            try:
                v = float(cell)
            except ValueError:
                raise ParseError(f"{what} line {ln}: non-numeric value {cell!r}") from None
            if not math.isfinite(v):
                raise ParseError(f"{what} line {ln}: non-finite value {cell!r}")
            vals.append(v)
        out[row[0]] = vals
    return head[1:], out


def read_tables(elapsed: str, preprocess: str, metadata: str | None, known: dict) -> list[DatasetRow]:
    """Join the three artifact CSVs (plus known features by name) into DatasetRows."""
    k1, el = _read_table(elapsed, "elapsed.csv")
    k2, pp = _read_table(preprocess, "preprocess.csv")
    if k1 != k2:
        raise SchemaError("elapsed.csv and preprocess.csv kernel columns differ")
    md = {}
    if metadata is not None:
        head, md = _read_table(metadata, "metadata.csv")
        order = [head.index(c) for c in METADATA_COLUMNS[1:]]
        md = {n: [v[i] for i in order] for n, v in md.items()}
    rows = []
    for name in el:
        if name not in known:
            raise SchemaError(f"no known features for {name!r}")
        g = md.get(name)
        rows.append(DatasetRow(name, tuple(known[name]), tuple(g[:4]) if g else None, g[4] if g else 0.0,
                               el[name], pp.get(name, [None] * len(k1))))
    return rows
