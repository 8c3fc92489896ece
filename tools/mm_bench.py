"""Matrix Market ingest throughput: native kp_mm_parse (all host threads and 1 thread) vs
the reference's parse_matrix_market algorithm (sparse.py:106-196, Python), same text.

    python tools/mm_bench.py [--lines 2000000] [--reference]

--reference imports the UNMODIFIED reference from /root/reference/pkg/src (build container
only; the GPU box has no /root/reference)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2403_17017_b200 import mmio  # noqa: E402


def make_text(n: int, side: int = 1 << 20, seed: int = 5) -> bytes:
    rng = np.random.default_rng(seed)
    r = rng.integers(1, side + 1, n)
    c = rng.integers(1, side + 1, n)
    v = rng.uniform(-1, 1, n)
    body = "\n".join(f"{a} {b} {x!r}" for a, b, x in zip(r.tolist(), c.tolist(), v.tolist()))
    return f"%%MatrixMarket matrix coordinate real general\n{side} {side} {n}\n{body}\n".encode()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lines", type=int, default=2_000_000)
    ap.add_argument("--reference", action="store_true")
    a = ap.parse_args()
    text = make_text(a.lines)
    out = {"lines": a.lines, "bytes": len(text)}
    for th, key in ((0, "native_all_threads"), (1, "native_1_thread")):
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            mmio.parse_arrays(text, n_threads=th)
            best = min(best, time.perf_counter() - t0)
        out[key + "_s"] = round(best, 4)
        out[key + "_MBps"] = round(len(text) / best / 1e6, 1)
    out["host_threads"] = os.cpu_count()
    if a.reference:
        sys.path.insert(0, "/root/reference/pkg/src")
        os.environ["KERNELPICK_PURE_KERNELS"] = "1"
        from kernelpick import sparse as ref
        t0 = time.perf_counter()
        m = ref.parse_matrix_market(text)
        out["reference_s"] = round(time.perf_counter() - t0, 3)
        out["reference_MBps"] = round(len(text) / out["reference_s"] / 1e6, 2)
        mine = mmio.parse_matrix_market(text)
        out["parity"] = bool(np.array_equal(mine.row_offsets, m.row_offsets) and
                             np.array_equal(mine.col_indices, m.col_indices) and
                             np.array_equal(mine.values.view(np.int64), m.values.view(np.int64)))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
