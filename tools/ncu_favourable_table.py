"""Summarise scripts/ncu_favourable.sh launch lists into a markdown table: per SpMV kernel
and matrix, median ncu duration and DRAM bytes (cold-cache, serialised launches), the
measured DRAM GB/s against the HBM peak, and the byte-model GB/s beside it.

    python tools/ncu_favourable_table.py gpurun_out/ncu_fav_*.csv > profiles/ncu_favourable_r01.md"""
import collections
import csv
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
kb = json.load(open(os.path.join(ROOT, "profiles", "kbench_r01.json")))
LABEL = {"k_adaptive": "Adaptive-CSR", "k_csr_bm": "CSR,BM", "k_csr_wm": "CSR,WM", "k_csr_tm": "CSR,TM",
         "k_coo_wm": "COO,WM", "k_ell_tm": "ELL,TM"}
print("# Per-kernel ncu evidence on favourable inputs (round 1)\n")
print("ncu `--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
      "--clock-control none` over `tools/kbench.py` (cold L2 per launch, serialised); the merge "
      "kernel serves CSR,MP and CSR,WO (listed once per matrix).  Byte-model GB/s from "
      f"`profiles/kbench_r01.json` (CUDA events).  Peak = {peak} GB/s (MEASURED_PEAKS.json).\n")
print("| matrix | kernel | launches | median us (ncu) | DRAM MB / launch | DRAM GB/s | frac of peak | byte-model frac (events) |")
print("|---|---|---|---|---|---|---|---|")
for path in sys.argv[1:]:
    mat = os.path.basename(path).replace("ncu_fav_", "").replace(".csv", "")
    rows = [r for r in csv.reader(open(path)) if len(r) > 6]
    if not rows:
        continue
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[1:]:
        per.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.OrderedDict()
    for v in per.values():
        base = v["name"].split("<")[0].split("::")[-1].replace("void ", "").strip()
        if base.startswith("unnamed>"):
            base = base.split(">::")[-1]
        agg.setdefault(base, []).append(v)
    for base, L in agg.items():
        t = statistics.median(x["gpu__time_duration.sum"] for x in L) * 1e-9
        b = statistics.median(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in L)
        lab = LABEL.get(base, "CSR,MP/WO" if base == "k_csr_merge" else base)
        ref = kb.get(mat, {}).get(lab if lab != "CSR,MP/WO" else "CSR,MP", {}).get("frac", "")
        print(f"| {mat} | {lab} (`{base}`) | {len(L)} | {t * 1e6:.1f} | {b / 1e6:.1f} | {b / t / 1e9:.0f} | "
              f"{b / t / 1e9 / peak:.2f} | {ref} |")
