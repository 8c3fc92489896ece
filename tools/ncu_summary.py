"""Summarise ncu reports / launch lists into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py --rep gpurun_out/full_C2.ncu-rep ... --launches gpurun_out/launches_C2.csv \
        --out profiles/ncu_r01.md --traffic-json profiles/traffic.json --workload C2
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 (LTS) %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1tex %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    h, units = r[0], r[1]
    res = []
    for v in r[2:]:
        d = {"kernel": short(v[h.index("Kernel Name")])}
        for m, lab in METRICS:
            if m in h:
                d[lab] = f"{v[h.index(m)]} {units[h.index(m)]}".strip()
        st = [(h[i], v[i]) for i in range(len(h)) if "smsp__pcsamp_warps_issue_stalled" in h[i]
              and not h[i].endswith("not_issued")]
        st = [(n.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x.replace(",", "")))
              for n, x in st if x not in ("", "n/a")]
        tot = sum(x for _, x in st) or 1.0
        d["top stalls"] = ", ".join(f"{n} {x / tot * 100:.0f}%" for n, x in sorted(st, key=lambda t: -t[1])[:4])
        try:
            d["_traffic"] = float(v[h.index("dram__bytes_read.sum")].replace(",", "")) * _scale(units[h.index("dram__bytes_read.sum")]) + \
                float(v[h.index("dram__bytes_write.sum")].replace(",", "")) * _scale(units[h.index("dram__bytes_write.sum")])
        except (ValueError, IndexError):
            pass
        res.append(d)
    return res


def short(name: str) -> str:
    """'void unnamed>::k_csr_merge<float, int, 1>(...)' -> 'k_csr_merge<float, int, 1>'."""
    base = name.split("(")[0] if "<" not in name.split("(")[0] else name[: name.index(">(") + 1] if ">(" in name else name
    base = base.replace("void ", "")
    return base.split("::")[-1] if "::" in base.split("<")[0] else base


def _scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.strip(), 1)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return {}
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[1:]:
        per.setdefault(r[ii], {"name": r[ki]})[r[mi]] = r[vi]
    agg = collections.OrderedDict()
    total = 0.0
    for v in per.values():
        n = short(v["name"]).split("<")[0]
        if not n.startswith("k_"):
            continue
        t = float(v.get("gpu__time_duration.sum", "0").replace(",", ""))
        agg.setdefault(n, []).append(t)
        total += t
    return {"total_ns": total, "kernels": {n: {"launches": len(l), "mean_us": sum(l) / len(l) / 1e3,
                                                "share": sum(l) / total if total else 0} for n, l in agg.items()}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--launches", nargs="*", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--traffic-json", default=None)
    ap.add_argument("--workload", default=None)
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    traffic = {}
    for rep in a.rep:
        lines += [f"## `{os.path.basename(rep)}` (ncu --set full, --clock-control none)", ""]
        for d in raw(rep):
            lines.append(f"### {d['kernel']}")
            for k, v in d.items():
                if k not in ("kernel", "_traffic"):
                    lines.append(f"- {k}: {v}")
            lines.append("")
            if "_traffic" in d:
                traffic[d["kernel"]] = d["_traffic"]
    for lp in a.launches:
        L = launches(lp)
        if not L:
            continue
        lines += [f"## launch list `{os.path.basename(lp)}` (ncu gpu__time_duration, cold + serialised: compare shares)",
                  "", "| kernel | launches | mean us | share of our GPU time |", "|---|---|---|---|"]
        for n, v in L["kernels"].items():
            lines.append(f"| {n} | {v['launches']} | {v['mean_us']:.2f} | {v['share'] * 100:.1f}% |")
        lines.append("")
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.traffic_json and a.workload:
        doc = {}
        if os.path.exists(a.traffic_json):
            doc = json.load(open(a.traffic_json))
        doc.setdefault(a.workload, {}).update({k: int(v) for k, v in traffic.items()})
        with open(a.traffic_json, "w") as f:
            json.dump(doc, f, indent=1)
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
