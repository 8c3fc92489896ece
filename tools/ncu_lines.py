"""Per-source-line instruction and stall shares of one kernel from an ncu report
(`ncu -i rep --page source --print-source cuda,sass`).  Usage: ncu_lines.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, agg = None, {}
for r in csv.reader(io.StringIO(out)):
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 5:
        continue
    d = dict(zip(hdr, r))
    try:
        ln = int(r[0])
        ie = float(d.get("Instructions Executed") or 0)
        smp = float(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    a = agg.setdefault(ln, [0.0, 0.0, r[1][:100]])
    a[0] += ie
    a[1] += smp
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot:.0f}, stall samples {ts:.0f}")
for ln, (ie, smp, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:n]:
    print(f"{ln:5d} inst {ie / tot * 100:5.1f}% stall {smp / ts * 100:5.1f}%  {s}")
