"""Selection latency with the bundle's trees compiled in (include/kp_seer_trees.h,
KP_SELECT_EMITTED) vs the packed-tree interpreter (KP_NO_EMITTED_TREES=1 ->
KP_SELECT_PARAM), on gathered-path plans: whole plan step (selection kernel + SWITCH +
body) as back-to-back graph launches and with a 512 MB L2 flush before each sample,
CUDA events on the launching stream, median of N.  JSON lines on stdout.

    python tools/select_latency.py [N]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import gen, kernels, seer  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
model = seer.SeerModel.load(os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json"))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(plan, s, flushed):
    ts = []
    for _ in range(N):
        if flushed:
            with torch.cuda.stream(s):
                flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        plan.launch(s)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


for name, k in (("C1", 10), ("C1", 100), ("C2", 10), ("C3", 100)):
    A = gen.config(name, device="cuda").to_device_csr(torch.float32)
    x = (torch.rand(A.n_cols, device="cuda", dtype=torch.float64) * 2 - 1).float()
    y = torch.empty(A.n_rows, device="cuda", dtype=torch.float32)
    s = torch.cuda.Stream()
    row = {"matrix": name, "k": k, "rows": A.n_rows, "nnz": A.nnz}
    for mode in ("emitted", "param"):
        if mode == "param":
            os.environ["KP_NO_EMITTED_TREES"] = "1"
        else:
            os.environ.pop("KP_NO_EMITTED_TREES", None)
        plan = seer.SeerPlan(model, A, x, y, k)
        assert plan.select_kind() == mode, (name, plan.select_kind())
        for _ in range(5):
            plan.launch(s)
        s.synchronize()
        o = plan.outcome()
        row["kernel"] = kernels.KERNELS[o.kernel]
        row["path"] = "gathered" if o.path else "known"
        row[f"{mode}_step_us_hot"] = round(timed(plan, s, False), 2)
        row[f"{mode}_step_us_flushed"] = round(timed(plan, s, True), 2)
        plan.close()
    os.environ.pop("KP_NO_EMITTED_TREES", None)
    print(json.dumps(row), flush=True)
    del A, x, y
    torch.cuda.empty_cache()
