"""Does a kernel chain cost more inside the plan's SWITCH body than as a top-level graph?
For (matrix, kernel, k): the gathered-path plan of a model whose selector is a
USE_GATHERED leaf and whose gathered tree is a `kernel` leaf (selection + feature pass +
SWITCH -> prep + k SpMVs) vs the same prep + k SpMVs captured as a plain graph vs the
feature pass alone.  CUDA events on the launching stream, L2 flushed, median of N.
JSON lines.

    python tools/body_overhead.py [C3:7:1,10,100 C1:5:1,10,100 ...]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import dtree, features, gen, kernels, seer  # noqa: E402

N = int(os.environ.get("N", "15"))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def med(fn, s):
    with torch.cuda.stream(s):
        fn()
    s.synchronize()
    ts = []
    for _ in range(N):
        with torch.cuda.stream(s):
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        with torch.cuda.stream(s):
            fn()
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


specs = sys.argv[1:] or ["C3:7:1,10,100", "C1:5:1,10,100", "C2:4:1,10"]
for spec in specs:
    name, kern, ks = spec.split(":")
    kern = int(kern)
    dt = torch.float64 if name == "C4" else torch.float32
    A = gen.config(name, device="cuda").to_device_csr(dt)
    x = torch.rand(A.n_cols, device="cuda", dtype=dt)
    y = torch.empty(A.n_rows, device="cuda", dtype=dt)
    s = torch.cuda.Stream()
    model = seer.SeerModel(dtree.leaf_tree(0, 8, 4), dtree.leaf_tree(kern, 8, 8),
                           dtree.leaf_tree(seer.USE_GATHERED, 2, 4))
    out = torch.empty(96, dtype=torch.uint8, device="cuda")
    gf = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gf, stream=s):
        features.gather_outcome(A, out=out)
    t_feat = med(gf.replay, s)
    for k in [int(v) for v in ks.split(",")]:
        plan = seer.SeerPlan(model, A, x, y, k)

        def body():
            P = kernels.prepare(A, kern, cache=False) if kern in kernels.NEEDS_PREP else None
            for _ in range(k):
                kernels.spmv(A, x, kern, y=y, prepared=P)

        with torch.cuda.stream(s):
            body()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            body()
        t_plan = med(lambda: plan.launch(s), s)
        t_body = med(g.replay, s)
        print(json.dumps({"matrix": name, "kernel": kernels.KERNELS[kern], "k": k, "plan_us": round(t_plan, 2),
                          "body_graph_us": round(t_body, 2), "feature_pass_us": round(t_feat, 2),
                          "switch_overhead_us": round(t_plan - t_body - t_feat, 2),
                          "per_iteration_extra_us": round((t_plan - t_body - t_feat) / k, 3)}), flush=True)
        plan.close()
        del g
    del A, x, y
    torch.cuda.empty_cache()
