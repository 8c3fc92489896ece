"""Seer-selected SpMV benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C2]

One STEP = the Seer hot path over one matrix (T_seer): fused selection
(selector tree -> gathered feature pass -> gathered/known tree, one kernel), the chosen
kernel's preprocessing (not cached across steps: charged every step), then k SpMV
iterations.  Default workload = BASELINE configs[1] (C2: R-MAT scale 20, edge factor 16,
permuted, fp32, k = 1), generated on the device with a counter-based hash (synthetic).

value      = CSR algorithmic bytes x k / device time of the step   [GB/s]
             (bytes = nnz*(4+4) + (R+1)*4 + C*4 + R*4, x counted once; inputs resident)
e2e        = same metric through the public API with HOST buffers: pinned host CSR + x
             copied H2D, the Seer pipeline, y copied D2H, all inside the timed region
roofline   = the chosen SpMV op's own byte model / its CUDA-event duration vs the
             measured HBM copy bandwidth (MEASURED_PEAKS.json)
sweep      = every fixed kernel's prep + k*SpMV on the same matrix; geomean and best-fixed
             speedups of Seer against them (the paper's 6.5x / 2x metrics)
cpu_baseline = the oracle port on this host (OpenMP CPU SpMV + compiled reference
             length_stats + restated predict), bounded ~10 s sample, rank 0 only
L2: the 141 MB matrix exceeds the 126 MB L2 and a 512 MB buffer is rewritten between
steps (outside the timed events) -> config["l2"] = "flushed".
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def _peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--iters", type=int, default=None, help="SpMV iterations k (default per config)")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--exchange", default="auto", choices=["auto", "fused", "nccl"],
                    help="C5: y exchange (fused epilogue stores over NVLink, or NCCL all-gather)")
    return ap.parse_args()


CFG = {  # BASELINE.json configs -> (k, dtype, description)
    "C1": (1, "float32", "uniform-random CSR 10k x 10k, ~100k nnz, fp32, k=1"),
    "C2": (1, "float32", "R-MAT s20 ef16 (0.57/0.19/0.19/0.05) permuted CSR 1M x 1M, ~16.1M nnz, fp32, k=1"),
    "C3": (100, "float32", "27-point stencil 159^3 (R=4,019,679, 107.2M nnz), fp32, k=100"),
    "C4": (1, "float64", "skewed 2M rows: Poisson(8) + 4 rows x 1M nnz, fp64, k=1"),
    "C5": (20, "float32", "R-MAT s26 ef16 row-stochastic (64M rows, ~1.0B nnz), fp32, 20 power iterations, "
                          "row-sharded over the ranks with an NCCL all-gather of y per iteration"),
}


def csr_bytes(R, C, Z, sv, so):
    return Z * (4 + sv) + (R + 1) * so + C * sv + R * sv


# ------------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [v.strip() for v in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------ helpers
def _load_model():
    from paper_2403_17017_b200 import seer
    path = os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json")
    if os.path.exists(path):
        return seer.SeerModel.load(path), "paper_2403_17017_b200/models/seer_b200.json"
    return seer.bootstrap_model(), "bootstrap rules (no B200 bundle yet)"


def _make_matrix(name, device):
    from paper_2403_17017_b200 import gen
    return gen.config(name, device=device)


# ------------------------------------------------------------------------ our arm
def run_ours(a):
    import torch
    import torch.distributed as dist
    from paper_2403_17017_b200 import _lib, kernels, seer
    from paper_2403_17017_b200.features import decode_outcome
    from paper_2403_17017_b200.device import DeviceCSR

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one rank per GPU; KP_BENCH_DIST_BACKEND=gloo (test only) lets N ranks share the GPUs
    # present so the multi-rank control flow can be exercised on a 1-GPU box
    backend = os.environ.get("KP_BENCH_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    L = _lib.load()

    k_default, dt_name, desc = CFG[a.workload]
    k = a.iters or k_default
    dtype = getattr(torch, dt_name)
    m = _make_matrix(a.workload, dev)
    A = m.to_device_csr(dtype, device=dev)
    del m
    R, C, Z = A.n_rows, A.n_cols, A.nnz
    sv, so = A.values.element_size(), A.row_offsets.element_size()
    bytes_csr = csr_bytes(R, C, Z, sv, so)
    model, model_src = _load_model()
    g = torch.Generator(device=dev).manual_seed(1234)
    x = (torch.rand(C, device=dev, dtype=torch.float64, generator=g) * 2 - 1).to(dtype)
    y = torch.empty(R, device=dev, dtype=dtype)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    obuf = torch.empty(_lib.OUTCOME_BYTES, dtype=torch.uint8, device=dev)
    ohost = torch.empty(_lib.OUTCOME_BYTES, dtype=torch.uint8, pin_memory=True)

    def read_outcome():
        ohost.copy_(obuf, non_blocking=True)
        stream.synchronize()
        return decode_outcome(ohost)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def seer_step(AA, xx, yy, marks=None):
        seer.select_async(model, AA, k, out=obuf)
        o = read_outcome()
        kern = int(o.kernel)
        P = kernels.prepare(AA, kern, cache=False) if kern in kernels.NEEDS_PREP else None
        if marks is not None:
            marks[0].record()
        for _ in range(k):
            kernels.spmv(AA, xx, kern, y=yy, prepared=P)
        if marks is not None:
            marks[1].record()
        return o, P

    def fixed_step(kern, marks=None):
        P = kernels.prepare(A, kern, cache=False) if kern in kernels.NEEDS_PREP else None
        if marks is not None:
            marks[0].record()
        for _ in range(k):
            kernels.spmv(A, x, kern, y=y, prepared=P)
        if marks is not None:
            marks[1].record()
        return P

    def timed(kk, steps, warm):
        """Fixed kernel kk: prep + k SpMVs captured as one CUDA graph (launched like the
        Seer plan), plus an eager pass with events around the SpMVs for the split."""
        fixed_step(kk)
        cs = torch.cuda.Stream()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=cs):
            fixed_step(kk)
        for _ in range(warm):
            gr.replay()
            fixed_step(kk)
        torch.cuda.synchronize()
        tot, inner = [], []
        for _ in range(steps):
            flush.zero_()
            e0, e1 = ev(), ev()
            e0.record()
            gr.replay()
            e1.record()
            e1.synchronize()
            tot.append(e0.elapsed_time(e1) * 1e-3)
            flush.zero_()
            m0, m1 = ev(), ev()
            fixed_step(kk, (m0, m1))
            m1.synchronize()
            inner.append(m0.elapsed_time(m1) * 1e-3)
        del gr
        return tot, inner

    # ---------------------------------------------------------------- warmup + timed (value)
    # The step runs as ONE CUDA graph (seer.SeerPlan): select -> device-side SWITCH on the
    # chosen kernel -> its preprocessing -> k SpMVs; no host round trip inside the step.
    plan = seer.SeerPlan(model, A, x, y, k)
    o_eager, _ = seer_step(A, x, y)
    torch.cuda.synchronize()
    # our kernels per graph step: the chosen body (prep + k SpMVs), + the selection kernel
    # on a gathered-path plan (the known path is resolved at plan build)
    n0 = L.kp_launch_count()
    fixed_step(int(o_eager.kernel))
    torch.cuda.synchronize()
    launches_per_step = (L.kp_launch_count() - n0) + (1 if o_eager.path else 0)
    for _ in range(a.warmup):
        plan.launch()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    step_t = []
    for _ in range(a.steps):
        flush.zero_()
        e0, e1 = ev(), ev()
        e0.record()
        plan.launch()
        e1.record()
        e1.synchronize()
        step_t.append(e0.elapsed_time(e1) * 1e-3)
    launches = launches_per_step * a.steps
    torch.cuda.synchronize()
    total = sum(step_t)
    if world > 1:
        dist.barrier()
        tt = torch.tensor([total], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total = float(tt.item())
    outcome = plan.outcome()
    kern = int(outcome.kernel)
    assert kern == int(o_eager.kernel), "graph and host-dispatched selection disagree"
    value = world * a.steps * k * bytes_csr / total / 1e9
    # host-dispatched variant (selection read back, then launches) for comparison
    eager_t = []
    for _ in range(max(3, a.steps // 2)):
        flush.zero_()
        e0, e1 = ev(), ev()
        e0.record()
        seer_step(A, x, y)
        e1.record()
        e1.synchronize()
        eager_t.append(e0.elapsed_time(e1) * 1e-3)
    # dominant kernel: the chosen SpMV op timed alone on this stream (CUDA events)
    prepared = kernels.prepare(A, kern) if kern in kernels.NEEDS_PREP else None
    spmv_t = []
    for _ in range(a.steps):
        flush.zero_()
        m0, m1 = ev(), ev()
        m0.record()
        kernels.spmv(A, x, kern, y=y, prepared=prepared)
        m1.record()
        m1.synchronize()
        spmv_t.append(m0.elapsed_time(m1) * 1e-3)

    # ---------------------------------------------------------------- roofline of the chosen SpMV op
    peak, peak_src = _peak_hbm()
    ell_w = None
    if kern == kernels.ELL_TM:
        hdr = prepared.buf[:64].cpu().view(torch.int64)
        ell_w = int(min(int(hdr[3]), prepared.ell_cap))
    kbytes = A.byte_model(kern, ell_w)
    per_launch = statistics.mean(spmv_t)
    achieved = kbytes / per_launch / 1e9
    traffic = _traffic_from_profiles(a.workload, kernels.KERNELS[kern])

    # ---------------------------------------------------------------- e2e through the public API
    # stop polling nvidia-smi before the e2e leg: its driver queries stall the pinned-copy
    # pipeline (measured 2.5 -> 2.9 ms/step); the samples cover the timed loop and the
    # kernel-only timings above
    clk = clocks.stop()
    e2e = _e2e(a, A, x, dtype, dev, model, k)
    if world > 1:  # whole-job e2e: every rank served its own matrix; slowest rank's step time
        tt = torch.tensor([e2e["ms_per_step"]], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e["ms_per_step"] = round(float(tt.item()), 4)
        e2e["value"] = round(world * k * bytes_csr / (e2e["ms_per_step"] * 1e-3) / 1e9, 2)
        e2e["h2d_bytes_per_step"] *= world
        e2e["d2h_bytes_per_step"] *= world

    # ---------------------------------------------------------------- per-kernel sweep
    sweep, geo, vs_best = None, None, None
    if not a.no_sweep and rank == 0:
        sweep = {}
        seer_mean = total / a.steps if world == 1 else sum(step_t) / a.steps
        for kk in range(len(kernels.KERNELS)):
            tot, inner = timed(kk, max(3, a.steps // 2), 2)
            t_tot, t_sp = statistics.median(tot), statistics.median(inner) / k
            w = None
            if kk == kernels.ELL_TM:
                P = kernels.prepare(A, kk, cache=False)
                w = int(min(int(P.buf[:64].cpu().view(torch.int64)[3]), P.ell_cap))
            sweep[kernels.KERNELS[kk]] = {
                "total_us": round(t_tot * 1e6, 2), "spmv_us": round(t_sp * 1e6, 2),
                "prep_us": round((t_tot - t_sp * k) * 1e6, 2),
                "spmv_gbs": round(A.byte_model(kk, w) / t_sp / 1e9, 1),
                "spmv_frac_of_peak": round(A.byte_model(kk, w) / t_sp / 1e9 / peak, 3)}
        ratios = [sweep[n]["total_us"] * 1e-6 / seer_mean for n in kernels.KERNELS]
        geo = math.exp(sum(math.log(r) for r in ratios) / len(ratios))
        vs_best = min(ratios)

    # ---------------------------------------------------------------- CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = _cpu_baseline(A, x, k, model, bytes_csr, a.cpu_seconds)

    if rank == 0:
        line = {
            "metric": "Seer-selected SpMV GB/s (% HBM roofline) and geomean speedup vs best fixed kernel",
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": round(total / a.steps * 1e3, 4), "higher_is_better": True, "scaling": "weak",
            "gflops": round(world * a.steps * k * 2 * Z / total / 1e9, 2),
            "vs_baseline": None, "dtype": "f32" if dtype == torch.float32 else "f64",
            "data": "synthetic (counter-hash generated on device)",
            "config": {"workload": a.workload, "desc": desc, "rows": R, "cols": C, "nnz": Z, "iterations": k,
                       "offsets": str(A.row_offsets.dtype).replace("torch.", ""), "l2": "flushed (512 MB write "
                       "between steps; matrix > L2)", "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                       "model": model_src, "byte_model": "nnz*(4+sv)+(R+1)*so+C*sv+R*sv"},
            "seer": {"kernel": kernels.KERNELS[kern], "path": "gathered" if outcome.path else "known",
                     "features": [outcome.max_d, outcome.min_d, outcome.mean_d, outcome.var_d] if outcome.path else None,
                     "step_us_median": round(statistics.median(step_t) * 1e6, 2),
                     "dispatch": ("one CUDA graph (kp_seer_plan): known path resolved on the device at plan "
                                  "build (PAPER.md:141 zero overhead), graph = chosen body" if not outcome.path else
                                  "one CUDA graph (kp_seer_plan): feature pass + gathered tree -> device-side SWITCH"),
                     "host_dispatched_step_us_median": round(statistics.median(eager_t) * 1e6, 2),
                     "spmv_us_mean": round(per_launch * 1e6, 2)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": kernels.KERNELS[kern],
                         "algorithmic_bytes_per_launch": kbytes, "peak_source": peak_src},
            "e2e": e2e,
            "gpu_launches": int(launches),
            "geomean_speedup_vs_fixed": None if geo is None else round(geo, 3),
            "speedup_vs_best_fixed": None if vs_best is None else round(vs_best, 3),
            "sweep": sweep,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


DEVICE_KERNEL = {"Adaptive-CSR": "k_adaptive", "CSR,BM": "k_csr_bm", "CSR,MP": "k_csr_merge",
                 "CSR,WM": "k_csr_wm", "CSR,WO": "k_csr_merge", "CSR,TM": "k_csr_tm", "COO,WM": "k_coo_wm",
                 "ELL,TM": "k_ell_tm"}


def _traffic_from_profiles(workload, kernel_label):
    """DRAM read+write bytes per launch of the dominant kernel from the committed
    `ncu --set full` capture (profiles/traffic.json, written by tools/ncu_summary.py)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f).get(workload, {})
    except Exception:
        return None
    name = DEVICE_KERNEL.get(kernel_label, "")
    for k, v in d.items():
        if k.split("<")[0] == name:
            return v
    return None


def _e2e(a, A, x, dtype, dev, model, k):
    """Public-API end to end: pinned host CSR + x -> H2D -> Seer plan -> y D2H, every step.

    The step's inputs live in ONE pinned host buffer (offsets, cols, vals, x at 256-byte
    aligned offsets) copied with one H2D; the device CSR / x are views of one staging
    buffer.  Served as a two-deep pipeline, the way a serving loop would: step i+1's inputs
    stream over PCIe on a copy stream into the other staging set while step i's plan runs
    and its y returns, so the step rate is bound by the H2D link (~55 GB/s measured), not by
    H2D + compute + D2H in series.  Each step still copies ALL of its inputs and reads back
    its result inside the timed region."""
    import torch
    from paper_2403_17017_b200 import seer
    from paper_2403_17017_b200.device import DeviceCSR
    parts = [A.row_offsets, A.col_indices, A.values, x]
    offs, o = [], 0
    for t in parts:
        offs.append(o)
        o += (t.numel() * t.element_size() + 255) // 256 * 256
    h_in = torch.empty(o, dtype=torch.uint8, pin_memory=True)
    for t, at in zip(parts, offs):
        nb = t.numel() * t.element_size()
        h_in[at:at + nb].copy_(t.contiguous().view(torch.uint8).reshape(-1).cpu())
    h_y = [torch.empty(A.n_rows, dtype=dtype, pin_memory=True) for _ in range(2)]
    sets = []
    for _ in range(2):
        d_in = torch.empty(o, dtype=torch.uint8, device=dev)
        views = [d_in[at:at + t.numel() * t.element_size()].view(t.dtype) for t, at in zip(parts, offs)]
        d_y = torch.empty(A.n_rows, dtype=dtype, device=dev)
        B = DeviceCSR(A.n_rows, A.n_cols, views[0], views[1], views[2])  # views the staging buffer
        sets.append((d_in, d_y, seer.SeerPlan(model, B, views[3], d_y, k)))
    bi = int(sum(t.numel() * t.element_size() for t in parts))
    bo = h_y[0].numel() * h_y[0].element_size()
    copy = torch.cuda.Stream(device=dev)
    comp = torch.cuda.current_stream()
    freed = [torch.cuda.Event(), torch.cuda.Event()]  # plan on set s finished reading its inputs
    landed = [torch.cuda.Event(), torch.cuda.Event()]
    for ev_ in freed:
        ev_.record(comp)

    def step(i):
        s = i % 2
        d_in, d_y, plan = sets[s]
        copy.wait_event(freed[s])
        with torch.cuda.stream(copy):
            d_in.copy_(h_in, non_blocking=True)
        landed[s].record(copy)
        comp.wait_event(landed[s])
        plan.launch(comp)
        h_y[s].copy_(d_y, non_blocking=True)
        freed[s].record(comp)

    for i in range(max(2, a.warmup)):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(4, a.steps // 2)
    e0.record(comp)
    copy.wait_event(e0)
    for i in range(steps):
        step(i)
    comp.wait_stream(copy)
    e1.record(comp)
    e1.synchronize()
    t = e0.elapsed_time(e1) * 1e-3 / steps
    bytes_csr = csr_bytes(A.n_rows, A.n_cols, A.nnz, A.values.element_size(), A.row_offsets.element_size())
    for _, _, plan in sets:
        plan.close()
    return {"value": round(k * bytes_csr / t / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": bi,
            "d2h_bytes_per_step": int(bo), "ms_per_step": round(t * 1e3, 4),
            "api": "pinned host CSR+x (one buffer) -> DeviceCSR staging views (copy stream, 2-deep) -> "
                   "seer.SeerPlan.launch (kp_seer_plan C-ABI) -> y to pinned host"}


def _cpu_baseline(A, x, k, model, bytes_csr, seconds):
    """Oracle port on this host: compiled reference length_stats (oracle/_ref) +
    restated epilogue/predict + OpenMP CPU SpMV, looped for ~``seconds``."""
    import numpy as np
    from oracle import oracle as orc
    off32, col, val = A.to_host()
    xh = x.cpu().numpy()
    off64 = off32.astype(np.int64)
    core = orc.ref_core()
    mdict = {n: t.to_dict() for n, t in (("selector", model.selector_tree), ("known", model.known_tree),
                                          ("gathered", model.gathered_tree))}

    def one():
        if core is not None:
            lo, hi, s1, s2 = core.length_stats(off64)
        else:
            lo, hi, s1, s2 = orc.length_stats(off64)
        f = orc.features_epilogue(lo, hi, s1, s2, A.n_rows, A.n_cols)
        kern, _ = orc.infer(mdict, A.n_rows, A.n_cols, A.nnz, k, f)
        for _ in range(k):
            orc.spmv_native(off32, col, val, xh)
        return kern

    one()
    t0 = time.perf_counter()
    reps = 0
    while True:
        one()
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds or reps >= 10000:
            break
    return {"value": round(reps * k * bytes_csr / el / 1e9, 3), "unit": "GB/s", "cores": orc.threads(),
            "kind": "port", "sample": f"{reps} full pipelines (features via "
            f"{'compiled reference _core' if core else 'oracle C'} + predict + {k} OpenMP SpMV) on the same matrix, "
            f"{el:.1f} s", "ms_per_step": round(el / reps * 1e3, 3)}


# ------------------------------------------------------------------------ reference arm
def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    k_default, dt_name, desc = CFG[a.workload]
    k = a.iters or k_default
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    m = _make_matrix(a.workload, dev)  # generation only (torch); nothing of ours computes below
    import numpy as np
    from oracle import oracle as orc
    off64, col64, val64 = m.numpy()
    dtype = np.float32 if dt_name == "float32" else np.float64
    off32 = off64.astype(np.int32) if m.nnz < 2**31 - 1 else off64
    col, val = col64.astype(np.int32), val64.astype(dtype)
    xh = (np.random.default_rng(1234).uniform(-1, 1, m.n_cols)).astype(dtype)
    sv = np.dtype(dtype).itemsize
    bytes_csr = csr_bytes(m.n_rows, m.n_cols, m.nnz, sv, off32.itemsize)
    model, _ = _load_model()
    mdict = {n: t.to_dict() for n, t in (("selector", model.selector_tree), ("known", model.known_tree),
                                          ("gathered", model.gathered_tree))}
    core = orc.ref_core()

    def step():
        lo, hi, s1, s2 = (core.length_stats(off64) if core is not None else orc.length_stats(off64))
        f = orc.features_epilogue(lo, hi, s1, s2, m.n_rows, m.n_cols)
        orc.infer(mdict, m.n_rows, m.n_cols, m.nnz, k, f)
        for _ in range(k):
            orc.spmv_native(off32, col, val, xh)

    for _ in range(a.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        step()
    el = time.perf_counter() - t0
    v = a.steps * k * bytes_csr / el / 1e9
    print(json.dumps({
        "impl": "reference",
        "metric": "Seer-selected SpMV GB/s (% HBM roofline) and geomean speedup vs best fixed kernel",
        "value": round(v, 3), "unit": "GB/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(el / a.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32" if dtype == np.float32 else "f64",
        "data": "synthetic (counter-hash generated)",
        "config": {"workload": a.workload, "desc": desc, "rows": m.n_rows, "cols": m.n_cols, "nnz": m.nnz,
                   "iterations": k},
        "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": orc.threads(), "kind": "port",
                         "sample": f"{a.steps} full pipelines: features via "
                                   f"{'compiled reference _core (oracle/_ref)' if core else 'oracle C restatement'}"
                                   f", restated predict, {k} OpenMP CPU SpMV (the reference has no SpMV)"},
        "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------------ C5: row-sharded
def run_sharded(a):
    """BASELINE configs[4]: the matrix is row-sharded over the ranks (nnz-balanced, K14),
    x replicated in the rank-padded layout, y local; each iteration's y slices are
    all-gathered in place over NVLink (NCCL) into the next x.  Selection = global
    features from the ranks' K1 partials (one 32-byte all-gather).  One step = the
    chosen kernel's preprocessing + k iterations; total work fixed as N grows (strong)."""
    import torch
    import torch.distributed as dist
    from paper_2403_17017_b200 import _lib, dist as kdist, gen, kernels

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:  # a 1-rank group so the fused exchange (symmetric memory) runs the N-rank code path
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    L = _lib.load()
    k_default, dt_name, desc = CFG["C5"]
    k = a.iters or k_default
    dtype = getattr(torch, dt_name)
    t0 = time.time()
    m = gen.config("C5", device=dev)  # every rank generates the same global matrix (counter hash)
    R, C, Z = m.n_rows, m.n_cols, m.nnz
    A, plan, _ = kdist.shard_device(m.row_offsets, m.col_indices, m.values, C, rank, world, dtype)
    del m
    torch.cuda.empty_cache()
    t_gen = time.time() - t0
    model, model_src = _load_model()
    run = kdist.ShardedSeer(model, A, plan, k, R, C, Z, exchange=a.exchange)
    kern = run.kernel
    x0 = torch.full((world * plan.r_max,), 1.0 / R, dtype=dtype, device=dev)
    sv, so = 4 if dtype == torch.float32 else 8, 4
    bytes_csr = csr_bytes(R, C, Z, sv, so)
    for _ in range(a.warmup):
        run.step(x0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    n0 = L.kp_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        run.step(x0)
    e1.record()
    e1.synchronize()
    launches = L.kp_launch_count() - n0
    total = e0.elapsed_time(e1) * 1e-3
    if world > 1:
        dist.barrier()
        tt = torch.tensor([total], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total = float(tt.item())
    # this rank's SpMV alone (dominant kernel) for the roofline
    P = kernels.prepare(A, kern) if kern in kernels.NEEDS_PREP else None
    ys = torch.empty(plan.local_rows, dtype=dtype, device=dev)
    ts = []
    for _ in range(5):
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record()
        kernels.spmv(A, run.bufs[0], kern, y=ys, prepared=P)
        m1.record()
        m1.synchronize()
        ts.append(m0.elapsed_time(m1) * 1e-3)
    clk = clocks.stop()
    peak, peak_src = _peak_hbm()
    kb = A.byte_model(kern, None if kern != kernels.ELL_TM else int(min(int(P.buf[:64].cpu().view(torch.int64)[3]), P.ell_cap)))
    per = statistics.median(ts)
    value = a.steps * k * bytes_csr / total / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": "Seer-selected SpMV GB/s (% HBM roofline) and geomean speedup vs best fixed kernel",
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": round(total / a.steps * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "gflops": round(a.steps * k * 2 * Z / total / 1e9, 2),
            "vs_baseline": None, "dtype": "f32" if dtype == torch.float32 else "f64",
            "data": "synthetic (counter-hash R-MAT generated on device)",
            "config": {"workload": "C5", "desc": desc, "rows": R, "cols": C, "nnz": Z, "iterations": k,
                       "parallelism": f"row-sharded x{world} (nnz-balanced, NCCL all-gather of y)",
                       "l2": "inputs larger than L2 (A: %.1f GB)" % (bytes_csr / 1e9), "model": model_src,
                       "byte_model": "nnz*(4+sv)+(R+1)*so+C*sv+R*sv per iteration, x counted once",
                       "generation_s": round(t_gen, 1)},
            "seer": {"kernel": kernels.KERNELS[kern], "path": "gathered" if run.outcome.path else "known",
                     "dispatch": "global selection from the ranks' K1 partials at setup (device)",
                     "exchange": ("fused: SpMV epilogue stores y into every rank's next x over NVLink "
                                  "(symmetric memory, kp_spmv_bcast) + device barrier" if run.exchange == "fused"
                                  else "NCCL in-place all-gather of y after each SpMV")},
            "roofline": {"bound": "hbm", "achieved": round(kb / per / 1e9, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(kb / per / 1e9 / peak, 4), "traffic": None, "kernel": kernels.KERNELS[kern],
                         "algorithmic_bytes_per_launch": kb, "peak_source": peak_src,
                         "note": "rank 0's local SpMV"},
            "e2e": None, "gpu_launches": int(launches), "cpu_baseline": None, "clocks": clk,
        }), flush=True)
    dist.destroy_process_group()


def main():
    a = _args()
    if a.impl == "reference":
        run_reference(a)
    elif a.workload == "C5":
        run_sharded(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
