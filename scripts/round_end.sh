# round-end validation on the final build: GPU tests, smoke, default bench (+ reference arm), C5 at N = 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log; tail -2 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
python - <<'PY'
import json
for f in ("bench", "bench_ref", "bench_c5"):
    d = json.loads(open(f"gpurun_out/{f}.log").read().strip().splitlines()[-1])
    print(f, d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"),
          d.get("clocks"), {k: v.get("speedup_vs_best_fixed") for k, v in (d.get("per_config") or {}).items()})
PY
