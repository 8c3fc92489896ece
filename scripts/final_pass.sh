#!/bin/bash
# Round-end measurement pass (one gpurun session): smoke + GPU tests, BASELINE configs
# C1-C5 through bench.py, per-kernel bandwidths, live Seer eval.  Outputs in gpurun_out/final/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/final
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
: > $O/bench_configs.jsonl
for w in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-5} --warmup 3 2> $O/bench_$w.err | tail -1 >> $O/bench_configs.jsonl
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 1200 python tools/kbench.py --out $O/kbench.json > $O/kbench.txt 2>&1
if [ -z "$NO_EVAL" ]; then
  timeout 2400 python tools/eval_seer.py --out $O/seer_live_eval.json > $O/eval.log 2>&1
fi
tail -2 $O/smoke.log; tail -2 $O/pytest_gpu.log; wc -l $O/bench_configs.jsonl; tail -3 $O/eval.log
