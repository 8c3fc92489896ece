#!/bin/bash
# Launch list of the bench command (cold-cache serialised per-launch times) + one
# `ncu --set full` capture of the dominant SpMV kernel; outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
W=${WORKLOAD:-C2}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_$W.csv python bench.py --workload $W --steps 3 --warmup 1 --no-sweep --no-cpu \
  > gpurun_out/ncu_bench_$W.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_csr_merge} -s ${SKIP:-4} -c 1 \
  -o gpurun_out/full_$W -f python bench.py --workload $W --steps 3 --warmup 1 --no-sweep --no-cpu \
  > gpurun_out/ncu_full_$W.log 2>&1; echo "full rc=$?"
ls -la gpurun_out/ | grep -E "launches|full_"
