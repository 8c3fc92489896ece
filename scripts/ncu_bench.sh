#!/bin/bash
# Launch list of OUR kernels in the bench command (cold-cache serialised per-launch times;
# kernels inside the conditional-graph plan are not profilable by ncu, so the list covers
# the host-dispatched step, the dominant-kernel loop and the sweep) + one `ncu --set full`
# capture of the dominant SpMV kernel.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
W=${WORKLOAD:-C2}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_" -c ${COUNT:-300} --csv --log-file gpurun_out/launches_$W.csv \
  python bench.py --workload $W --steps 3 --warmup 1 --no-cpu > gpurun_out/ncu_bench_$W.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_csr_merge} -s ${SKIP:-4} -c 1 \
  -o gpurun_out/full_$W -f python bench.py --workload $W --steps 3 --warmup 1 --no-sweep --no-cpu \
  > gpurun_out/ncu_full_$W.log 2>&1; echo "full rc=$?"
