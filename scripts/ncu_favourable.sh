#!/bin/bash
# ncu launch metrics (duration, DRAM read/write) of every SpMV kernel on its favourable
# input (tools/kbench.py runs, 3 timed reps each) -> gpurun_out/ncu_fav_*.csv
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for M in band2k band4 band27 C3 band27d; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_(csr|coo|ell|adaptive)" --csv --log-file gpurun_out/ncu_fav_$M.csv \
    python tools/kbench.py --mats $M --reps 3 > gpurun_out/ncu_fav_$M.log 2>&1; echo "$M rc=$?"
done
