#!/bin/bash
# ncu --set full captures of selected (matrix, kernel) pairs; reports land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
cap() {  # name mats kernel regex
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$4 -s 2 -c 1 \
    -o gpurun_out/$1 -f python tools/kbench.py --mats $2 --kernels $3 --reps 1 > gpurun_out/$1.log 2>&1
  echo "$1 rc=$?"
}
for spec in $CAPS; do IFS=: read n m k r <<< "$spec"; cap $n $m $k $r; done
ls -la gpurun_out/*.ncu-rep
