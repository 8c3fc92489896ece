#!/bin/bash
# ncu --set full of kernel regex $K on kbench matrix $M kernel index $KI -> gpurun_out/full_$TAG.ncu-rep
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-3} -c 1 -o gpurun_out/full_$TAG -f \
  python tools/kbench.py --mats $M --kernels $KI --reps 4 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu $TAG rc=$?"
