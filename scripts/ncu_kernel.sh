#!/bin/bash
# ncu --set full of one kernel (regex KREGEX, skip SKIP launches) inside tools/kbench.py on
# matrix MATS with kernels KERNS; report -> gpurun_out/full_${TAG}.ncu-rep.  Plus a plain
# kbench timing pass first (no profiler) -> gpurun_out/kbench_${TAG}.txt
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 600 python tools/kbench.py --mats ${MATS:-C2} --kernels ${KERNS:-0,1,2,3,4,5,6,7} --reps 10 \
  > gpurun_out/kbench_${TAG}.txt 2>&1; echo "kbench rc=$?"
if [ -n "$KREGEX" ]; then
  for K in $KREGEX; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-3} -c 1 \
      -o gpurun_out/full_${TAG}_$K -f python tools/kbench.py --mats ${MATS:-C2} --kernels ${NCU_KERNS:-${KERNS:-2,6}} --reps 4 \
      > gpurun_out/ncu_${TAG}_$K.log 2>&1; echo "ncu $K rc=$?"
  done
fi
cat gpurun_out/kbench_${TAG}.txt
