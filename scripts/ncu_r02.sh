# r02 ncu evidence: full captures of the merge kernel (C2 WO, C4 WO) + the default bench launch list
set -x
for spec in "C2 4" "C4 4"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_csr_merge --launch-skip 2 --launch-count 1 \
     -f -o gpurun_out/full_$1_wo_r02 python tools/ncu_one.py $1 $2 > gpurun_out/ncu_$1.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C2_r02.csv \
   python bench.py --steps 2 --warmup 1 --no-configs --no-cpu --no-sweep > gpurun_out/ncu_bench.log 2>&1
