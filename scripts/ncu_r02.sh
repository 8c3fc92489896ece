# r02 ncu evidence for the final kernels: full captures (C2 WO, C4 WO, C2 TM with its long-row tail) + bench launch list
for spec in "C2 4 k_csr_merge" "C4 4 k_csr_merge" "C2 5 k_long_rows"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 --launch-skip 2 --launch-count 1 \
     -f -o gpurun_out/full_$1_k$2_r02 python tools/ncu_one.py $1 $2 > gpurun_out/ncu_$1_$2.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(csr|coo|ell|ad|prep|carry|row|seer|tree|wave|emitted|long|set)" -c 200 --csv \
   --log-file gpurun_out/launches_C2_r02.csv python bench.py --steps 3 --warmup 3 --no-configs --no-cpu > gpurun_out/ncu_bench.log 2>&1
