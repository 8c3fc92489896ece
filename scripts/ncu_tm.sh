for spec in "band300 5 k_csr_tm" "band300 5 k_long_rows" "C2 5 k_long_rows"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 --launch-skip 2 --launch-count 1 \
     -f -o gpurun_out/full_$1_$3 python tools/ncu_one.py $1 $2 > gpurun_out/ncu_$1_$3.log 2>&1
done
