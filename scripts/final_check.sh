timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
time timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
time timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
for spec in "C2 4 k_csr_merge" "C4 4 k_csr_merge" "C3 7 k_ell_tm"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 --launch-skip 2 --launch-count 1 \
     -f -o gpurun_out/final_$1_$3 python tools/ncu_one.py $1 $2 > gpurun_out/ncu_final_$1.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(csr|coo|ell|ad|prep|carry|row|seer|tree|wave|emitted|long|set|unpack)" -c 200 --csv \
   --log-file gpurun_out/launches_C2_final.csv python bench.py --steps 3 --warmup 3 --no-configs --no-cpu > gpurun_out/ncu_bench.log 2>&1
