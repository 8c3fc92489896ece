# k_csr_bm_short trailing barrier (race fix): cost on the short-row inputs, then racecheck
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_orig.so
for r in 1 2; do
for v in cur bmfix; do
  cp build_ab/libkpb200_$v.so $L
  echo "== $v rep $r"
  timeout 600 python tools/kbench.py --mats C2,road,u1m,rmat15,st43 --kernels 1 --reps 10 2>&1 | grep CSR
done; done
cp build_ab/libkpb200_orig.so $L
mkdir -p gpurun_out/san
KP_WAVE_WARPS=7 timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_kernels.py > gpurun_out/san/racecheck.txt 2>&1; echo "exit=$?" >> gpurun_out/san/racecheck.txt
grep -E "SUMMARY|all ok|exit=" gpurun_out/san/racecheck.txt
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_long_rows.py -q -x 2>&1 | tail -1
