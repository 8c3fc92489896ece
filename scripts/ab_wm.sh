timeout 600 python -m pytest tests/test_gpu_long_rows.py -x -q > gpurun_out/long_tests.log 2>&1; echo "rc=$?" >> gpurun_out/long_tests.log
for t in 64 32 16 8; do
  echo "== M $t" >> gpurun_out/ab_wm.txt
  KP_WM_LONG_MULT=$t timeout 600 python tools/kbench.py --mats C1,C2,C3,band27,u1m,band300,road,pl,st43,rmat15 --kernels 3 --reps 10 >> gpurun_out/ab_wm.txt 2>&1
done
