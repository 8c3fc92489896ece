timeout 900 python -m pytest tests/test_gpu_long_rows.py tests/test_gpu_spmv.py tests/test_gpu_plan.py -x -q > gpurun_out/long_tests.log 2>&1; echo "rc=$?" >> gpurun_out/long_tests.log
timeout 400 python tools/kbench.py --mats C1,C2,C3,C4,band27,pl,rmat15 --kernels 3,5 --reps 10 > gpurun_out/kbench_long.txt 2>&1
