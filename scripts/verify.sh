# full GPU parity, merge-kernel kbench, default bench line
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
timeout 300 python tools/kbench.py --mats ${MATS:-C2,C3,C4,band27,C2d,band27d,pl,C1} --kernels ${KERN:-2,4} --reps 10 > gpurun_out/kbench.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
