L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_cur.so
for v in ellprep1 ellprep8; do
  cp build_ab/libkpb200_$v.so $L
  echo "== $v" >> gpurun_out/ab_ell.txt
  timeout 600 python tools/kbench.py --mats const8big,C3,band27,const32,C2,road --kernels 7 --reps 5 >> gpurun_out/ab_ell.txt 2>&1
done
cp build_ab/libkpb200_ellprep8.so $L
timeout 600 python -m pytest tests/test_gpu_spmv.py -x -q -k "kernel_parity or ell" > gpurun_out/ell_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ell_tests.log
cp build_ab/libkpb200_cur.so $L
