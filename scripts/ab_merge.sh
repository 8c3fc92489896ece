# A/B of merge-kernel library builds: parity (v2 variants) + kbench on merge kernels
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_cur.so
O=gpurun_out/ab_merge.txt
cp build_ab/libkpb200_v2.so $L
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_dist.py -x -q > gpurun_out/ab_merge_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ab_merge_tests.log
for r in 1 2; do
for v in ${VARIANTS:-old v2 v2m4}; do
  for c in ${CARVES:-unset}; do
    cp build_ab/libkpb200_$v.so $L
    if [ $c = unset ]; then unset KP_MERGE_CARVE; else export KP_MERGE_CARVE=$c; fi
    echo "== $v carve $c rep $r" >> $O
    timeout 300 python tools/kbench.py --mats ${MATS:-C2,C4,band27,C2d,pl,C1,u1m} --kernels 2,4 --reps 10 >> $O 2>&1
  done
done; done
unset KP_MERGE_CARVE
cp build_ab/libkpb200_cur.so $L
