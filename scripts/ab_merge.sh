# A/B of merge-kernel library builds: parity (first variant) + kbench on merge kernels
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_cur.so
O=gpurun_out/ab_merge.txt
V1=$(echo ${VARIANTS:-v2 v3} | awk '{print $NF}')
cp build_ab/libkpb200_$V1.so $L
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_dist.py tests/test_gpu_plan.py -x -q > gpurun_out/ab_merge_tests.log 2>&1
echo "tests ($V1) rc=$?" >> gpurun_out/ab_merge_tests.log
for r in 1 2; do
for v in ${VARIANTS:-v2 v3}; do
    cp build_ab/libkpb200_$v.so $L
    echo "== $v carve default rep $r" >> $O
    timeout 300 python tools/kbench.py --mats ${MATS:-C2,C4,band27,C2d,band27d,pl,C1,C3} --kernels 2,4 --reps 10 >> $O 2>&1
done; done
cp build_ab/libkpb200_cur.so $L
