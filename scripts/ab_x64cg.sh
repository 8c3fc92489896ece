# A/B: fp64 x gathers L2-only (.cg) vs through L1, every kernel on fp64 inputs
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_orig.so
for r in 1 2; do
for v in cur x64cg; do
  cp build_ab/libkpb200_$v.so $L
  echo "== $v rep $r"
  timeout 900 python tools/kbench.py --mats C4,C2d,band27d,pld --kernels 0,1,2,3,4,5,6,7 --reps 10 2>&1 | grep -v "^$"
done; done
cp build_ab/libkpb200_orig.so $L
