# A/B: x gathers through L1 (cur, ld.global.nc), L1 no-allocate (xna), L2-only .cg (xcg)
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_orig.so
for r in 1 2; do
for v in cur xna xcg; do
  cp build_ab/libkpb200_$v.so $L
  echo "== $v rep $r"
  timeout 600 python tools/kbench.py --mats C2,C4,C3,band27,pl,C2d --kernels 2,5,7 --reps 10 2>&1 | grep CSR
done; done
cp build_ab/libkpb200_orig.so $L
