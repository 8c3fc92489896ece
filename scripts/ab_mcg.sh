# A/B: fp64 merge-kernel gathers L2-only (.cg) vs through L1
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_orig.so
for r in 1 2; do
for v in cur mcg; do
  cp build_ab/libkpb200_$v.so $L
  echo "== $v rep $r"
  timeout 900 python tools/kbench.py --mats C4,C2d,band27d,pld,C3d,band2kd,C2 --kernels 2,4 --reps 10 2>&1 | grep CSR
done; done
cp build_ab/libkpb200_orig.so $L
