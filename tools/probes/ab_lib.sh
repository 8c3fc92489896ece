# A/B of library builds: copies build_ab/libkpb200_<v>.so in place, runs kbench, restores
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_orig.so
for v in ${VARIANTS:-cur}; do
  cp build_ab/libkpb200_$v.so $L
  echo "== $v"
  python tools/kbench.py --mats ${MATS:-C2,C4} --kernels ${KERNS:-4} --reps 10 2>&1 | grep -v "^#" | tail -16
done
cp build_ab/libkpb200_orig.so $L
