# A/B of library builds on the feature pass (tools/k1_bench.py)
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_orig.so
for v in ${VARIANTS:-cur}; do
  cp build_ab/libkpb200_$v.so $L
  echo "== $v"
  python tools/k1_bench.py 2>&1 | tail -12
done
cp build_ab/libkpb200_orig.so $L
