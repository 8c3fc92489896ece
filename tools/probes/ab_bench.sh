# A/B of library builds through bench.py (one JSON line per variant and repeat)
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_orig.so
for r in 1 2; do
for v in ${VARIANTS:-cur}; do
  cp build_ab/libkpb200_$v.so $L
  printf "%s " $v
  python bench.py --workload ${WL:-C2} --steps 3 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"
done; done
cp build_ab/libkpb200_orig.so $L
