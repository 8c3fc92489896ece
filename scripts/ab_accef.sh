# A/B: L2 evict-first on the accumulator reads (accef) and the single-destination y stores (accyef)
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_orig.so
for r in 1 2; do
for v in cur accef accyef; do
  cp build_ab/libkpb200_$v.so $L
  echo "== $v rep $r"
  timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', d['comm']['col_slices'], d['value'], d['ms_per_step'], d['roofline']['ms'], d['parity']['ok'])"
  timeout 900 python tools/shard_scaling.py --parts 8 --col-slices auto --reps 5 2>&1 | grep "^8 auto" | cut -c1-90
done; done
cp build_ab/libkpb200_orig.so $L
