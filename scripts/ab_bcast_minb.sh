# A/B: fused-exchange (kB) fp32 merge kernel at 3 CTAs (cur) vs the compiler's allocation (b0)
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_orig.so
for v in cur b0; do
  cp build_ab/libkpb200_$v.so $L
  echo "== $v"
  timeout 600 python tools/probes/colslice_probe.py --slices 3 2>&1 | grep -v "^rows"
  KP_COL_SLICES=1 timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('S=1', d['value'], d['ms_per_step'], d['roofline']['ms'])"
  timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('auto', d['comm']['col_slices'], d['value'], d['ms_per_step'], d['roofline']['ms'], d['roofline']['unblocked_ms'], d['parity']['ok'])"
done
cp build_ab/libkpb200_orig.so $L
