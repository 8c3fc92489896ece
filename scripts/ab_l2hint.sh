# A/B: L2 evict-first on streamed loads (ef), + evict-last on x gathers (efel), vs cur
L=paper_2403_17017_b200/libkpb200.so
cp $L build_ab/libkpb200_orig.so
for r in 1 2; do
for v in cur ef efel; do
  cp build_ab/libkpb200_$v.so $L
  echo "== $v rep $r"
  timeout 600 python tools/probes/colslice_probe.py --slices 3,4 2>&1 | grep -v "^rows\|bcast-kernel full" | grep "CSR,WO"
  timeout 600 python tools/kbench.py --mats C2,C4,C3,band27,pl --kernels 1,2 --reps 10 2>&1 | grep CSR
  timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5 auto', d['comm']['col_slices'], d['value'], d['ms_per_step'], d['roofline']['ms'], d['roofline']['unblocked_ms'], d['parity']['ok'])"
done; done
cp build_ab/libkpb200_orig.so $L
