mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -2
for r in 1 2; do
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', d['comm']['col_slices'], d['value'], d['ms_per_step'], d['roofline']['ms'], d['parity']['ok'])"
done
