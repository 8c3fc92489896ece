# C5 with vertex reordering (default) vs --no-reorder, and the dist tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -2
for flag in "" "--no-reorder"; do
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 $flag > gpurun_out/c5_ro.json 2> gpurun_out/c5_ro.err; echo "rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/c5_ro.json').read().strip().splitlines()[-1]); print('C5 $flag', d['comm']['col_slices'], d['value'], d['ms_per_step'], d['roofline']['ms'], d['roofline']['unblocked_ms'], d['parity'], d['e2e']['value'], d['config']['reorder'], d['config']['setup_s'])"
cp gpurun_out/c5_ro.json "gpurun_out/c5_ro_${flag:-default}.json"
done
