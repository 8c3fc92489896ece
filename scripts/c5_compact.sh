# compressed-row column blocks: dist GPU tests, per-rank slice sweep, C5 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -3
timeout 1500 python tools/shard_scaling.py --parts 1,8 --col-slices 2,3,4,6,auto > gpurun_out/shard_compact.txt 2>&1; grep -v "^{" gpurun_out/shard_compact.txt | cut -c1-110 | tail -12
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 > gpurun_out/c5_compact.json 2> gpurun_out/c5_compact.err
python -c "import json; d=json.loads(open('gpurun_out/c5_compact.json').read().strip().splitlines()[-1]); print('C5', d['comm']['col_slices'], d['value'], d['ms_per_step'], d['roofline']['ms'], d['roofline']['unblocked_ms'], d['parity'], d['e2e']['value'], d['e2e']['serial_value'])"
