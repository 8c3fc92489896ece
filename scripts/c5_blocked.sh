# column-blocked C5: dist GPU tests, the N = 1 bench line, and the per-rank projection
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/dist_tests.txt 2>&1; tail -3 gpurun_out/dist_tests.txt
timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 > gpurun_out/c5_blocked.json 2> gpurun_out/c5_blocked.err
python -c "import json; d=json.loads(open('gpurun_out/c5_blocked.json').read().strip().splitlines()[-1]); print('C5', d['comm']['col_slices'], d['value'], d['ms_per_step'], d['roofline'], d['parity'])"
timeout 1200 python tools/shard_scaling.py --parts 1,2,4,8 --col-slices 1,2,4,auto --out gpurun_out/shard_scaling_blocked.json > gpurun_out/shard_scaling_blocked.txt 2>&1; tail -25 gpurun_out/shard_scaling_blocked.txt
