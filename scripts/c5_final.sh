# final C5 numbers (column blocking auto) + the full GPU suite
mkdir -p gpurun_out
for r in 1 2; do
timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 > gpurun_out/c5_final_$r.json 2> gpurun_out/c5_final_$r.err
python -c "import json; d=json.loads(open('gpurun_out/c5_final_$r.json').read().strip().splitlines()[-1]); print('C5', d['comm']['col_slices'], d['value'], d['ms_per_step'], d['roofline']['ms'], d['roofline']['unblocked_ms'], d['parity']['ok'], d['config']['setup_s'], d['clocks'])"
done
timeout 1200 python tools/shard_scaling.py --parts 1,2,4,8 --col-slices 1,auto --out gpurun_out/shard_scaling_final.json > gpurun_out/shard_scaling_final.txt 2>&1; tail -3 gpurun_out/shard_scaling_final.txt
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_final.txt 2>&1; tail -3 gpurun_out/gpu_tests_final.txt
