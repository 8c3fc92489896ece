# C5 with its end-to-end leg, the C5 reference arm, and the dist tests (incl. bench --gpus 2 control flow)
mkdir -p gpurun_out
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 > gpurun_out/c5_e2e.json 2> gpurun_out/c5_e2e.err; echo "c5 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/c5_e2e.json').read().strip().splitlines()[-1]); print('C5', d['value'], d['ms_per_step'], d['e2e'], d['parity']['ok'])"
tail -3 gpurun_out/c5_e2e.err
time timeout 900 python bench.py --impl reference --workload C5 --steps 3 --warmup 3 > gpurun_out/c5_ref.json 2> gpurun_out/c5_ref.err; echo "ref rc=$?"
tail -c 1500 gpurun_out/c5_ref.json; tail -3 gpurun_out/c5_ref.err
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -2
