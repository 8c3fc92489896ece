# final C5 numbers with compressed-row blocks, the per-rank projection, GPU suite, sanitizers
mkdir -p gpurun_out
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 > gpurun_out/c5_final.json 2> gpurun_out/c5_final.err
python -c "import json; d=json.loads(open('gpurun_out/c5_final.json').read().strip().splitlines()[-1]); print('C5', d['comm']['col_slices'], d['value'], d['ms_per_step'], d['roofline']['ms'], d['roofline']['unblocked_ms'], d['parity']['ok'], d['e2e']['value'], d['e2e']['serial_value'], d['clocks'])"
timeout 1500 python tools/shard_scaling.py --parts 1,2,4,8 --col-slices 1,auto --out gpurun_out/shard_scaling_final.json > gpurun_out/shard_scaling_final.txt 2>&1; tail -1 gpurun_out/shard_scaling_final.txt
timeout 1500 python tools/shard_scaling.py --parts 1,8 --col-slices 2,3,4,6 > gpurun_out/shard_sweep_final.txt 2>&1; tail -1 gpurun_out/shard_sweep_final.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -1 gpurun_out/gputest.log
KP_WAVE_WARPS=7 bash scripts/sanitize.sh; for t in memcheck racecheck synccheck; do grep -E "ERROR SUMMARY|RACECHECK SUMMARY|exit=" gpurun_out/san/$t.txt | tail -2; done
