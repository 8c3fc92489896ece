# persistent merge wave vs residency A/B (kbench), then SWITCH-body overhead probe
for w in 0 3552 2368 4736; do
  echo "== wave $w" >> gpurun_out/wave.txt
  timeout 300 python tools/kbench.py --mats C2,C4,band27,C2d --kernels 2,4 --reps 10 --wave-warps $w >> gpurun_out/wave.txt 2>&1
done
echo "== wave 2368 carve 72" >> gpurun_out/wave.txt
KP_MERGE_CARVE=72 timeout 300 python tools/kbench.py --mats C2,C4,band27,C2d --kernels 2,4 --reps 10 --wave-warps 3552 >> gpurun_out/wave.txt 2>&1
timeout 600 python tools/body_overhead.py > gpurun_out/body_overhead.jsonl 2> gpurun_out/body_overhead.err
