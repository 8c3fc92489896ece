timeout 300 python -m pytest tests/test_gpu_emitted.py -x -q > gpurun_out/emit_test.log 2>&1
for c in unset 25 44 58 72 100; do
  if [ $c = unset ]; then unset KP_MERGE_CARVE; else export KP_MERGE_CARVE=$c; fi
  echo "== carve $c" >> gpurun_out/carve.txt
  timeout 300 python tools/kbench.py --mats C2,C4,band27,C2d,pl --kernels 2,4 --reps 10 >> gpurun_out/carve.txt 2>&1
done
