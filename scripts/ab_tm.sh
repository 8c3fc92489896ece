for t in 256 128 64 32; do
  echo "== T $t" >> gpurun_out/ab_tm.txt
  KP_TM_LONG=$t timeout 600 python tools/kbench.py --mats C1,C2,C3,band27,const32,u1m,band300,road,pl,st43 --kernels 5 --reps 10 >> gpurun_out/ab_tm.txt 2>&1
done
