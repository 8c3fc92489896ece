for cfg in "4 8" "32 8" "32 16" "32 32" "64 32"; do
  set -- $cfg
  echo "== mean $1 thread $2" >> gpurun_out/ab_bm.txt
  KP_BM_TINY_MEAN=$1 KP_BM_THREAD=$2 timeout 600 python tools/kbench.py --mats C1,C2,C3,band27,road,u1m,pl,rmat15,st43,const32 --kernels 1 --reps 10 >> gpurun_out/ab_bm.txt 2>&1
done
