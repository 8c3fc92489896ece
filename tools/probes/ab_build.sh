# Build an A/B variant of libkpb200.so into build_ab/libkpb200_<name>.so with extra nvcc flags.
#   tools/probes/ab_build.sh <name> "-DFOO -DBAR"
set -e
cd "$(dirname "$0")/../.."
N=$1; shift
D=build_ab/obj_$N
mkdir -p $D build_ab
C=${SRC:-paper_2403_17017_b200/csrc}
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden $*"
nvcc $F -fmad=false -c $C/kp_reduce.cu -o $D/kp_reduce.o &
for f in kp_spmv kp_graph kp_coo2csr kp_pack; do nvcc $F -Xcompiler -fopenmp -c $C/$f.cu -o $D/$f.o & done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC,-fopenmp -o build_ab/libkpb200_$N.so \
  $D/kp_reduce.o $D/kp_spmv.o $D/kp_graph.o $D/kp_coo2csr.o $D/kp_pack.o paper_2403_17017_b200/csrc/build/kp_mmio.o paper_2403_17017_b200/csrc/build/kp_watchdog.o paper_2403_17017_b200/csrc/build/kp_nvtx.o -lcudart -lgomp -ldl -lpthread
echo built build_ab/libkpb200_$N.so
