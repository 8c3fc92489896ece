// fp64 random-gather floor (C4): stream col (int32) + val (fp64) and gather x[col] (fp64)
// with the merge kernel's access shape (warp tiles of 256 items, 8 per lane, striped), no
// row reduction.  Separates C4's gather cost from the merge kernel's reduction cost.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC gather64_probe.cu -o gather64_probe.so
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ int ldc(const int *p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ldv(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

template <int kMinB>
__global__ void __launch_bounds__(256, kMinB) k_g64(const int *__restrict__ col, const double *__restrict__ val,
                                                   const double *__restrict__ x, double *__restrict__ out, int64_t n) {
    extern __shared__ double dyn[];
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * 8;
    double acc = 0.0;
    const int64_t tiles = n / 256;
    for (int64_t t = blockIdx.x * 8 + (threadIdx.x >> 5); t < tiles; t += nw) {
        const int64_t b = t * 256 + lane;
        int c[8];
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            c[i] = ldc(col + b + 32 * i);
            v[i] = ldv(val + b + 32 * i);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += v[i] * __ldg(x + c[i]);
    }
    if (acc == -1.0) dyn[threadIdx.x] = acc;
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int g64_run(int min_blocks, int smem, const void *col, const void *val, const void *x, void *out,
                       int64_t n, int grid, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    auto c = (const int *)col;
    auto v = (const double *)val;
    auto xx = (const double *)x;
    auto o = (double *)out;
    if (min_blocks == 2) {
        cudaFuncSetAttribute(k_g64<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_g64<2><<<grid, 256, smem, s>>>(c, v, xx, o, n);
    } else if (min_blocks == 3) {
        cudaFuncSetAttribute(k_g64<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_g64<3><<<grid, 256, smem, s>>>(c, v, xx, o, n);
    } else {
        cudaFuncSetAttribute(k_g64<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_g64<4><<<grid, 256, smem, s>>>(c, v, xx, o, n);
    }
    return (int)cudaGetLastError();
}
