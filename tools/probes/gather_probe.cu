// Random-gather floor on B200: stream col (+ val) and gather x[col] with different load
// flavours, no row reduction (each thread keeps a running sum).  Separates the SpMV's
// gather cost from its segmented-reduction cost.  Built as a .so, driven by
// tools/probes/gather_probe.py on the real C2 column array.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC gather_probe.cu -o gather_probe.so
#include <cstdint>
#include <cuda_runtime.h>

template <int M>
__device__ __forceinline__ float gx(const float *p) {
    float v;
    if constexpr (M == 0) v = __ldg(p);
    else if constexpr (M == 1) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    else if constexpr (M == 2) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    else if constexpr (M == 3) asm volatile("ld.global.ca.f32 %0, [%1];" : "=f"(v) : "l"(p));
    else if constexpr (M == 4) asm volatile("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p));
    else v = (float)(uintptr_t)p;  // no gather
    return v;
}
__device__ __forceinline__ int ldc(const int *p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ldv(const float *p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// warp tiles of 256 items (8 per lane, striped), grid-stride over tiles
template <int M, bool kVal>
__global__ void __launch_bounds__(256) k_gather(const int *__restrict__ col, const float *__restrict__ val,
                                                const float *__restrict__ x, float *__restrict__ out, int64_t n) {
    extern __shared__ float dyn[];  // footprint only (L1 capacity experiments)
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * 8;
    float acc = 0.f;
    const int64_t tiles = n / 256;
    for (int64_t t = blockIdx.x * 8 + (threadIdx.x >> 5); t < tiles; t += nw) {
        const int64_t b = t * 256 + lane;
        int c[8];
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            c[i] = ldc(col + b + 32 * i);
            v[i] = kVal ? ldv(val + b + 32 * i) : 1.f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += v[i] * gx<M>(x + c[i]);
    }
    if (acc == -1.f) dyn[threadIdx.x] = acc;
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

static int g_smem = 0, g_carve = -1;
extern "C" void gp_config(int smem, int carve) { g_smem = smem; g_carve = carve; }
template <int M, bool kVal>
static void launch(const int *col, const float *val, const float *x, float *out, int64_t n, int grid, cudaStream_t s) {
    cudaFuncSetAttribute(k_gather<M, kVal>, cudaFuncAttributeMaxDynamicSharedMemorySize, g_smem);
    if (g_carve >= 0) cudaFuncSetAttribute(k_gather<M, kVal>, cudaFuncAttributePreferredSharedMemoryCarveout, g_carve);
    k_gather<M, kVal><<<grid, 256, g_smem, s>>>(col, val, x, out, n);
}

extern "C" int gp_run(int mode, int with_val, const void *col, const void *val, const void *x, void *out, int64_t n,
                      int grid, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    auto c = (const int *)col;
    auto v = (const float *)val;
    auto xx = (const float *)x;
    auto o = (float *)out;
#define GP(M)                                                   \
    if (mode == M) {                                            \
        if (with_val) launch<M, true>(c, v, xx, o, n, grid, s); \
        else launch<M, false>(c, v, xx, o, n, grid, s);         \
    }
    GP(0) GP(1) GP(2) GP(3) GP(4) GP(5)
#undef GP
    return (int)cudaGetLastError();
}
