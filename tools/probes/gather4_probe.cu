// TMA tile::gather4 vs LSU gathers for SpMV's x[col] (C2's real columns), no reduction.
// x is viewed as a 2-D tensor of 8-float rows (one 32-byte sector per row); one
// cp.async.bulk.tensor.2d...tile::gather4 fetches the 4 rows holding 4 gathered elements
// into shared memory, completing on an mbarrier; the consumer reads element c % 8 of row
// c / 8.  Question: does the TMA path sustain more random sectors per SM-clock than the
// L1TEX gather path (~1 / clk / SM, profiles/gather_floor_r01.txt)?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC gather4_probe.cu -o gather4_probe.so -lcuda
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int ldc(const int *p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// warp tile = 256 elements (8 per lane, striped); lane l issues 2 gather4 for its elements
// t = 0..7 (rows col/8 of elements l + 32t), i.e. 64 gather4 per tile, 8 KB of rows; two
// tile buffers per warp (the next tile's gathers fly while this one is consumed).
constexpr int kWarps = 8;
__global__ void __launch_bounds__(kWarps * 32, 1) k_g4(const __grid_constant__ CUtensorMap tmap, const int *__restrict__ col,
                                                    float *__restrict__ out, int64_t n) {
    extern __shared__ __align__(128) float sm[];  // [warp][2][256 rows][8]
    __shared__ __align__(8) uint64_t bar[kWarps][2];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *buf = sm + (size_t)w * 2 * 256 * 8;
    if (lane == 0) {
        for (int b = 0; b < 2; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][b])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t tiles = n / 256, nw = (int64_t)gridDim.x * kWarps;
    float acc = 0.f;
    int it = 0;
    auto issue = [&](int64_t t, int b) {
        int c[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = ldc(col + t * 256 + lane + 32 * i);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w][b])),
                         "r"(256 * 32) : "memory");
        __syncwarp();
#pragma unroll
        for (int g = 0; g < 2; ++g) {  // rows of elements lane + 32 (4g + 0..3) -> slots 4g..4g+3
            float *dst = buf + ((size_t)b * 256 + (size_t)(lane * 8 + g * 4)) * 8;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
                "l"(&tmap), "r"(0), "r"(c[4 * g] >> 3), "r"(c[4 * g + 1] >> 3), "r"(c[4 * g + 2] >> 3),
                "r"(c[4 * g + 3] >> 3), "r"(smem_u32(&bar[w][b]))
                : "memory");
        }
        return 0;
    };
    int64_t t = blockIdx.x * kWarps + w;
    int cc[2][8];
    if (t < tiles) {
#pragma unroll
        for (int i = 0; i < 8; ++i) cc[0][i] = ldc(col + t * 256 + lane + 32 * i) & 7;
        issue(t, 0);
    }
    for (; t < tiles; t += nw, ++it) {
        const int b = it & 1;
        const int64_t tn = t + nw;
        if (tn < tiles) {
#pragma unroll
            for (int i = 0; i < 8; ++i) cc[b ^ 1][i] = ldc(col + tn * 256 + lane + 32 * i) & 7;
            issue(tn, b ^ 1);
        }
        // wait for this tile's rows
        const uint32_t ph = (uint32_t)((it >> 1) & 1);
        asm volatile(
            "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                smem_u32(&bar[w][b])),
            "r"(ph)
            : "memory");
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int slot = lane * 8 + (i / 4) * 4 + (i % 4);
            acc += buf[((size_t)b * 256 + slot) * 8 + cc[b][i]];
        }
        __syncwarp();
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int g4_run(const void *col, const void *x, int64_t n_cols, void *out, int64_t n, int grid, void *stream) {
    CUtensorMap m;
    cuuint64_t dims[2] = {8, (cuuint64_t)(n_cols / 8)};
    cuuint64_t strides[1] = {8 * sizeof(float)};
    cuuint32_t box[2] = {8, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(x), dims, strides, box,
                                        es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 1000 + (int)r;
    const int smem = kWarps * 2 * 256 * 8 * sizeof(float);
    cudaFuncSetAttribute(k_g4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_g4<<<grid, kWarps * 32, smem, (cudaStream_t)stream>>>(m, (const int *)col, (float *)out, n);
    return (int)cudaGetLastError();
}
