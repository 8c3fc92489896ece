// kp_internal.cuh -- shared device helpers for libkpb200 (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/kernelpick_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libkpb200 is written for sm_100a (B200) only"
#endif

namespace kp {

constexpr int kNumSMs = 148;  // B200; launch code queries the device at runtime anyway

extern unsigned long long g_launches;  // kp_launch_count()

#define KP_CUDA_TRY(expr)                                   \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return KP_ECUDA;             \
    } while (0)

#define KP_LAUNCHED()                                       \
    do {                                                    \
        ++::kp::g_launches;                                 \
        if (cudaPeekAtLastError() != cudaSuccess) {         \
            cudaGetLastError();                             \
            return KP_ECUDA;                                \
        }                                                   \
    } while (0)

int num_sms();

// NVTX ranges around every C-ABI entry (domain "kernelpick"): a profiler (nsys, ncu
// --nvtx) sees each Seer stage -- selection, feature pass, preparation, SpMV, plan
// build/launch -- by name.  Header-only NVTX3; without an attached tool each range is a
// null-pointer check.
struct NvtxRange {
    explicit NvtxRange(const char *name);
    ~NvtxRange();
};
#define KP_NVTX(name) ::kp::NvtxRange _kp_nvtx_range(name)
const char *kernel_label(int32_t kernel);

// Trees by value for the plan's selection kernel (kp_reduce.cu, used by kp_graph.cu).
constexpr int kParamTreeNodes = 127;  // depth <= 6
struct ParamTrees {
    int32_t n[3];
    int32_t pad;
    kp_tree_node node[3][kParamTreeNodes];
};

int plan_trees_load(const void *d_sel, const void *d_known, const void *d_gath, ParamTrees *T);
// true iff T (loaded by plan_trees_load) equals the trees compiled in from include/kp_seer_trees.h
bool emitted_trees_match(const ParamTrees &T);
int launch_plan_select(const void *d_off, int32_t off_type, int64_t n_rows, int64_t n_cols, int64_t nnz,
                       int64_t iters, const ParamTrees &T, bool emitted, kp_outcome *d_out, void *d_ws,
                       cudaGraphConditionalHandle h, cudaStream_t s);

// ----------------------------------------------------------------- load helpers

// Streamed (read-once) data: non-coherent path, do not allocate in L1 so the x
// gathers keep the L1.  KP_STREAM_L2_EF (A/B): also mark the lines evict-first in L2 so
// the streams do not push the x gathers' lines out.
#ifndef KP_STREAM_L2_EF
#define KP_STREAM_L2_EF 0
#endif
#if KP_STREAM_L2_EF
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t *p) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(l2_evict_first_policy()));
    return v;
}
__device__ __forceinline__ float ld_stream(const float *p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(l2_evict_first_policy()));
    return v;
}
__device__ __forceinline__ double ld_stream(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(l2_evict_first_policy()));
    return v;
}
#else
__device__ __forceinline__ int32_t ld_stream(const int32_t *p) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream(const float *p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_stream(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
#endif
__device__ __forceinline__ int64_t ld_stream(const int64_t *p) {
    int64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.s64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int4 ld_stream4(const int4 *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ longlong2 ld_stream2ll(const longlong2 *p) {
    longlong2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.s64 {%0,%1}, [%2];"
                 : "=l"(r.x), "=l"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// x gathers: read-only path, L1-allocating (reuse across rows / lanes).
#ifndef KP_X_L2_EL
#define KP_X_L2_EL 0
#endif
#if KP_X_L2_EL  // A/B: x gathers marked evict-last in L2
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ float ld_x(const float *p) {
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(l2_evict_last_policy()));
    return v;
}
__device__ __forceinline__ double ld_x(const double *p) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(l2_evict_last_policy()));
    return v;
}
#elif defined(KP_X_MODE) && KP_X_MODE == 1  // A/B: x gathers not allocated in L1
__device__ __forceinline__ float ld_x(const float *p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_x(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
#elif defined(KP_X_MODE) && KP_X_MODE == 2  // A/B: x gathers cached in L2 only (.cg)
__device__ __forceinline__ float ld_x(const float *p) { return __ldcg(p); }
__device__ __forceinline__ double ld_x(const double *p) { return __ldcg(p); }
#elif defined(KP_X_CG_F64) && KP_X_CG_F64  // fp64 gathers L2-only (.cg), fp32 through L1
__device__ __forceinline__ float ld_x(const float *p) { return __ldg(p); }
__device__ __forceinline__ double ld_x(const double *p) { return __ldcg(p); }
#else
template <typename T>
__device__ __forceinline__ T ld_x(const T *p) { return __ldg(p); }
#endif

// ----------------------------------------------------------------- warp helpers
template <int G, typename T>
__device__ __forceinline__ T group_sum(T v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Offsets: widen to int64 for index arithmetic.
template <typename O>
__device__ __forceinline__ int64_t ldo(const O *p) { return (int64_t)__ldg(p); }

// ----------------------------------------------------------------- mbarrier / bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 1-D TMA bulk copy global -> shared (SASS UBLKCP), completion on an mbarrier.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

}  // namespace kp
