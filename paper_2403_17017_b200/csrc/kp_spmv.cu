// kp_spmv.cu -- the SpMV kernel family Seer selects between (Table III
// order :311-318) and the preprocessing the cost model charges (
// PAPER.md:280).  sm_100a, CUDA cores + LSU / TMA-bulk; no tensor cores (SpMV is
// ~0.2 flop/B, far below the ridge).
//
//   id kernel          schedule                                         prep
//   0  Adaptive-CSR    row blocks: short rows staged in smem (stream),   K13 (flags+scan)
//                      long rows split into CTA pieces (vector-L)
//   1  CSR,BM          one CTA per row, block reduction                 -
//   2  CSR,MP          merge-path CTA tiles (Merrill & Garland), smem    K10 partition
//   3  CSR,WM          G lanes per row (G = 2..32 from nnz/rows), shfl   -
//   4  CSR,WO          merge-path tiles, in-kernel 32-ary diagonal search -
//   5  CSR,TM          thread per row; each CTA's nnz window staged into K-
//                      smem by 1-D TMA bulk copies (double buffered)
//   6  COO,WM          warp owns 256 nnz, blocked loads, segmented scan  K11 row ids
//   7  ELL,TM          column-major ELL, thread per row (+CSR tail)      K12 (+K1 width)
//
// Determinism: no floating-point atomics anywhere.  Rows split across work units are
// finished by k_carry_fixup, which sums the carries of a run of units in a fixed
// (lane-strided + shuffle-tree) order, so y is bit-identical run to run.
#include <stdlib.h>
#include <cstddef>

#include <cooperative_groups.h>

#include "kp_internal.cuh"

namespace kp {
int launch_k1_stats_into(const void *off, int32_t off_type, int64_t n_rows, int64_t *out4, void *ws,
                         cudaStream_t s);
int ensure_kernel_attrs();
}

namespace kp {
namespace {

constexpr int kAlign = 256;
__host__ __device__ constexpr size_t align_up(size_t v, size_t a = kAlign) { return (v + a - 1) / a * a; }

// ---------------------------------------------------------------- prepared layout
struct PrepHeader {
    int64_t kernel;
    int64_t n_units;   // device-written for adaptive
    int64_t stats[4];  // ELL: (lo, hi, s1, s2) of row lengths (K1)
    int64_t cap;       // ELL reserved width
    int64_t n_tail;    // ELL: rows longer than the width (device-written by K12) ...
    int64_t n_long;    // ... of which this many have > kEllLongTail elements past it
    int64_t n_short;   // ... and this many not (list-fill counter)
    int64_t pad[6];
};
static_assert(sizeof(PrepHeader) <= kAlign, "header");
constexpr size_t kRedWsBytes = 40960;  // >= kp_reduce_workspace_bytes()

// ---------------------------------------------------------------- tunables
constexpr int kIPT = 8;         // merge items / nnz per thread
constexpr int kCooChunk = 32 * kIPT;      // 256 nnz per warp
constexpr int kTmRows = 256;              // CSR,TM rows per CTA tile
constexpr int kAdBlockNnz = 2048;         // adaptive: nnz window of a short row block
constexpr int kAdLongT = 1024;            // adaptive: rows longer than this are "long"
constexpr int kAdCap = kAdBlockNnz + kAdLongT;
constexpr int kAdRows = 256;              // adaptive: max rows per short block
constexpr int64_t kAdLongChunk = 8192;    // adaptive: nnz per long-row piece

template <typename V>
__device__ __forceinline__ V fma_acc(V acc, V a, V b) { return fma(a, b, acc); }

// Fused row-sharded exchange (kp_spmv_bcast): the SpMV's y stores go straight to every
// rank's next-x buffer (this rank's slice of it) through NVLink peer mappings, so no
// separate all-gather runs after the kernel.  y[self] is the local copy the fix-up reads.
// Launch with programmatic stream serialization (PDL): the dependent kernel's CTAs are
// scheduled while the previous kernel drains and block in griddepcontrol.wait, hiding the
// launch gap between a SpMV and its carry fix-up (captured as a programmatic graph edge).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// accumulator reads of kp_spmv_bcast_acc: read once, coherent (acc may alias y[self]);
// KP_ACC_EF (A/B): L2 evict-first, so the accumulator stream does not displace the
// column slice's x lines
#ifndef KP_ACC_EF
#define KP_ACC_EF 0
#endif
template <typename V>
__device__ __forceinline__ V ld_acc(const V *p) {
#if KP_ACC_EF
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if constexpr (sizeof(V) == 4) {
        float v;
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
        return v;
    } else {
        double v;
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
        return v;
    }
#else
    return *p;
#endif
}

#ifndef KP_Y1_EF
#define KP_Y1_EF 0
#endif
template <typename V>
__device__ __forceinline__ void st_y1(V *p, V v) {
#if KP_Y1_EF
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if constexpr (sizeof(V) == 4)
        asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
    else
        asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#else
    *p = v;
#endif
}

// x gathers of the merge kernels.  KP_MERGE_X_CG_F64 (A/B): fp64 gathers L2-only (.cg),
// fp32 through L1 as everywhere else
#ifndef KP_MERGE_X_CG_F64
#define KP_MERGE_X_CG_F64 0
#endif
__device__ __forceinline__ float ld_x_merge(const float *p) { return ld_x(p); }
__device__ __forceinline__ double ld_x_merge(const double *p) {
#if KP_MERGE_X_CG_F64
    return __ldcg(p);
#else
    return ld_x(p);
#endif
}

template <typename V>
struct YDst {
    V *y[KP_MAX_PEERS];
    // column-blocked accumulation (kp_spmv_bcast_acc): the merge kernel's row stores add
    // acc[r] (null: none).  Each row is stored exactly once there (by the unit holding its
    // end), so acc is added once; the fix-up then adds carries onto y[self] as usual.
    // acc may alias y[self]: the same thread reads acc[r] before it stores y[.][r].
    const V *acc;
    // compressed-row column blocks: row r of the matrix is row rid[r] of y / acc (null:
    // identity).  Every access to y / acc by row index goes through row().
    const int32_t *rid;
    int32_t n, self;
    __device__ __forceinline__ int64_t row(int64_t r) const { return rid ? (int64_t)rid[r] : r; }
    __device__ __forceinline__ void put(int64_t i, V v) const {
        // fully unrolled with a predicate: a dynamic index into this by-value parameter
        // struct would force a local-memory copy of it
#pragma unroll
        for (int p = 0; p < KP_MAX_PEERS; ++p)
            if (p < n) y[p][i] = v;
    }
};

// ================================================================= long-row deferral (WM, TM)
// The row-mapped schedules (CSR,WM: a group of G lanes per row; CSR,TM: a thread per row)
// walk each row with one lane group, so a row far longer than the schedule's mean becomes
// a serial chain of dependent batches -- the 10-1000x pitfalls of PAPER.md Table II on
// power-law inputs (C2: WM 1.36 ms, TM 2.9 ms against 85 us for WO).  Rows longer than the
// schedule's threshold T are LISTED instead (one atomic per long row, in the SpMV
// workspace) and finished by k_long_rows, launched with PDL right behind the sweep: a warp
// per row up to kLongCta elements, a CTA per row beyond, each with a fixed reduction order
// (y stays bit-identical run to run).  The workspace is zeroed once at allocation; the
// tail's last CTA re-zeroes the counter.  No row can exceed n_cols elements, so T >= n_cols
// disables the list and the tail launch altogether.
struct DeferWs {
    unsigned int count, n_huge, n_giant, done;
    // [0, huge_at): rows up to kLongCta elements (a warp each); [huge_at, giant_at): up to
    // kLongCluster (a CTA each); [giant_at, ...): longer (a thread-block cluster each)
    int64_t rows[1];
};
constexpr int64_t kLongCta = 4096;
constexpr int64_t kLongGiant = 65536;
constexpr int kLongThreads = 512;
// One atomic per list per warp (the lanes that list a row of the same tier coalesce): a
// matrix whose rows are ALL long (a 300-wide band under CSR,TM) lists every row, and
// per-lane atomics on one counter serialised at the L2 (band 300: TM 107 us).
__device__ __forceinline__ void defer_append(unsigned int *cnt, int64_t *rows, int64_t row) {
    namespace cg = cooperative_groups;
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(cnt, (unsigned)g.size());
    base = g.shfl(base, 0);
    rows[base + g.thread_rank()] = row;
}
__device__ __forceinline__ void defer_row(DeferWs *dw, int64_t row, int64_t len, int64_t huge_at, int64_t giant_at) {
    if (len > kLongGiant) defer_append(&dw->n_giant, dw->rows + giant_at, row);
    else if (len > kLongCta) defer_append(&dw->n_huge, dw->rows + huge_at, row);
    else defer_append(&dw->count, dw->rows, row);
}

// ================================================================= CSR,WM (K4)
// Predicated batch of U strided elements: all U (col, val) loads are issued before the
// first x gather, so a lane keeps 2U + U requests in flight instead of one chain.
template <int U, int S, typename V>
__device__ __forceinline__ V batch_dot(const int32_t *__restrict__ col, const V *__restrict__ val,
                                       const V *__restrict__ x, int64_t j, int64_t e, V sum) {
    int32_t c[U];
    V v[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
        const int64_t q = j + (int64_t)i * S;
        c[i] = q < e ? ld_stream(col + q) : 0;
        v[i] = q < e ? ld_stream(val + q) : V(0);
    }
#pragma unroll
    for (int i = 0; i < U; ++i)
        if (j + (int64_t)i * S < e) sum = fma_acc(sum, v[i], ld_x(x + c[i]));
    return sum;
}

template <typename V, typename O, int G>
__global__ void __launch_bounds__(256) k_csr_wm(const O *__restrict__ off, const int32_t *__restrict__ col,
                                                const V *__restrict__ val, const V *__restrict__ x,
                                                V *__restrict__ y, int64_t n_rows, DeferWs *dw, int64_t long_t,
                                                int64_t huge_at, int64_t giant_at) {
    constexpr int U = 4;
    const int64_t row = ((int64_t)blockIdx.x * 256 + threadIdx.x) / G;
    if (row >= n_rows) return;  // whole groups exit together (G divides 32)
    const int gl = threadIdx.x % G;
    const int64_t s = ldo(off + row), e = ldo(off + row + 1);
    if (e - s > long_t) {  // listed for k_long_rows (the whole group leaves together)
        if (gl == 0) defer_row(dw, row, e - s, huge_at, giant_at);
        return;
    }
    V sum = 0;
    for (int64_t j = s + gl; j < e; j += (int64_t)U * G) sum = batch_dot<U, G>(col, val, x, j, e, sum);
    if constexpr (G > 1) {
        const unsigned mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(mask, sum, o);
    }
    if (gl == 0) y[row] = sum;
}

// ================================================================= CSR,BM (K5)
template <typename V>
__device__ __forceinline__ V block_sum(V v, V *sred) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = group_sum<32>(v);
    if (lane == 0) sred[w] = v;
    __syncthreads();
    V t = 0;
    if (w == 0) {
        t = lane < (int)(blockDim.x >> 5) ? sred[lane] : V(0);
        t = group_sum<32>(t);
    }
    return t;  // valid in thread 0
}

// Block-mapped: a CTA per row, so long rows get 128 x 4 gathers in flight and one block
// reduction.  A CTA spent on a row of a handful of elements is the schedule's pitfall
// (round-1 corpus: 5-70x behind the best kernel on short-row matrices, C2 443 us, road
// networks 69x), so rows are taken four at a time: each of the CTA's 4 warps sums one row
// of up to kBmShort elements (lane-strided batches + shuffle tree), and the group's longer
// rows then get the whole CTA, one after another (block_sum, as before).  Fixed reduction
// orders either way: y is bit-identical run to run.
constexpr int64_t kBmShort = 256;
template <typename V, typename O>
__global__ void __launch_bounds__(128) k_csr_bm(const O *__restrict__ off, const int32_t *__restrict__ col,
                                                const V *__restrict__ val, const V *__restrict__ x,
                                                V *__restrict__ y, int64_t n_rows) {
    __shared__ V sred[32];
    __shared__ int64_t s_s[4], s_e[4];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t r0 = (int64_t)blockIdx.x * 4; r0 < n_rows; r0 += (int64_t)gridDim.x * 4) {
        const int64_t row = r0 + w;
        int64_t s = 0, e = 0;
        if (row < n_rows) {
            s = ldo(off + row);
            e = ldo(off + row + 1);
        }
        if (e - s <= kBmShort) {  // short (or past the end): this warp
            if (row < n_rows) {
                V sum = 0;
                for (int64_t j = s + lane; j < e; j += 4 * 32) sum = batch_dot<4, 32>(col, val, x, j, e, sum);
                sum = group_sum<32>(sum);
                if (lane == 0) y[row] = sum;
            }
            s = e = 0;  // nothing left for the CTA
        }
        if (lane == 0) {
            s_s[w] = s;
            s_e[w] = e;
        }
        __syncthreads();
        for (int q = 0; q < 4; ++q) {  // the group's long rows: the whole CTA each
            const int64_t qs = s_s[q], qe = s_e[q];
            if (qe - qs <= kBmShort) continue;  // uniform over the CTA
            V sum = 0;
            for (int64_t j = qs + threadIdx.x; j < qe; j += 4 * 128) sum = batch_dot<4, 128>(col, val, x, j, qe, sum);
            const V t = block_sum(sum, sred);
            if (threadIdx.x == 0) y[r0 + q] = t;
            __syncthreads();  // sred reuse
        }
        __syncthreads();  // s_s / s_e reuse
    }
}

// CSR,BM for a KNOWN mean of at most kBmTinyMean elements per row (road networks, meshes,
// power-law graphs): rows of a few elements leave even a warp per row latency-bound (road
// 23x behind CSR,TM with the 4-row groups above), so the CTA takes a block of 128 rows per
// step and sorts them by length in shared memory: rows of up to `thread_max` (kBmThread)
// elements are summed by their own thread (the whole block's short rows in one trip), rows
// up to kBmShort by a warp each, the longer ones by the whole CTA (block_sum).  A row's
// length class fixes its reduction order, so y is bit-identical run to run.  Thresholds by
// A/B (profiles/ab_bm_r02.txt, per SpMV, this variant vs the 4-row groups): road 2067 ->
// 111 us, C2 276 -> 145 us, power-law 1042 -> 834 us, C1 10.3 us either way; means above
// 16 keep the 4-row groups (const 32: 967 vs 1407 us, 27-point stencils 28.7 vs 24.6 us at
// mean 27 is the one loss the cut leaves out).
constexpr int kBmThreads = 128;
constexpr int64_t kBmThread = 32;
constexpr double kBmTinyMean = 16.0;
template <typename V, typename O>
__global__ void __launch_bounds__(kBmThreads) k_csr_bm_short(const O *__restrict__ off, const int32_t *__restrict__ col,
                                                       const V *__restrict__ val, const V *__restrict__ x,
                                                       V *__restrict__ y, int64_t n_rows, int64_t thread_max) {
    __shared__ V sred[32];
    __shared__ int64_t s_w[kBmThreads], s_c[kBmThreads];
    __shared__ int s_nw, s_nc;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    for (int64_t r0 = (int64_t)blockIdx.x * kBmThreads; r0 < n_rows; r0 += (int64_t)gridDim.x * kBmThreads) {
        if (tid == 0) {
            s_nw = 0;
            s_nc = 0;
        }
        __syncthreads();
        const int64_t row = r0 + tid;
        if (row < n_rows) {
            const int64_t s = ldo(off + row), e = ldo(off + row + 1);
            if (e - s <= thread_max) {  // this thread
                V sum = 0;
                for (int64_t j = s; j < e; j += 4) sum = batch_dot<4, 1>(col, val, x, j, e, sum);
                y[row] = sum;
            } else if (e - s <= kBmShort) {
                s_w[atomicAdd(&s_nw, 1)] = row;
            } else {
                s_c[atomicAdd(&s_nc, 1)] = row;
            }
        }
        __syncthreads();
        const int nw = s_nw, nc = s_nc;
        for (int i = w; i < nw; i += kBmThreads / 32) {  // a warp each
            const int64_t rw = s_w[i];
            const int64_t s = ldo(off + rw), e = ldo(off + rw + 1);
            V sum = 0;
            for (int64_t j = s + lane; j < e; j += 4 * 32) sum = batch_dot<4, 32>(col, val, x, j, e, sum);
            sum = group_sum<32>(sum);
            if (lane == 0) y[rw] = sum;
        }
        for (int i = 0; i < nc; ++i) {  // the whole CTA each
            const int64_t rc = s_c[i];
            const int64_t s = ldo(off + rc), e = ldo(off + rc + 1);
            V sum = 0;
            for (int64_t j = s + tid; j < e; j += 4 * kBmThreads) sum = batch_dot<4, kBmThreads>(col, val, x, j, e, sum);
            const V t = block_sum(sum, sred);
            if (tid == 0) y[rc] = t;
            __syncthreads();  // sred reuse
        }
        // the counters and lists are reset / refilled by the next group: every warp must
        // have read them first (racecheck: thread 0 could zero s_nw / s_nc while a slower
        // warp had yet to read them, dropping that warp's rows)
        __syncthreads();
    }
}

// ================================================================= CSR,TM (K3)
// Thread per row, warp-specialised TMA pipeline.  A persistent CTA = 8 consumer warps
// (256 threads, RPT rows each per tile) + 1 producer warp; 2 stages of <= 3072 nnz (fp32)
// measured best on short-row inputs (band 4: 0.81 of the HBM peak vs 0.70 with 3 x 2048).  Per tile of 256*RPT rows
// the producer pulls the row-offset window [r0, r1] and the nnz window
// [off[r0], off[r1]) of cols and vals into one of 2 shared-memory stages with 1-D TMA
// bulk copies (SASS UBLKCP) completing on the stage's `full` mbarrier; consumer warps
// release a stage through its `empty` mbarrier, so no CTA-wide barrier sits in the
// loop.  RPT is chosen on the host from the KNOWN mean row length (window ~3/4 of a
// stage).  Medium rows get enlarged stages (below); a window larger than its stage (skew)
// falls back to direct per-thread global walks for that tile.
constexpr int kTmStages = 2;
constexpr int kTmMaxRpt = 4;
// gathers in flight per consumer thread: 4 for short-row stages (band 4: 0.81 of HBM vs
// 0.70 at 8) and for the enlarged medium-row stages (split rows, below)
constexpr int kTmUWide = 4;
constexpr int kTmSplitWide = 2;  // consumer threads per row in the medium-row stages
// Medium rows (the tile window of 256 rows exceeds kCap at the known mean, e.g. 27-point
// stencils) get a LARGER stage instead of the per-thread global walk: capacity sized from
// the known mean, up to what two stages of one CTA per SM can hold (kCapMax), so the
// thread-per-row gathers stay coalesced across consecutive rows (ELL's access pattern
// without its preparation).
template <typename V, typename O>
struct TmCfg {
    static constexpr int kCap = sizeof(V) == 4 ? 3072 : 1536;                    // nnz per stage (short rows)
    static constexpr int kOffs = kTmRows * kTmMaxRpt + 8;                          // offsets per stage
    static constexpr size_t kOffBytes = (kOffs * sizeof(O) + 127) / 128 * 128;
    static constexpr size_t kSmemMax = 216 * 1024;                                 // 2 stages, 1 CTA / SM
    static constexpr int kCapMax = (int)((kSmemMax / kTmStages - kOffBytes) / (4 + sizeof(V))) / 128 * 128;
    __host__ __device__ static constexpr size_t col_bytes(int cap) { return ((size_t)cap * 4 + 127) / 128 * 128; }
    __host__ __device__ static constexpr size_t stage_bytes(int cap) {
        return kOffBytes + col_bytes(cap) + ((size_t)cap * sizeof(V) + 127) / 128 * 128;
    }
};

// kSplit > 1 (medium-row stages): kSplit consumer threads per row, each summing a
// contiguous part of it; a warp holds 32 / kSplit consecutive rows x kSplit parts
// (consecutive rows in consecutive lanes, so the gathers stay coalesced) and combines the
// parts with shuffles in a fixed order: kSplit x the gathers in flight per tile.
// Measured on C3 / band 27 / band 27 fp64 (fraction of HBM), parts combined through
// shared memory + a consumer barrier: (U, split) = (16, 1) 0.63 / 0.72 / 0.83, (8, 2)
// 0.69-0.72 / 0.74-0.76 / 0.89-0.90, (4, 2) 0.67 / 0.77 / 0.90, (16, 2) 0.53 / 0.57 / 0.91,
// (8, 3) 0.52 / 0.55 / 0.88; (8, 2) with the in-warp shuffle combine (no barrier, ncu
// showed 17 % barrier stalls): 0.71 / 0.77 / 0.93; then (4, 2): C3 195 -> 188 us, band 27
// 184 -> 174 us, band 27 fp64 equal (graph A/B; (12, 2) 213 / 203 / 242 us).
template <typename V, typename O, bool kTma, int kTmU, int kSplit>
__global__ void __launch_bounds__(kTmRows * kSplit + 32) k_csr_tm(const O *__restrict__ off, const int32_t *__restrict__ col,
                                                         const V *__restrict__ val, const V *__restrict__ x,
                                                         V *__restrict__ y, int64_t n_rows, int rpt, int kCap,
                                                         DeferWs *dw, int64_t long_t, int64_t huge_at,
                                                         int64_t giant_at) {
    using Cfg = TmCfg<V, O>;
    const size_t stage = Cfg::stage_bytes(kCap);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kTmStages], empty[kTmStages];
    __shared__ int64_t s_base[kTmStages];  // element index staged at col slot 0; -1 = direct
    const int64_t tile_rows = (int64_t)kTmRows * rpt;
    const int64_t n_tiles = (n_rows + tile_rows - 1) / tile_rows;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    auto st_off = [&](int k) { return reinterpret_cast<O *>(smem_raw + k * stage); };
    auto st_col = [&](int k) { return reinterpret_cast<int32_t *>(smem_raw + k * stage + Cfg::kOffBytes); };
    auto st_val = [&](int k) {
        return reinterpret_cast<V *>(smem_raw + k * stage + Cfg::kOffBytes + Cfg::col_bytes(kCap));
    };
    if (tid == 0) {
        for (int k = 0; k < kTmStages; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], kTmRows * kSplit / 32);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kTmRows * kSplit / 32) {  // ---------------------------------- producer
        if (lane != 0) return;
        const int64_t nnz = ldo(off + n_rows);
        auto bounds = [&](int64_t t, int64_t &s, int64_t &e) {
            const int64_t r0 = t * tile_rows;
            s = ldo(off + r0);
            e = ldo(off + (r0 + tile_rows < n_rows ? r0 + tile_rows : n_rows));
        };
        int64_t sn = 0, en = 0;
        if ((int64_t)blockIdx.x < n_tiles) bounds(blockIdx.x, sn, en);
        int i = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
            const int k = i % kTmStages;
            const int64_t s = sn, e = en;
            if (t + gridDim.x < n_tiles) bounds(t + gridDim.x, sn, en);  // prefetch next tile's window
            if (i >= kTmStages) mbar_wait(&empty[k], (uint32_t)(((i / kTmStages) - 1) & 1));
            const int64_t r0 = t * tile_rows;
            const int64_t r1 = r0 + tile_rows < n_rows ? r0 + tile_rows : n_rows;
            // offsets window [r0, r1], rounded up to 16 B while in bounds (n_rows + 1 entries)
            const int64_t n1 = r1 - r0 + 1;
            constexpr int kOV = 16 / (int)sizeof(O);
            int64_t nb = kTma ? (n1 + kOV - 1) / kOV * kOV : 0;
            if (r0 + nb > n_rows + 1) nb = kTma ? n1 / kOV * kOV : 0;
            O *so = st_off(k);
            for (int64_t q = nb; q < n1; ++q) so[q] = off[r0 + q];
            // nnz window [a, e) with a 16-byte aligned, end rounded up while in bounds
            const int64_t a = s & ~(int64_t)3;
            const bool fits = kTma && e > s && ((e + 3) & ~(int64_t)3) - a <= kCap;
            int32_t *sc = st_col(k);
            V *sv = st_val(k);
            int64_t eb = (e + 3) & ~(int64_t)3;
            if (eb > nnz) eb = e & ~(int64_t)3;  // last window of the matrix: hand-copy the tail
            if (!fits || eb < a) eb = a;
            if (fits)
                for (int64_t j = eb; j < e; ++j) {
                    sc[j - a] = __ldg(col + j);
                    sv[j - a] = __ldg(val + j);
                }
            s_base[k] = fits ? a : -1;
            const uint32_t n = (uint32_t)(eb - a);
            const uint32_t tx = (uint32_t)(nb * sizeof(O)) + n * (uint32_t)(sizeof(int32_t) + sizeof(V));
            mbar_arrive_expect_tx(&full[k], tx);
            if (nb) bulk_g2s(so, off + r0, (uint32_t)(nb * sizeof(O)), &full[k]);
            if (n) {
                bulk_g2s(sc, col + a, n * (uint32_t)sizeof(int32_t), &full[k]);
                bulk_g2s(sv, val + a, n * (uint32_t)sizeof(V), &full[k]);
            }
        }
        return;
    }
    // ------------------------------------------------------------------ consumers
    int i = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
        const int k = i % kTmStages;
        mbar_wait(&full[k], (uint32_t)((i / kTmStages) & 1));
        const int64_t base = s_base[k];
        const O *so = st_off(k);
        const int32_t *sc = st_col(k) - base;
        const V *sv = st_val(k) - base;
        const int64_t r0 = t * tile_rows;
        auto row_sum = [&](int64_t s, int64_t e) {
            V sum = 0;
            if (base >= 0) {
                for (int64_t j = s; j < e; j += kTmU) {  // kTmU gathers in flight per thread
                    int32_t c[kTmU];
                    V v[kTmU];
#pragma unroll
                    for (int u = 0; u < kTmU; ++u) {
                        c[u] = j + u < e ? sc[j + u] : 0;
                        v[u] = j + u < e ? sv[j + u] : V(0);
                    }
#pragma unroll
                    for (int u = 0; u < kTmU; ++u)
                        if (j + u < e) sum = fma_acc(sum, v[u], ld_x(x + c[u]));
                }
            } else {
                for (int64_t j = s; j < e; j += 4) sum = batch_dot<4, 1>(col, val, x, j, e, sum);
            }
            return sum;
        };
        if constexpr (kSplit > 1) {  // rpt = 1 (host)
            // the kSplit parts of a row sit in the SAME warp (lane groups of 32 / kSplit
            // consecutive rows), so the combine is a shuffle, not a CTA barrier
            constexpr int kG = 32 / kSplit;
            const int rl = warp * kG + (lane % kG), part = lane / kG;
            bool act = r0 + rl < n_rows;
            V sum = V(0);
            if (act) {
                const int64_t s = (int64_t)so[rl], e = (int64_t)so[rl + 1];
                if (e - s > long_t) {  // listed for k_long_rows
                    act = false;
                    if (part == 0) defer_row(dw, r0 + rl, e - s, huge_at, giant_at);
                } else {
                    const int64_t chunk = (e - s + kSplit - 1) / kSplit;
                    const int64_t a = s + part * chunk, b = a + chunk < e ? a + chunk : e;
                    sum = row_sum(a, b);
                }
            }
#pragma unroll
            for (int o = kG * (kSplit / 2); o >= kG; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);  // fixed order
            if (part == 0 && act) y[r0 + rl] = sum;
        } else {
#pragma unroll
            for (int q = 0; q < kTmMaxRpt; ++q) {
                const int rl = tid + q * kTmRows;
                if (q >= rpt || r0 + rl >= n_rows) break;
                const int64_t s = (int64_t)so[rl], e = (int64_t)so[rl + 1];
                if (e - s > long_t) defer_row(dw, r0 + rl, e - s, huge_at, giant_at);  // listed for k_long_rows
                else y[r0 + rl] = row_sum(s, e);
            }
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[k])) : "memory");
    }
}

// ================================================================= ELL,TM (K9 + K12)
// Thread per row over the warp-sliced ELL (width W = min(max_len, cap)).  Rows longer than
// W (listed by K12) keep their first W elements here; k_ell_tail adds the rest.
template <typename V, typename O>
__global__ void __launch_bounds__(256) k_ell_tm(const PrepHeader *__restrict__ hdr, const int32_t *__restrict__ ecol,
                                                const V *__restrict__ evalv, const V *__restrict__ x,
                                                V *__restrict__ y, int64_t n_rows) {
    // the PDL-launched tail kernel may be scheduled now (it waits for this grid's completion)
    asm volatile("griddepcontrol.launch_dependents;");
    const int64_t row = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (row >= n_rows) return;
    const int64_t wmax = __ldg(&hdr->stats[1]);
    const int64_t cap = __ldg(&hdr->cap);
    const int64_t W = wmax < cap ? wmax : cap;
    V sum = 0;
    // warp-sliced column-major layout: the 32 rows of a warp own a contiguous [W][32]
    // slab, so slot k of this row is at slab + 32*k -> each warp streams one contiguous
    // region (DRAM-page / TLB friendly, unlike a global n_rows stride); 8 slots
    // (16 loads) in flight per thread before the x gathers.
    const int64_t slab = (row >> 5) * 32 * W + (row & 31);
    const int32_t *pc = ecol + slab;
    const V *pv = evalv + slab;
    // software pipeline: slots k+8..k+15 are loading while slots k..k+7 gather x
    int32_t nc[8];
    V nv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        nc[i] = i < W ? ld_stream(pc + i * 32) : 0;
        nv[i] = i < W ? ld_stream(pv + i * 32) : V(0);
    }
    for (int64_t k = 0; k < W; k += 8) {
        int32_t c[8];
        V v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            c[i] = nc[i];
            v[i] = nv[i];
        }
        if (k + 8 < W) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                nc[i] = k + 8 + i < W ? ld_stream(pc + (k + 8 + i) * 32) : 0;
                nv[i] = k + 8 + i < W ? ld_stream(pv + (k + 8 + i) * 32) : V(0);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (k + i < W) sum = fma_acc(sum, v[i], ld_x(x + c[i]));
    }
    y[row] = sum;
}

// Hybrid tail of ELL,TM: rows longer than the width W (K12's lists) get their elements
// W.. added here, in a fixed order (y stays bit-identical run to run): rows with more than
// kEllLongTail remaining elements by a whole CTA each (block reduction), the others by one
// warp each (lane-strided batches + shuffle tree).  Launched with PDL right behind
// k_ell_tm: it waits for the sweep's y stores, and exits at once when K12 listed no row
// (W = max_len, the favourable case).  (The tail used to continue serially in the row's
// own thread: C2 4.3 ms, C4 115 ms.)
constexpr int64_t kEllLongTail = 4096;
constexpr int kEllTailThreads = 512;
template <typename V, typename O>
__global__ void __launch_bounds__(kEllTailThreads) k_ell_tail(const PrepHeader *__restrict__ hdr,
                                                              const int64_t *__restrict__ tail, int64_t tail_slots,
                                                              const O *__restrict__ off, const int32_t *__restrict__ col,
                                                              const V *__restrict__ val, const V *__restrict__ x,
                                                              V *__restrict__ y) {
    __shared__ V sred[32];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t nt = hdr->n_tail, nl = hdr->n_long;
    if (nt == 0) return;
    const int64_t wmax = hdr->stats[1], cap = hdr->cap;
    const int64_t W = wmax < cap ? wmax : cap;
    // long rows (listed from the back of the buffer): one CTA each
    for (int64_t t = blockIdx.x; t < nl; t += gridDim.x) {
        const int64_t row = tail[tail_slots - 1 - t];
        const int64_t s = ldo(off + row) + W, e = ldo(off + row + 1);
        V sum = 0;
        for (int64_t j = s + threadIdx.x; j < e; j += 4 * kEllTailThreads)
            sum = batch_dot<4, kEllTailThreads>(col, val, x, j, e, sum);
        const V tot = block_sum(sum, sred);
        if (threadIdx.x == 0) y[row] += tot;
        __syncthreads();  // sred is reused by the next row
    }
    // the other listed rows: one warp each
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < nt - nl; t += nw) {
        const int64_t row = tail[t];
        const int64_t s = ldo(off + row) + W, e = ldo(off + row + 1);
        V sum = 0;
        for (int64_t j = s + lane; j < e; j += 4 * 32) sum = batch_dot<4, 32>(col, val, x, j, e, sum);
        sum = group_sum<32>(sum);
        if (lane == 0) y[row] += sum;
    }
}

// Finishes the rows CSR,WM / CSR,TM listed (see DeferWs): whole rows, written once.
// Rows past kLongGiant elements take a thread-block CLUSTER of kLongCluster CTAs each (the
// CTAs stride the row together, 8 x 512 x 4 gathers in flight; rank 0 folds the CTAs'
// partials through distributed shared memory in rank order -- C4's 1 M-element rows in one
// pass instead of one CTA walking them); rows past kLongCta a CTA each; the rest a warp each.
constexpr int kLongCluster = 8;
template <typename V, typename O>
__global__ void __launch_bounds__(kLongThreads) k_long_rows(DeferWs *__restrict__ dw, const O *__restrict__ off,
                                                            const int32_t *__restrict__ col, const V *__restrict__ val,
                                                            const V *__restrict__ x, V *__restrict__ y,
                                                            int64_t huge_at, int64_t giant_at) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ V sred[32];
    __shared__ V s_part;
    __shared__ int64_t s_n[3];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
        s_n[0] = (int64_t)*reinterpret_cast<volatile unsigned int *>(&dw->count);
        s_n[1] = (int64_t)*reinterpret_cast<volatile unsigned int *>(&dw->n_huge);
        s_n[2] = (int64_t)*reinterpret_cast<volatile unsigned int *>(&dw->n_giant);
    }
    __syncthreads();
    const int64_t n = s_n[0], nh = s_n[1], ng = s_n[2];
    if (n == 0 && nh == 0 && ng == 0) return;  // the common case: nothing listed, nothing to reset
    const volatile int64_t *rows = dw->rows;
    // giant rows: a cluster each (identical trip sequence in every CTA of a cluster)
    const unsigned cr = cl.block_rank();
    const int64_t cid = blockIdx.x / kLongCluster, ncl = gridDim.x / kLongCluster;
    for (int64_t t = cid; t < ng; t += ncl) {
        const int64_t row = rows[giant_at + t];
        const int64_t s = ldo(off + row), e = ldo(off + row + 1);
        V sum = 0;
        constexpr int S = kLongThreads * kLongCluster;
        for (int64_t j = s + (int64_t)cr * kLongThreads + threadIdx.x; j < e; j += 4 * (int64_t)S)
            sum = batch_dot<4, S>(col, val, x, j, e, sum);
        const V tot = block_sum(sum, sred);
        if (threadIdx.x == 0) s_part = tot;
        cl.sync();
        if (cr == 0 && threadIdx.x == 0) {
            V acc = 0;
            for (int r = 0; r < kLongCluster; ++r) acc += *cl.map_shared_rank(&s_part, r);
            y[row] = acc;
        }
        cl.sync();  // s_part / sred are reused by the next row
    }
    // large rows: a CTA each
    for (int64_t t = blockIdx.x; t < nh; t += gridDim.x) {
        const int64_t row = rows[huge_at + t];
        const int64_t s = ldo(off + row), e = ldo(off + row + 1);
        V sum = 0;
        for (int64_t j = s + threadIdx.x; j < e; j += 4 * kLongThreads) sum = batch_dot<4, kLongThreads>(col, val, x, j, e, sum);
        const V tot = block_sum(sum, sred);
        if (threadIdx.x == 0) y[row] = tot;
        __syncthreads();  // sred reuse
    }
    // the others: a warp each (lane-strided batches + shuffle tree)
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += nw) {
        const int64_t row = rows[t];
        const int64_t s = ldo(off + row), e = ldo(off + row + 1);
        V sum = 0;
        for (int64_t j = s + lane; j < e; j += 4 * 32) sum = batch_dot<4, 32>(col, val, x, j, e, sum);
        sum = group_sum<32>(sum);
        if (lane == 0) y[row] = sum;
    }
    // every CTA has read the counts: the last one re-zeroes the lists for the next launch
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&dw->done, 1u) == gridDim.x - 1) {
            dw->count = 0;
            dw->n_huge = 0;
            dw->n_giant = 0;
            dw->done = 0;
            __threadfence();
        }
    }
}

__global__ void k_prep_hdr(PrepHeader *hdr, int64_t kernel, int64_t cap) {
    PrepHeader h = {};
    h.kernel = kernel;
    h.cap = cap;
    *hdr = h;
}

// K12: CSR -> warp-sliced column-major ELL of width W = min(max_len, cap): slot (row, k)
// at (row/32)*32*W + 32*k + row%32; padding = (col 0, val 0).  Rows longer than W are
// appended to the tail list (one global atomic per CTA; list order is irrelevant: every
// listed row is summed whole by one warp).
template <typename V, typename O>
__global__ void __launch_bounds__(256) k_prep_ell(PrepHeader *__restrict__ hdr, const O *__restrict__ off,
                                                  const int32_t *__restrict__ col, const V *__restrict__ val,
                                                  int32_t *__restrict__ ecol, V *__restrict__ evalv,
                                                  int64_t *__restrict__ tail, int64_t tail_slots, int64_t n_rows) {
    __shared__ int s_cnt, s_lcnt;
    __shared__ int64_t s_base, s_lbase;
    const int64_t row = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int64_t wmax = hdr->stats[1];
    const int64_t cap = hdr->cap;
    const int64_t W = wmax < cap ? wmax : cap;
    if (threadIdx.x == 0) s_cnt = s_lcnt = 0;
    __syncthreads();
    int slot_in_cta = -1;
    bool is_long = false;
    if (row < n_rows) {
        const int64_t s = ldo(off + row), e = ldo(off + row + 1);
        // 8 slots per trip: all 16 loads issued before the stores (a slot-at-a-time loop
        // kept one load pair in flight per thread: 64 M x 8 const rows took ~36 ms)
        for (int64_t k0 = 0; k0 < W; k0 += 8) {
            int32_t c[8];
            V v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t j = s + k0 + i;
                const bool in = k0 + i < W && j < e;
                c[i] = in ? __ldg(col + j) : 0;
                v[i] = in ? __ldg(val + j) : V(0);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (k0 + i >= W) break;
                const int64_t slot = (row >> 5) * 32 * W + (k0 + i) * 32 + (row & 31);
                ecol[slot] = c[i];
                evalv[slot] = v[i];
            }
        }
        if (e - s > W) {
            is_long = e - s - W > kEllLongTail;
            slot_in_cta = atomicAdd(is_long ? &s_lcnt : &s_cnt, 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // n_tail counts every listed row; short rows fill the list from the front, long
        // rows from the back (tail_slots >= every listed row: no overlap)
        if (s_cnt + s_lcnt > 0) atomicAdd((unsigned long long *)&hdr->n_tail, (unsigned long long)(s_cnt + s_lcnt));
        if (s_cnt > 0) s_base = (int64_t)atomicAdd((unsigned long long *)&hdr->n_short, (unsigned long long)s_cnt);
        if (s_lcnt > 0) s_lbase = (int64_t)atomicAdd((unsigned long long *)&hdr->n_long, (unsigned long long)s_lcnt);
    }
    __syncthreads();
    if (slot_in_cta >= 0) {
        if (is_long) tail[tail_slots - 1 - (s_lbase + slot_in_cta)] = row;
        else tail[s_base + slot_in_cta] = row;
    }
}

// ================================================================= block-level segmented scan
// Inclusive scan over threads of (flag, value) with op (fa,va)o(fb,vb) = (fa|fb, fb ? vb : va+vb).
template <typename V>
struct SegPair {
    int f;
    V v;
};
template <typename V>
__device__ __forceinline__ SegPair<V> seg_op(SegPair<V> a, SegPair<V> b) {
    return SegPair<V>{a.f | b.f, b.f ? b.v : a.v + b.v};
}
// Returns the EXCLUSIVE prefix for this thread (identity: f=0, v=0) and the block total.
template <typename V>
__device__ __forceinline__ SegPair<V> block_seg_exscan(SegPair<V> p, SegPair<V> &total, SegPair<V> *swarp) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    SegPair<V> inc = p;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        SegPair<V> t{__shfl_up_sync(0xffffffffu, inc.f, o), __shfl_up_sync(0xffffffffu, inc.v, o)};
        if (lane >= o) inc = seg_op(t, inc);
    }
    if (lane == 31) swarp[w] = inc;
    __syncthreads();
    if (w == 0) {
        SegPair<V> wv = lane < nw ? swarp[lane] : SegPair<V>{0, V(0)};
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            SegPair<V> t{__shfl_up_sync(0xffffffffu, wv.f, o), __shfl_up_sync(0xffffffffu, wv.v, o)};
            if (lane >= o) wv = seg_op(t, wv);
        }
        if (lane < nw) swarp[lane] = wv;  // inclusive warp prefixes
    }
    __syncthreads();
    SegPair<V> ex{__shfl_up_sync(0xffffffffu, inc.f, 1), __shfl_up_sync(0xffffffffu, inc.v, 1)};
    if (lane == 0) ex = SegPair<V>{0, V(0)};
    if (w > 0) ex = seg_op(swarp[w - 1], ex);
    total = swarp[nw - 1];
    return ex;
}

// ================================================================= carries / fix-up
// A unit u (COO chunk, merge tile, adaptive long piece) that leaves row rho unfinished
// records carry_row[u] = rho, carry_val[u] = its partial (carry_row = -1: none).  The
// unit that finishes rho wrote y[rho] = its own partial.  Fix-up: a warp takes 32
// consecutive units (lane = unit), segments them by carry row with a shuffle scan
// (fixed order) and the last lane of each run adds the run's sum to y[rho].  A run that
// continues past the warp's 32 units is finished by the warp where it STARTED, which
// walks the following units 32 at a time (lane-strided sum + shuffle tree); warps whose
// first run started earlier skip it.  Deterministic, no atomics.
template <typename V, bool kB = false>
__global__ void __launch_bounds__(256) k_carry_fixup(const int32_t *__restrict__ crow, const V *__restrict__ cval,
                                                     const int64_t *__restrict__ n_units_dev, int64_t n_units_host,
                                                     V *__restrict__ y, YDst<V> dst = YDst<V>{}) {
    // programmatic dependent launch: this grid may be resident before the producing SpMV
    // grid finishes; wait here until its carries are complete and visible
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t n_units = n_units_dev ? *n_units_dev : n_units_host;
    const int lane = threadIdx.x & 31;
    // grid-stride over groups of 32 units: the launch is sized for the work, not for a
    // host-side upper bound of the (device-counted) unit number
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t wbase = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; wbase < n_units;
         wbase += nwarps * 32) {
        const int64_t u = wbase + lane;
        const int32_t r = u < n_units ? crow[u] : -2;
        const V v = (u < n_units && r >= 0) ? cval[u] : V(0);
        int32_t prev = __shfl_up_sync(0xffffffffu, r, 1);
        if (lane == 0) prev = wbase > 0 ? crow[wbase - 1] : -3;
        const bool head = r != prev;
        // inclusive segmented scan within the warp
        SegPair<V> inc{head ? 1 : 0, v};
    #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            SegPair<V> t{__shfl_up_sync(0xffffffffu, inc.f, o), __shfl_up_sync(0xffffffffu, inc.v, o)};
            if (lane >= o) inc = seg_op(t, inc);
        }
        int32_t next = __shfl_down_sync(0xffffffffu, r, 1);
        if (lane == 31) next = (u + 1 < n_units) ? crow[u + 1] : -4;
        // does this lane's run start inside this warp?  (lane of the run head)
        const unsigned heads = __ballot_sync(0xffffffffu, head);
        const unsigned below = heads & ((lane == 31) ? 0xffffffffu : ((2u << lane) - 1u));
        const bool started_here = below != 0;  // a head at or before this lane within the warp
        const bool run_end_here = next != r;
        if (r >= 0 && started_here && run_end_here) {
            if constexpr (kB) {
                const int64_t rr = dst.row(r);
                dst.put(rr, dst.y[dst.self][rr] + inc.v);
            } else {
                y[r] += inc.v;
            }
        }
        // run open at the warp end that started in this warp: continue over later units
        const bool cont = (lane == 31) && r >= 0 && started_here && !run_end_here;
        if (__ballot_sync(0xffffffffu, cont)) {
            const int32_t rho = __shfl_sync(0xffffffffu, r, 31);
            V acc = 0;
            // 8 batches of 32 units per trip, all loads issued first; rho never reappears after
            // its run ends, so matches past the end of the run cannot occur
            for (int64_t b = wbase + 32;; b += 256) {
                int32_t rr[8];
                V vv[8];
    #pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int64_t q = b + 32 * i + lane;
                    rr[i] = q < n_units ? crow[q] : -5;
                    vv[i] = q < n_units ? cval[q] : V(0);
                }
                bool open = true;
    #pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const bool in = rr[i] == rho;
                    if (in) acc += vv[i];
                    open = open && __ballot_sync(0xffffffffu, in) == 0xffffffffu;
                }
                if (!open) break;  // the run ended inside this trip
            }
            acc = group_sum<32>(acc);
            if (lane == 31) {
                if constexpr (kB) {
                    const int64_t rr = dst.row(rho);
                    dst.put(rr, dst.y[dst.self][rr] + (inc.v + acc));
                } else {
                    y[rho] += inc.v + acc;
                }
            }
        }
    }
}

// ================================================================= merge-path tiles (K6 MP, K7 WO)
// Merge of A = row ends off[1..R] with B = nnz indices 0..Z-1 (Merrill & Garland).
// Diagonal d -> (i rows consumed, d - i nnz consumed).  Work unit = one WARP tile of
// 256 merge items: the warp stages its row ends (int32, relative to the tile's first
// nnz) and products val*x[col] in its own shared-memory slice (batched loads, no
// CTA barrier), each lane merges 8 items sequentially, a warp segmented scan (shfl)
// carries partial rows between lanes, and the row left open at the tile end is the
// unit's carry (finished by k_carry_fixup).
template <typename O>
__device__ __forceinline__ int64_t merge_search_global(const O *off, int64_t n_rows, int64_t nnz, int64_t d) {
    int64_t lo = d - nnz > 0 ? d - nnz : 0;
    int64_t hi = d < n_rows ? d : n_rows;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ldo(off + mid + 1) <= d - mid - 1) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Warp-cooperative 32-ary version (5 rounds of 32 parallel probes for 2^25 items).
template <typename O>
__device__ __forceinline__ int64_t merge_search_warp_in(const O *off, int64_t d, int64_t lo, int64_t hi) {
    const int lane = threadIdx.x & 31;
    while (hi - lo > 32) {
        const int64_t step = (hi - lo + 32) / 33;  // probes at lo + step*(lane+1) - 1
        int64_t p = lo + step * (lane + 1) - 1;
        if (p >= hi) p = hi - 1;
        const bool go_right = ldo(off + p + 1) <= d - p - 1;  // predicate monotone in p
        const unsigned m = __ballot_sync(0xffffffffu, go_right);
        const int cnt = __popc(m);  // lanes 0..cnt-1 true (monotone)
        int64_t nlo = cnt == 0 ? lo : (lo + step * cnt - 1) + 1;
        int64_t nhi = cnt == 32 ? hi : lo + step * (cnt + 1) - 1;
        if (nhi > hi) nhi = hi;
        if (nlo > nhi) nlo = nhi;
        lo = nlo;
        hi = nhi;
    }
    const int64_t p = lo + lane;  // final <= 32 candidates: one probe per lane
    const bool gr = p < hi && ldo(off + p + 1) <= d - p - 1;
    return lo + __popc(__ballot_sync(0xffffffffu, gr));
}
template <typename O>
__device__ __forceinline__ int64_t merge_search_warp(const O *off, int64_t n_rows, int64_t nnz, int64_t d) {
    return merge_search_warp_in(off, d, d - nnz > 0 ? d - nnz : 0, d < n_rows ? d : n_rows);
}

// CTA-shared first round of the WO start search: the CTA's warps start at nearby diagonals,
// so one 256-point grid of Q(p) = off[p+1] + p + 1 (strictly increasing; the merge
// coordinate of diagonal d is #{p : Q(p) <= d}) over the union of their search intervals,
// loaded once (one probe per thread), narrows every warp to one grid cell before its own
// 32-ary search: one dependent round instead of log33(256) ~ 1.6 of the per-warp search.
template <typename O>
__device__ __forceinline__ int64_t merge_search_cta(const O *off, int64_t n_rows, int64_t nnz, int64_t d,
                                                    int64_t d_first, int64_t d_last, int64_t *s_q) {
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t lo = d_first - nnz > 0 ? d_first - nnz : 0;
    const int64_t hi = d_last < n_rows ? d_last : n_rows;
    const int64_t step = (hi - lo + 256) / 257;
    {
        const int64_t p = lo + step * (tid + 1) - 1;
        s_q[tid] = p < hi ? (int64_t)ldo(off + p + 1) + p + 1 : INT64_MAX;
    }
    __syncthreads();
    int c = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) c += s_q[lane * 8 + t] <= d ? 1 : 0;
    c = __reduce_add_sync(0xffffffffu, c);
    int64_t l = c == 0 ? lo : lo + step * c;  // p_{c-1} + 1
    int64_t h = c == 256 ? hi : lo + step * (c + 1) - 1;  // p_c
    if (h > hi) h = hi;
    const int64_t lo_d = d - nnz > 0 ? d - nnz : 0, hi_d = d < n_rows ? d : n_rows;
    if (l < lo_d) l = lo_d;
    if (h > hi_d) h = hi_d;
    if (l > h) l = h;
    return merge_search_warp_in(off, d, l, h);
}

// merge items per lane: 8 (256-item units); fp64 may use 4 (128-item units) to halve the
// per-lane arrays and raise the resident warps
#ifndef KP_MERGE_IPT64
#define KP_MERGE_IPT64 8
#endif
template <typename V>
constexpr int kMergeIPT = sizeof(V) == 8 ? KP_MERGE_IPT64 : kIPT;
// fp64: 3 CTAs (24 warps) in 80 registers -- with the values loaded late (kLateVals) the
// probe-ahead pipeline fits without spilling (with them pipelined it spilled ~150 B per
// thread at 80 registers and ran best at 2 CTAs).  fp32: 3 CTAs (<= 85
// registers; the kernel needs 71-80) with the larger L1 that leaves (merge_warps_per_sm):
// C2 85 us vs 89 us for 4 CTAs at 64 registers, band 27 263 vs 243 us -- the headline's
// random gathers want L1, regular streams want warps.  The fused-exchange fp32 variant
// keeps the compiler's allocation (~112 / 2 CTAs: faster on the DRAM-bound C5 shards,
// 916 vs 877 GB/s with a forced 4 CTAs).
#ifndef KP_MERGE_MINB_F32
#define KP_MERGE_MINB_F32 3
#endif
#ifndef KP_MERGE_MINB_F64
#define KP_MERGE_MINB_F64 3
#endif
// late values (see k_csr_merge): measured against values pipelined one unit ahead, per
// SpMV (min of 2, profiles/ab_merge_late_r02.txt): C2 WO 82.9 -> 80.9 us, C3 265 -> 253,
// band 27 259 -> 245, power-law 302 -> 288, C4 fp64 (3 CTAs instead of 2) 132 -> 128,
// band 27 fp64 415 -> 355, C5 equal
#ifndef KP_MERGE_LATE_F32
#define KP_MERGE_LATE_F32 1
#endif
#ifndef KP_MERGE_LATE_F64
#define KP_MERGE_LATE_F64 1
#endif
#ifndef KP_MERGE_MINB_F32B
#define KP_MERGE_MINB_F32B 3
#endif
template <typename V, bool kB = false>
constexpr int kMergeMinBlocks = sizeof(V) == 4 ? (kB ? KP_MERGE_MINB_F32B : KP_MERGE_MINB_F32) : KP_MERGE_MINB_F64;
constexpr int kMergeWarps = 8;        // warps per CTA

// Persistent merge-path warps (Merrill & Garland, restructured for B200).  The merge of
// A = row ends off[1..R] with B = nnz indices 0..Z-1 (row r's end item sits at merge
// position q_r = off[r+1] + r) is cut into units of 256 items; warp `wid` owns the
// contiguous RANGE of units [wid*upw, (wid+1)*upw), sized on the host so that one wave of
// warps covers the matrix (upw = units per warp).  The warp finds its first coordinate
// once (CSR,MP: from the K10 partition; CSR,WO: 32-ary warp search in-kernel) and then
// walks its units: each unit's row count comes from a ballot over the next row ends
// (q_r < d1), so no per-unit search or partition entry exists, and the open row's
// partial is carried to the next unit in a register.  Only the carry left open at a
// range end goes through k_carry_fixup (~one per warp instead of one per unit).
// Per unit: striped (coalesced) col/val loads of up to 256 nnz from j0 (speculative past
// the unit's nnz end; read-once, L1 no-allocate), x gathers, products staged in the
// warp's padded smem slice and read back blocked (lane l -> positions 8l..8l+7).  The
// probing lane of every row with elements in the unit sets the bit of the row's last
// position in a 256-bit mask (8 words per warp); each lane's byte of it gives its segment
// heads, a thread-local + warp segmented scan leaves every position's running row sum,
// which goes back into the same slice; the probing lanes then read their rows' sums at
// their last positions and store y coalesced (empty rows: 0).  The shared footprint is
// one product slice + 32 B per warp (8.7 KB per CTA fp32, 17 KB fp64): the gathers'
// miss tracking lives in L1, and the carveout the kernel leaves to L1 sets how many
// gathers an SM keeps in flight (merge_attrs sizes it).
template <typename V, typename O, bool kPrep, bool kB = false>
__global__ void __launch_bounds__(kMergeWarps * 32, kMergeMinBlocks<V, kB>) k_csr_merge(
    const O *__restrict__ off, const int32_t *__restrict__ col, const V *__restrict__ val, const V *__restrict__ x,
    V *__restrict__ y, int64_t n_rows, int64_t nnz, int64_t n_units, int64_t upw, int64_t n_ranges,
    const int64_t *__restrict__ part, int32_t *__restrict__ crow, V *__restrict__ cval, YDst<V> dst = YDst<V>{}) {
    constexpr int kI = kMergeIPT<V>, kT = 32 * kI;  // items per lane / per unit
    constexpr int kPad = kT + kT / 32;
    constexpr unsigned kLaneBits = kI == 32 ? 0xffffffffu : ((1u << kI) - 1u);
    __shared__ __align__(16) V s_prod[kMergeWarps][kPad];
    __shared__ unsigned s_last[kMergeWarps][2 * (kT / 32)];  // two row-last masks (units u, u+1)
    // let the PDL-launched carry fix-up be scheduled now: its griddepcontrol.wait still
    // waits for this grid's completion and memory flush, only the launch latency is hidden
    asm volatile("griddepcontrol.launch_dependents;");
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * kMergeWarps + w;
    int64_t r0 = 0;
    // CSR,WO: in-kernel start search, first round shared by the CTA (its grid of probes
    // lives in the product slices, dead until the barrier below).  Graph A/B against the
    // per-warp 32-ary search (per SpMV, same box): C4 fp64 149.5 -> 141.3 us, band 27
    // 282.6 -> 272.4 us, C2 equal, small inputs +0.2..0.7 us per iteration (the CTA
    // barrier); keeping both searches behind a size switch lost the large-input gain
    // (code generation of the main loop), so WO always uses this one.
    if constexpr (!kPrep) {
        static_assert(sizeof(s_prod) >= kMergeWarps * 32 * sizeof(int64_t), "search grid alias");
        int64_t *s_q = reinterpret_cast<int64_t *>(&s_prod[0][0]);
        const int64_t w0 = (int64_t)blockIdx.x * kMergeWarps;
        const int64_t wl = w0 + kMergeWarps - 1 < n_ranges - 1 ? w0 + kMergeWarps - 1 : n_ranges - 1;
        const int64_t wc = wid < n_ranges ? wid : wl;
        r0 = merge_search_cta(off, n_rows, nnz, wc * upw * kT, w0 * upw * kT, wl * upw * kT, s_q);
        __syncthreads();
    }
    if (wid >= n_ranges) return;
    const int64_t total = n_rows + nnz;
    const int64_t u_begin = wid * upw;
    const int64_t u_end = u_begin + upw < n_units ? u_begin + upw : n_units;
    V *prod = s_prod[w];
    unsigned *last = s_last[w];
    if (lane < 2 * (kT / 32)) last[lane] = 0u;
    __syncwarp();
    if (kPrep) r0 = part[wid];
    int64_t row_start = ldo(off + r0);  // r0 < n_rows: the range starts before the last item
    V carry = V(0);
    const int jb = lane * kI;
    // software pipeline: unit u+1's (col, val) loads are issued as soon as unit u's row count
    // fixes where they start, so their HBM latency overlaps unit u's gathers / scans
    // kLateVals: the window load pipelines only the columns (they address the gathers);
    // each unit loads its own values next to its gathers -- the values' registers are not
    // live across the previous unit (fp64: 16 registers)
    constexpr bool kLateVals = sizeof(V) == 8 ? KP_MERGE_LATE_F64 : KP_MERGE_LATE_F32;
    auto load_cv = [&](int64_t j0, int32_t (&c)[kI], V (&v)[kI]) {
        if (j0 + kT <= nnz) {  // common case: unpredicated, immediate offsets
            const int32_t *cp = col + j0 + lane;
            const V *vp = val + j0 + lane;
#pragma unroll
            for (int t = 0; t < kI; ++t) {
                c[t] = ld_stream(cp + t * 32);
                if constexpr (!kLateVals) v[t] = ld_stream(vp + t * 32);
            }
        } else {
#pragma unroll
            for (int t = 0; t < kI; ++t) {
                const int64_t j = j0 + lane + t * 32;
                c[t] = j < nnz ? ld_stream(col + j) : 0;
                if constexpr (!kLateVals) v[t] = j < nnz ? ld_stream(val + j) : V(0);
            }
        }
    };
    auto store_y = [&](int64_t r, V v) {
        if constexpr (kB) {
            // one destination (the accumulating column blocks, a 1-rank exchange): the
            // kernel's own y (== dst.y[dst.self]) -- the general put re-reads its pointer
            // table from the constant bank per store (ncu: +70 % constant-cache requests)
            if (dst.n == 1) st_y1(y + r, v);
            else dst.put(r, v);
        } else {
            y[r] = v;
        }
    };
    // Row-end probe of the unit [d0, d1) starting at row rs (rows before rs are finished):
    // rows ending inside it satisfy off[r+1] + r < d1 (monotone in r -> ballot + popc).
    // Row k (= rs + k) spans relative positions [s_k, e_k) of the unit's nnz window j0 =
    // d0 - rs: e_k = off[rs+k+1] - j0 in [0, nz], s_k = e_{k-1} (k = 0: its start, clipped).
    // The lane of every row with elements in the unit sets the bit of its last position in
    // mask `mk`; round 0's (e, s) stay in this lane's registers for the write-out.
    struct Probe {
        int nr;
        int e0, s0;
        int64_t end_re;  // off[rs + nr]: end of the last row ending in the unit (= its start if nr == 0)
    };
    auto probe = [&](int64_t rs, int64_t rs_start, int64_t d0, int64_t d1, unsigned *mk) {
        Probe q{0, 0, 0, rs_start};
        const int64_t j0 = d0 - rs;
        int64_t rr = rs + lane;
        int64_t re = rr < n_rows ? ldo(off + rr + 1) : INT64_MAX / 2;
        for (int round = 0;; ++round) {
            const bool in = rr < n_rows && re + rr < d1;
            const unsigned m = __ballot_sync(0xffffffffu, in);
            const int cnt = __popc(m);
            int64_t pe = __shfl_up_sync(0xffffffffu, re, 1);
            if (lane == 0) pe = q.end_re;
            if (in) {
                const int e = (int)(re - j0);
                const int st = pe > j0 ? (int)(pe - j0) : 0;
                if (e > st) atomicOr(&mk[(e - 1) >> 5], 1u << ((e - 1) & 31));  // row's last position
                if (round == 0) {
                    q.e0 = e;
                    q.s0 = st;
                }
            }
            if (cnt > 0) q.end_re = __shfl_sync(0xffffffffu, re, cnt - 1);
            q.nr += cnt;
            if (cnt < 32) break;
            rr += 32;
            re = rr < n_rows ? ldo(off + rr + 1) : INT64_MAX / 2;
        }
        return q;
    };
    // Software pipeline, one unit ahead: unit u+1's row-end probe and its (col, val) loads
    // are issued while unit u's gathers are in flight, so each unit starts with its row
    // count known -- its x gathers are predicated to its own nz elements (the window's
    // tail belongs to the next unit: no gather is issued twice) and its mask is already
    // built (two mask buffers per warp alternate).
    int32_t cn[kI];
    V vn[kI];
    int buf = 0;
    Probe cur{0, 0, 0, row_start};
    if (u_begin < u_end) {
        const int64_t d1 = u_begin * kT + kT < total ? u_begin * kT + kT : total;
        cur = probe(r0, row_start, u_begin * kT, d1, last);
        load_cv(u_begin * kT - r0, cn, vn);
    }
    for (int64_t u = u_begin; u < u_end; ++u) {
        const int64_t d0 = u * kT;
        const int64_t d1 = d0 + kT < total ? d0 + kT : total;
        const int64_t j0 = d0 - r0;
        const int nr = cur.nr;
        const int nz = (int)((d1 - d0) - nr);
        unsigned *mk = last + buf * (kT / 32);
        // x gathers of this unit's own elements only
        V p[kI];
        V vv[kI];
#pragma unroll
        for (int t = 0; t < kI; ++t) {
            const bool own = lane + t * 32 < nz;
            if constexpr (kLateVals) vv[t] = own ? ld_stream(val + j0 + lane + t * 32) : V(0);
            else vv[t] = vn[t];
            p[t] = own ? ld_x_merge(x + cn[t]) : V(0);
        }
        // accumulating stores (kp_spmv_bcast_acc): the first 32 rows' acc values load here,
        // next to the gathers, instead of as a dependent load in front of each store
        V a_pre = V(0);
        int32_t rr_pre = 0;  // this lane's first-round destination row (row map applied)
        if constexpr (kB) {
            if (lane < nr) {
                rr_pre = (int32_t)dst.row(r0 + lane);
                if (dst.acc) a_pre = ld_acc(dst.acc + rr_pre);
            }
        }
        // next unit: its (col, val) window and its row-end probe, overlapping the gathers
        Probe nxt{0, 0, 0, cur.end_re};
        if (u + 1 < u_end) {
            const int64_t r0n = r0 + nr;
            const int64_t d2 = d1 + kT < total ? d1 + kT : total;
            // fp32: the window loads first (their latency overlaps the probe); fp64 probes
            // first -- with the window's 24 registers live across the probe it spills
            if constexpr (sizeof(V) == 4) load_cv(d1 - r0n, cn, vn);
            nxt = probe(r0n, cur.end_re, d1, d2, last + (buf ^ 1) * (kT / 32));
            if constexpr (sizeof(V) != 4) load_cv(d1 - r0n, cn, vn);
        }
#pragma unroll
        for (int t = 0; t < kI; ++t) p[t] *= vv[t];
        if (nr == 0) {
            // the whole unit is one row's elements (long rows): no row ends, no marks, no
            // scans -- lane sums + a shuffle tree into the running carry (fixed order)
            V sum = V(0);
#pragma unroll
            for (int t = 0; t < kI; ++t) sum += p[t];
            carry += group_sum<32>(sum);
            cur = nxt;
            buf ^= 1;
            continue;
        }
        // stage products (positions >= nz are zero), read back blocked
#pragma unroll
        for (int t = 0; t < kI; ++t) {
            const int k = lane + t * 32;
            prod[k + (k >> 5)] = p[t];
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < kI; ++t) p[t] = prod[jb + t + ((jb + t) >> 5)];
        // segment heads: position 0, and every position after a row's last one
        const unsigned mine = (mk[jb >> 5] >> (jb & 31)) & kLaneBits;
        const unsigned prev_bits = __shfl_up_sync(0xffffffffu, mine, 1);
        const bool prev_last = lane == 0 || ((prev_bits >> (kI - 1)) & 1u);
        const unsigned heads_local = ((mine << 1) | (prev_last ? 1u : 0u)) & kLaneBits;
        // thread-local segmented scan
        V acc[kI];
#pragma unroll
        for (int t = 0; t < kI; ++t) acc[t] = ((heads_local >> t) & 1u || t == 0) ? p[t] : acc[t - 1] + p[t];
        const int first_head = heads_local ? __ffs(heads_local) - 1 : kI;
        // warp segmented scan of the lanes' last-segment sums; the head flags travel as
        // one ballot mask (lane l combines lane l-o unless a head lies in (l-o, l])
        V inc = acc[kI - 1];
        {
            const unsigned heads = __ballot_sync(0xffffffffu, heads_local != 0u);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const V up = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o && ((heads >> (lane - o + 1)) & ((1u << o) - 1u)) == 0) inc = up + inc;
            }
        }
        V cin = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane == 0) cin = V(0);
        __syncwarp();  // every lane has read its products and mask word
        // running row sums back into the slice (blocked); this unit's mask is cleared
#pragma unroll
        for (int t = 0; t < kI; ++t) prod[jb + t + ((jb + t) >> 5)] = t < first_head ? acc[t] + cin : acc[t];
        if (lane < kT / 32) mk[lane] = 0u;
        __syncwarp();
        // rows r0 .. r0+nr-1: the probing lanes read their sums at the rows' last positions
        // and store y coalesced; the open row's partial (after the last row end) is the carry
        for (int base = 0; base < nr; base += 32) {
            int e = cur.e0, st = cur.s0;
            if (base > 0) {  // rows past the first 32 (units of short / empty rows): re-probe (L1)
                const int64_t rq = r0 + base + lane;
                const int64_t rq_end = base + lane < nr ? ldo(off + rq + 1) : 0;
                int64_t pq = __shfl_up_sync(0xffffffffu, rq_end, 1);
                if (lane == 0) pq = ldo(off + r0 + base);
                e = (int)(rq_end - j0);
                st = pq > j0 ? (int)(pq - j0) : 0;
            }
            if (base + lane < nr) {
                V v = e > st ? prod[(e - 1) + ((e - 1) >> 5)] : V(0);
                if (base + lane == 0) v += carry;
                int64_t rr = r0 + base + lane;
                if constexpr (kB) {
                    rr = base == 0 ? (int64_t)rr_pre : dst.row(rr);
                    if (dst.acc) v += base == 0 ? a_pre : ld_acc(dst.acc + rr);
                }
                store_y(rr, v);
            }
        }
        const int e_last = (int)(cur.end_re - j0);
        carry = e_last < nz ? prod[(nz - 1) + ((nz - 1) >> 5)] : V(0);
        r0 += nr;
        cur = nxt;
        buf ^= 1;
        __syncwarp();
    }
    if (lane == 0) {
        const bool open = r0 < n_rows;
        crow[wid] = open ? (int32_t)r0 : -1;
        cval[wid] = open ? carry : V(0);
    }
}

// K10: merge-path partition = the first coordinate of every warp range (one warp per
// range, 32-ary search over the row ends; O(#ranges) ~ one wave of warps, independent
// of the matrix size).  part[n_ranges] = n_rows.
template <typename O, int kT>
__global__ void __launch_bounds__(256) k_prep_mp(const O *__restrict__ off, int64_t n_rows, int64_t nnz,
                                                 int64_t upw, int64_t n_ranges, int64_t *__restrict__ part) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid > n_ranges) return;
    const int64_t total = n_rows + nnz;
    int64_t d = wid * upw * kT;
    if (d > total) d = total;
    const int64_t r = merge_search_warp(off, n_rows, nnz, d);
    if ((threadIdx.x & 31) == 0) part[wid] = wid == n_ranges ? n_rows : r;
}

// ================================================================= COO,WM (K8 + K11)
// Persistent warps over row-sorted COO: warp `wid` owns the contiguous RANGE of 256-nnz
// chunks [wid*cpw, (wid+1)*cpw) (cpw sized on the host so one wave of resident warps covers
// the matrix); lane l holds the chunk's 8 nnz at [base + 8l, base + 8l + 8) (blocked;
// 32-byte vector loads of row ids and cols).  Warp segmented scan by row id; a row
// finished inside the chunk is written, the row open at the chunk end carries to the next
// chunk in a register, and only the row open at the RANGE end goes through k_carry_fixup.
// Empty rows (gaps between consecutive row ids) are zero-filled by the element that
// follows the gap, so y needs no memset.
// fp32: 5 CTAs (40 warps) per SM in 48 registers without spills (C2 107 -> 95 us, band-27
// 0.50 -> 0.70 of HBM); fp64 keeps 64 registers (48 spills and runs slower)
template <typename V>
constexpr int kCooMinBlocks = sizeof(V) == 4 ? 5 : 4;
template <typename V, bool kVec>
__global__ void __launch_bounds__(256, kCooMinBlocks<V>) k_coo_wm(const int32_t *__restrict__ rid, const int32_t *__restrict__ col,
                                                const V *__restrict__ val, const V *__restrict__ x,
                                                V *__restrict__ y, int64_t n_rows, int64_t nnz, int64_t n_chunks,
                                                int64_t cpw, int64_t n_ranges, int32_t *__restrict__ crow,
                                                V *__restrict__ cval) {
    asm volatile("griddepcontrol.launch_dependents;");  // early PDL trigger (see k_csr_merge)
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= n_ranges) return;
    const int64_t c_begin = wid * cpw;
    const int64_t c_end = c_begin + cpw < n_chunks ? c_begin + cpw : n_chunks;
    // row of the element before the range, and the partial of that row accumulated inside
    // this range (0 at the range start: earlier ranges publish their own carries)
    int32_t prow = c_begin > 0 ? __ldg(rid + c_begin * kCooChunk - 1) : -1;
    V carry = V(0);
    bool open = false;
    // chunk loader: 32-byte vector loads for full chunks, predicated scalars for the last
    auto load = [&](int64_t base, int32_t (&r)[kIPT], int32_t (&c)[kIPT], V (&v)[kIPT]) {
        const int64_t j0 = base + lane * kIPT;
        if (kVec && base + kCooChunk <= nnz) {
            const int4 *rp = reinterpret_cast<const int4 *>(rid + j0);
            const int4 *cp = reinterpret_cast<const int4 *>(col + j0);
            const int4 ra = ld_stream4(rp), rb = ld_stream4(rp + 1);
            const int4 ca = ld_stream4(cp), cb = ld_stream4(cp + 1);
            r[0] = ra.x; r[1] = ra.y; r[2] = ra.z; r[3] = ra.w; r[4] = rb.x; r[5] = rb.y; r[6] = rb.z; r[7] = rb.w;
            c[0] = ca.x; c[1] = ca.y; c[2] = ca.z; c[3] = ca.w; c[4] = cb.x; c[5] = cb.y; c[6] = cb.z; c[7] = cb.w;
            const int4 *vp = reinterpret_cast<const int4 *>(val + j0);  // 8 values = 2 (fp32) / 4 (fp64) x 16 B
#pragma unroll
            for (int q = 0; q < (int)(kIPT * sizeof(V) / 16); ++q) {
                const int4 w = ld_stream4(vp + q);
                memcpy(&v[q * 16 / sizeof(V)], &w, 16);
            }
        } else {
#pragma unroll
            for (int k = 0; k < kIPT; ++k) {
                const int64_t j = j0 + k;
                r[k] = j < nnz ? ld_stream(rid + j) : INT32_MAX;  // sentinel past the end: never written
                c[k] = j < nnz ? ld_stream(col + j) : 0;
                v[k] = j < nnz ? ld_stream(val + j) : V(0);
            }
        }
    };
    for (int64_t chunk = c_begin; chunk < c_end; ++chunk) {
        const int64_t base = chunk * kCooChunk;
        const int64_t j0 = base + lane * kIPT;
        int32_t r[kIPT];
        V p[kIPT];
        const bool full = base + kCooChunk <= nnz;
        {
            int32_t c[kIPT];
            V vv[kIPT];
            load(base, r, c, vv);
#pragma unroll
            for (int k = 0; k < kIPT; ++k) p[k] = vv[k] * ld_x(x + c[k]);
        }
        // first row of the next chunk (row-end test of the chunk's last element)
        const int32_t nxt_chunk = (lane == 31 && base + kCooChunk < nnz) ? __ldg(rid + base + kCooChunk) : INT32_MAX;
        int32_t prev = __shfl_up_sync(0xffffffffu, r[kIPT - 1], 1);
        if (lane == 0) prev = prow;
        int32_t next = __shfl_down_sync(0xffffffffu, r[0], 1);
        if (lane == 31) next = nxt_chunk;
        // thread-local segmented inclusive scan; elements before the lane's first head
        // continue the previous lane's segment (carry_in from the warp scan below)
        V acc[kIPT];
        int first_head_k = kIPT;
        {
            int32_t pr = prev;
#pragma unroll
            for (int k = 0; k < kIPT; ++k) {
                const bool head = r[k] != pr;
                if (head && first_head_k == kIPT) first_head_k = k;
                acc[k] = (head || k == 0) ? p[k] : acc[k - 1] + p[k];
                pr = r[k];
            }
        }
        // warp segmented scan of the lanes' last-segment sums (head flags as a ballot mask)
        V inc = acc[kIPT - 1];
        {
            const unsigned heads = __ballot_sync(0xffffffffu, first_head_k < kIPT);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const V up = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o && ((heads >> (lane - o + 1)) & ((1u << o) - 1u)) == 0) inc = up + inc;
            }
        }
        V carry_in = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane == 0) carry_in = V(0);
        // gap fill + row ends
        int32_t pr = prev;
        V vlast = V(0);
#pragma unroll
        for (int k = 0; k < kIPT; ++k) {
            const int32_t rk = r[k];
            if (rk != INT32_MAX) {
                for (int64_t g = (int64_t)pr + 1; g < rk; ++g) y[g] = V(0);  // rows strictly between are empty
                const int32_t nx = (k + 1 < kIPT) ? r[k + 1] : next;
                V v = (k < first_head_k) ? acc[k] + carry_in : acc[k];
                if (rk == prow) v += carry;  // row continued from the previous chunk of this range
                if (nx != rk) y[rk] = v;     // row ends here
                if (j0 + k == nnz - 1)       // trailing empty rows after the very last nnz
                    for (int64_t g = (int64_t)rk + 1; g < n_rows; ++g) y[g] = V(0);
                vlast = v;
                pr = rk;
            }
        }
        // the row open at the chunk end carries to the next chunk (lane 31 holds it)
        const int32_t rl = __shfl_sync(0xffffffffu, r[kIPT - 1], 31);
        open = __shfl_sync(0xffffffffu, next == r[kIPT - 1] && full && base + kCooChunk < nnz, 31);
        carry = open ? __shfl_sync(0xffffffffu, vlast, 31) : V(0);
        prow = rl;
    }
    if (lane == 0) {
        crow[wid] = open ? prow : -1;
        cval[wid] = open ? carry : V(0);
    }
}

// K11: CSR -> COO row ids.  One CTA per 2048 consecutive nnz: the rows that START
// inside the window are the contiguous range [ra, rb) (two binary searches), each
// marks its start position in shared memory (atomicMax picks the last of several rows
// sharing an offset, i.e. the non-empty one), and a block max-scan seeded with the
// row containing the window's first element fills every position.  Reads the
// offsets once and writes each row id once (vectorised), no per-element search.
constexpr int kCooPrepIPT = 16;                      // row ids per thread
constexpr int kCooPrepItems = 256 * kCooPrepIPT;  // 4096 nnz per CTA tile

template <typename O>
__device__ __forceinline__ int64_t upper_bound_off(const O *off, int64_t n_rows, int64_t v) {
    int64_t lo = 0, hi = n_rows + 1;  // first index in off[0..n_rows] with off[i] > v
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ldo(off + mid) <= v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Pass 1: c0[b] = row containing element b*2048, scattered by the rows themselves (a
// non-empty row r covers the block starts in [off[r], off[r+1])): one coalesced pass over
// the offsets, each block start written exactly once, no searches.
template <typename O>
__global__ void __launch_bounds__(256) k_prep_coo_starts(const O *__restrict__ off, int64_t n_rows,
                                                         int32_t *__restrict__ c0) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rows) return;
    const int64_t a = ldo(off + r), e = ldo(off + r + 1);
    for (int64_t b = (a + kCooPrepItems - 1) / kCooPrepItems; b * kCooPrepItems < e; ++b) c0[b] = (int32_t)r;
}

// Pass 2: the rows starting inside block b are (c0[b], c0[b+1]] (non-empty ones; empty
// rows in between share offsets and lose the atomicMax to the non-empty row).
template <typename O>
__global__ void __launch_bounds__(256) k_prep_coo(const O *__restrict__ off, int64_t n_rows, int64_t nnz,
                                                  const int32_t *__restrict__ c0s, int32_t *__restrict__ rid) {
    constexpr int P = kCooPrepIPT;
    // marks padded one slot per 32 so the blocked read (thread t: slots P*t .. P*t+P-1) is
    // bank-conflict free
    __shared__ int32_t s_mark[kCooPrepItems + kCooPrepItems / 32];
    __shared__ int32_t s_wmax[8];
    const int64_t j0 = (int64_t)blockIdx.x * kCooPrepItems;
    const int64_t j1 = j0 + kCooPrepItems < nnz ? j0 + kCooPrepItems : nnz;
    const int64_t nb = (nnz + kCooPrepItems - 1) / kCooPrepItems;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t c0 = c0s[blockIdx.x];  // row containing j0
    const int64_t ra = c0 + 1;
    const int64_t rb = blockIdx.x + 1 < nb ? (int64_t)c0s[blockIdx.x + 1] + 1 : n_rows;
    for (int k = tid; k < kCooPrepItems; k += 256) s_mark[k + (k >> 5)] = -1;
    __syncthreads();
    for (int64_t r = ra + tid; r < rb; r += 256) {
        const int64_t o = ldo(off + r);
        if (o < j1) {
            const int k = (int)(o - j0);
            atomicMax(&s_mark[k + (k >> 5)], (int32_t)r);
        }
    }
    __syncthreads();
    // blocked max-scan: thread t owns positions P*t .. P*t+P-1
    int32_t v[P];
    int32_t m = -1;
#pragma unroll
    for (int i = 0; i < P; ++i) {
        const int k = tid * P + i;
        const int32_t q = s_mark[k + (k >> 5)];
        m = q > m ? q : m;
        v[i] = m;
    }
    int32_t inc = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = t > inc ? t : inc;
    }
    if (lane == 31) s_wmax[w] = inc;
    __syncthreads();
    int32_t carry = (int32_t)c0;
    for (int i = 0; i < w; ++i) carry = s_wmax[i] > carry ? s_wmax[i] : carry;
    int32_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane > 0) carry = ex > carry ? ex : carry;
#pragma unroll
    for (int i = 0; i < P; ++i) v[i] = v[i] > carry ? v[i] : carry;
    const int64_t jb = j0 + tid * P;
    if (jb + P <= j1) {
        int4 *dst = reinterpret_cast<int4 *>(rid + jb);
#pragma unroll
        for (int q = 0; q < P / 4; ++q) dst[q] = make_int4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < P; ++i)
            if (jb + i < j1) rid[jb + i] = v[i];
    }
}

// ================================================================= Adaptive-CSR (K13)
// Units: a "short block" of consecutive rows (each <= kAdLongT nnz) whose starts fall in
// one kAdBlockNnz window and one kAdRows row window, or one kAdLongChunk piece of a
// long row.  unit_row[u] = first row; unit_piece[u] = -1 (short) or piece index.
// The short block's last row is unit_row[u+1] (or n_rows).
template <typename O>
__device__ __forceinline__ int64_t ad_units_of_row(const O *off, int64_t r, int64_t n_rows) {
    const int64_t len = ldo(off + r + 1) - ldo(off + r);
    if (len > kAdLongT) return (len + kAdLongChunk - 1) / kAdLongChunk;
    if (r == 0) return 1;
    const int64_t plen = ldo(off + r) - ldo(off + r - 1);
    if (plen > kAdLongT) return 1;
    if (r % kAdRows == 0) return 1;
    if (ldo(off + r) / kAdBlockNnz != ldo(off + r - 1) / kAdBlockNnz) return 1;
    return 0;
}

constexpr int kScanItems = 256 * 16;  // rows per scan block

template <typename O>
__global__ void __launch_bounds__(256) k_ad_count(const O *__restrict__ off, int64_t n_rows,
                                                  int64_t *__restrict__ bsum) {
    __shared__ int64_t sw[8];
    const int64_t r0 = (int64_t)blockIdx.x * kScanItems;
    int64_t c = 0;
    for (int k = threadIdx.x; k < kScanItems; k += 256) {
        const int64_t r = r0 + k;
        if (r < n_rows) c += ad_units_of_row(off, r, n_rows);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int i = 0; i < 8; ++i) t += sw[i];
        bsum[blockIdx.x] = t;
    }
}

// single CTA: exclusive scan of block sums in place, total -> *total
__global__ void __launch_bounds__(1024) k_scan_bsum(int64_t *__restrict__ bsum, int64_t nb, int64_t *__restrict__ total) {
    __shared__ int64_t sw[32];
    __shared__ int64_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
        const int64_t i = b0 + threadIdx.x;
        const int64_t v = i < nb ? bsum[i] : 0;
        int64_t inc = v;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) sw[w] = inc;
        __syncthreads();
        if (w == 0) {
            int64_t wv = sw[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int64_t t = __shfl_up_sync(0xffffffffu, wv, o);
                if (lane >= o) wv += t;
            }
            sw[lane] = wv;
        }
        __syncthreads();
        const int64_t excl = s_carry + (w > 0 ? sw[w - 1] : 0) + inc - v;
        if (i < nb) bsum[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = s_carry;
}

template <typename O>
__global__ void __launch_bounds__(256) k_ad_write(const O *__restrict__ off, int64_t n_rows,
                                                  const int64_t *__restrict__ bsum, int32_t *__restrict__ urow,
                                                  int32_t *__restrict__ upiece) {
    // each thread owns 16 consecutive rows of the block (blocked), scans locally
    __shared__ int64_t sw[8];
    constexpr int kPer = kScanItems / 256;
    const int64_t r0 = (int64_t)blockIdx.x * kScanItems + threadIdx.x * kPer;
    int64_t cnt[kPer];
    int64_t tsum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int64_t r = r0 + k;
        cnt[k] = r < n_rows ? ad_units_of_row(off, r, n_rows) : 0;
        tsum += cnt[k];
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t inc = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) sw[w] = inc;
    __syncthreads();
    int64_t wpre = 0;
    for (int i = 0; i < w; ++i) wpre += sw[i];
    int64_t u = bsum[blockIdx.x] + wpre + inc - tsum;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int64_t r = r0 + k;
        if (cnt[k] == 0) continue;
        const int64_t len = ldo(off + r + 1) - ldo(off + r);
        if (len > kAdLongT) {
            for (int64_t q = 0; q < cnt[k]; ++q) { urow[u + q] = (int32_t)r; upiece[u + q] = (int32_t)q; }
        } else {
            urow[u] = (int32_t)r;
            upiece[u] = -1;
        }
        u += cnt[k];
    }
}

template <typename V, typename O>
struct AdSmem {
    V prod[kAdCap];
    int64_t roff[kAdRows + 1];
    V sred[32];
};

template <typename V, typename O>
__global__ void __launch_bounds__(256) k_adaptive(const O *__restrict__ off, const int32_t *__restrict__ col,
                                                  const V *__restrict__ val, const V *__restrict__ x,
                                                  V *__restrict__ y, int64_t n_rows,
                                                  const int32_t *__restrict__ urow, const int32_t *__restrict__ upiece,
                                                  const int64_t *__restrict__ n_units_dev, int32_t *__restrict__ crow,
                                                  V *__restrict__ cval) {
    __shared__ AdSmem<V, O> sm;
    const int64_t U = *n_units_dev;
    for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
        const int64_t ra = urow[u];
        const int32_t pc = upiece[u];
        if (pc >= 0) {
            // vector-L piece of a long row
            const int64_t rs = ldo(off + ra), re = ldo(off + ra + 1);
            const int64_t s = rs + (int64_t)pc * kAdLongChunk;
            const int64_t e = s + kAdLongChunk < re ? s + kAdLongChunk : re;
            V sum = 0;
            int64_t j = s + threadIdx.x;
            for (; j + 3 * 256 < e; j += 4 * 256) {
                const int32_t c0 = ld_stream(col + j), c1 = ld_stream(col + j + 256), c2 = ld_stream(col + j + 512),
                              c3 = ld_stream(col + j + 768);
                const V v0 = ld_stream(val + j), v1 = ld_stream(val + j + 256), v2 = ld_stream(val + j + 512),
                        v3 = ld_stream(val + j + 768);
                sum = fma_acc(sum, v0, ld_x(x + c0));
                sum = fma_acc(sum, v1, ld_x(x + c1));
                sum = fma_acc(sum, v2, ld_x(x + c2));
                sum = fma_acc(sum, v3, ld_x(x + c3));
            }
            for (; j < e; j += 256) sum = fma_acc(sum, ld_stream(val + j), ld_x(x + ld_stream(col + j)));
            const V t = block_sum(sum, sm.sred);
            if (threadIdx.x == 0) {
                const int64_t npieces = (re - rs + kAdLongChunk - 1) / kAdLongChunk;
                if (npieces == 1) {
                    y[ra] = t;
                    crow[u] = -1;
                } else if (pc == npieces - 1) {
                    y[ra] = t;  // finishing piece writes; earlier pieces are carries
                    crow[u] = -1;
                } else {
                    crow[u] = (int32_t)ra;
                    cval[u] = t;
                }
            }
        } else {
            const int64_t rb = (u + 1 < U) ? (int64_t)urow[u + 1] : n_rows;
            const int nrows = (int)(rb - ra);
            const int64_t s = ldo(off + ra);
            for (int k = threadIdx.x; k <= nrows; k += 256) sm.roff[k] = ldo(off + ra + k) - s;
            const int nz = (int)(ldo(off + rb) - s);
            for (int b = 0; b < nz; b += 256 * 6) {  // 6 independent (col, val) pairs per thread
                int32_t c[6];
                V v[6];
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const int k = b + threadIdx.x + i * 256;
                    c[i] = k < nz ? ld_stream(col + s + k) : 0;
                    v[i] = k < nz ? ld_stream(val + s + k) : V(0);
                }
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const int k = b + threadIdx.x + i * 256;
                    if (k < nz) sm.prod[k] = v[i] * ld_x(x + c[i]);
                }
            }
            if (threadIdx.x == 0) crow[u] = -1;
            __syncthreads();
            // G lanes per row, G = min(32, pow2floor(256 / nrows))
            int G = 1;
            while (G < 32 && G * 2 * nrows <= 256) G <<= 1;
            const int grp = threadIdx.x / G, gl = threadIdx.x % G;
            V sum = 0;
            if (grp < nrows) {
                const int a = (int)sm.roff[grp], b = (int)sm.roff[grp + 1];
                for (int k = a + gl; k < b; k += G) sum += sm.prod[k];
            }
            // reduce inside groups (G is CTA-uniform; groups never straddle warps)
            for (int o = 1; o < G; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if (grp < nrows && gl == 0) y[ra + grp] = sum;
        }
        __syncthreads();
    }
}

// ================================================================= shard partition (K14)
template <typename O>
__global__ void k_shard_partition(const O *__restrict__ off, int64_t n_rows, int32_t parts, int64_t *__restrict__ cuts) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > parts) return;
    const int64_t nnz = ldo(off + n_rows);
    if (p == parts) { cuts[p] = n_rows; return; }
    const int64_t target = (int64_t)((__int128)p * nnz / parts);
    int64_t lo = 0, hi = n_rows;  // lower_bound(off[0..n_rows], target)
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ldo(off + mid) < target) lo = mid + 1;
        else hi = mid;
    }
    cuts[p] = lo;
}

// ================================================================= host helpers
int wm_group(const kp_csr *A) {
    // G lanes per row so that each lane issues ~U = 4 independent (col, val) pairs per
    // row (batch_dot): G = clamp(pow2 >= mean / 4, 2, 32), from the KNOWN mean nnz/rows.
    const double mean = A->n_rows > 0 ? (double)A->nnz / (double)A->n_rows : 0.0;
    int G = 2;
    while (G < 32 && G * 4 < mean) G <<= 1;
    return G;
}

// CSR,TM stage capacity (nnz): the short-row default, or -- when 256 rows of the KNOWN mean
// length overflow it -- a stage sized for 256 rows with 25 % slack (up to kCapMax).
template <typename V, typename O>
int tm_capacity(const kp_csr *A) {
    using Cfg = TmCfg<V, O>;
    const double mean = A->n_rows > 0 ? (double)A->nnz / (double)A->n_rows : 1.0;
    const double need = 1.25 * kTmRows * mean + 128;
    if (need <= Cfg::kCap) return Cfg::kCap;
    const int64_t c = ((int64_t)need + 127) / 128 * 128;
    return (int)(c < Cfg::kCapMax ? c : Cfg::kCapMax);
}

// CSR,TM rows per thread: tile window ~3/4 of a stage at the KNOWN mean row length.
int tm_rows_per_thread(const kp_csr *A, int cap) {
    const double mean = A->n_rows > 0 ? (double)A->nnz / (double)A->n_rows : 1.0;
    int rpt = 1;
    while (rpt < kTmMaxRpt && 2.0 * rpt * kTmRows * (mean > 1 ? mean : 1.0) <= 0.75 * cap) rpt <<= 1;
    return rpt;
}

int64_t merge_tile_items(const kp_csr *A) { return 32 * (A->val_type == KP_F64 ? kMergeIPT<double> : kMergeIPT<float>); }
int64_t merge_tiles(const kp_csr *A) { return (A->n_rows + A->nnz + merge_tile_items(A) - 1) / merge_tile_items(A); }
// Persistent merge geometry: units of 256 merge items, `upw` consecutive units per warp so
// that one wave of resident warps (occupancy API, cached per instantiation) covers the
// matrix.  Used identically by the K10 partition and the SpMV launch.
struct MergeGeom {
    int64_t n_units, upw, n_ranges;
};
template <typename V, typename O>
int merge_warps_per_sm() {
    // Residency and carveout together: the register budget (launch bounds) fixes how many
    // CTAs fit; the shared-memory carveout is then the SMALLEST configuration that holds
    // them, so L1 -- where the x gathers' misses are tracked -- gets the rest (a carveout
    // left to the driver let the CTAs outnumber what was resident: a second partial wave
    // of the persistent grid, and a 132-228 KB carve starved the gathers).  Measured on
    // the v2 kernel, per SpMV (min of 2): C2 fp32 carve 32 KB 85.0 us vs 87.0 driver default
    // (old kernel 93.2), band 27 263 us (273); C4 fp64 64 KB 140 us, C2 fp64 105 us.
    // Per device (the attribute is per context); KP_MERGE_CARVE=<percent> overrides (A/B).
    static int warps_per_sm[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    dev &= 63;
    if (!warps_per_sm[dev]) {
        void (*fns[4])(const O *, const int32_t *, const V *, const V *, V *, int64_t, int64_t, int64_t, int64_t,
                       int64_t, const int64_t *, int32_t *, V *, YDst<V>) = {
            k_csr_merge<V, O, true>, k_csr_merge<V, O, false>, k_csr_merge<V, O, true, true>,
            k_csr_merge<V, O, false, true>};
        const char *cv = getenv("KP_MERGE_CARVE");
        for (auto f : fns) {
            int nb = 0, pc = cv ? atoi(cv) : -1;
            cudaFuncAttributes fa = {};
            if (pc < 0 && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kMergeWarps * 32, 0) == cudaSuccess &&
                nb > 0 && cudaFuncGetAttributes(&fa, f) == cudaSuccess) {
                const size_t need = (size_t)nb * (fa.sharedSizeBytes + 1024);  // + the per-CTA reserve
                int smem_max = 0;
                cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
                if (smem_max <= 0) smem_max = 228 * 1024;
                pc = (int)((need * 100 + smem_max - 1) / smem_max);
                if (pc > 100) pc = 100;
            }
            if (pc >= 0) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pc);
        }
        cudaGetLastError();
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_csr_merge<V, O, true>, kMergeWarps * 32, 0) !=
                cudaSuccess ||
            nb <= 0) {
            cudaGetLastError();
            nb = 3;
        }
        warps_per_sm[dev] = nb * kMergeWarps;
    }
    return warps_per_sm[dev];
}
int64_t g_wave_warps = 0;  // kp_debug_set_wave_warps (0 = occupancy-derived)
// Persistent-kernel wave: every resident warp.  (Halving it when x exceeds L2 helped
// random gathers that miss to DRAM -- C5 merge 10.47 -> 10.12 ms -- but cost banded
// matrices with a large x 35-50 % (band-4, 32 M rows: merge 466 -> 716 us), and the
// gather locality is not known at launch; reverted.)
int64_t wave_target(const kp_csr *, size_t, int warps_per_sm) { return (int64_t)num_sms() * warps_per_sm; }
template <typename V, typename O>
MergeGeom merge_geom(const kp_csr *A) {
    const int warps_per_sm = merge_warps_per_sm<V, O>();
    MergeGeom G;
    G.n_units = merge_tiles(A);
    const int64_t target = g_wave_warps > 0 ? g_wave_warps : wave_target(A, sizeof(V), warps_per_sm);
    G.upw = (G.n_units + target - 1) / target;
    if (G.upw < 1) G.upw = 1;
    G.n_ranges = (G.n_units + G.upw - 1) / G.upw;
    return G;
}
int64_t coo_chunks(const kp_csr *A) { return (A->nnz + kCooChunk - 1) / kCooChunk; }
template <typename V>
MergeGeom coo_geom(const kp_csr *A) {
    static int warps_per_sm = 0;
    if (!warps_per_sm) {
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_coo_wm<V, true>, 256, 0) != cudaSuccess || nb <= 0) {
            cudaGetLastError();
            nb = 8;
        }
        warps_per_sm = nb * 8;
    }
    MergeGeom G;
    G.n_units = coo_chunks(A);
    const int64_t target = g_wave_warps > 0 ? g_wave_warps : wave_target(A, sizeof(V), warps_per_sm);
    G.upw = (G.n_units + target - 1) / target;
    if (G.upw < 1) G.upw = 1;
    G.n_ranges = (G.n_units + G.upw - 1) / G.upw;
    return G;
}
int64_t ad_units_max(const kp_csr *A) {
    return A->n_rows + A->nnz / kAdLongChunk + 2;
}
int64_t ad_scan_blocks(const kp_csr *A) { return (A->n_rows + kScanItems - 1) / kScanItems; }

bool valid_csr(const kp_csr *A) {
    if (!A || A->n_rows < 0 || A->n_cols < 0 || A->nnz < 0) return false;
    if (A->off_type != KP_I32 && A->off_type != KP_I64) return false;
    if (A->val_type != KP_F32 && A->val_type != KP_F64) return false;
    if (A->n_rows >= INT32_MAX || A->n_cols > INT32_MAX) return false;
    if (A->off_type == KP_I32 && A->nnz >= INT32_MAX) return false;
    if (!A->row_offsets) return false;
    if (A->nnz > 0 && (!A->col_indices || !A->values)) return false;
    return true;
}

size_t val_bytes(const kp_csr *A) { return A->val_type == KP_F32 ? 4 : 8; }

struct Layout {
    size_t hdr = 0, red = 0, a = 0, b = 0, c = 0, total = 0;
};

// ELL tail list capacity: at most nnz / (cap + 1) rows are longer than W >= cap ... or,
// when W = max_len < cap, none
int64_t ell_tail_slots(const kp_csr *A, int64_t cap) { return A->nnz / (cap + 1) + 1; }

Layout prep_layout(int32_t kernel, const kp_csr *A, int64_t cap) {
    Layout L;
    size_t o = align_up(sizeof(PrepHeader));
    switch (kernel) {
        case KP_ELL_TM: {
            L.red = o; o += align_up(kRedWsBytes);
            const size_t rpad = (size_t)((A->n_rows + 31) / 32 * 32);
            L.a = o; o += align_up((size_t)cap * rpad * sizeof(int32_t));
            L.b = o; o += align_up((size_t)cap * rpad * val_bytes(A));
            // tail list: rows longer than W >= ... at most nnz / (cap + 1) of them
            L.c = o; o += align_up((size_t)ell_tail_slots(A, cap) * sizeof(int64_t));
            break;
        }
        case KP_COO_WM:
            L.a = o; o += align_up((size_t)A->nnz * sizeof(int32_t) + 64);
            L.b = o; o += align_up((size_t)((A->nnz + kCooPrepItems - 1) / kCooPrepItems + 1) * sizeof(int32_t));
            break;
        case KP_CSR_MP: L.a = o; o += align_up((size_t)(merge_tiles(A) + 1) * sizeof(int64_t)); break;
        case KP_ADAPTIVE_CSR: {
            const int64_t U = ad_units_max(A);
            L.a = o; o += align_up((size_t)U * sizeof(int32_t));
            L.b = o; o += align_up((size_t)U * sizeof(int32_t));
            L.c = o; o += align_up((size_t)(ad_scan_blocks(A) + 1) * sizeof(int64_t));
            break;
        }
        default: break;
    }
    L.total = o;
    return L;
}

// Long-row threshold of the row-mapped schedules (DeferWs): WM lists rows longer than 64
// lanes-worth of its group (16 batches of 4 per lane), TM rows longer than 128 elements;
// both from the KNOWN shape only.  INT64_MAX (no list, no tail launch) when no
// row can be that long (n_cols <= T).
int64_t long_threshold(int32_t kernel, const kp_csr *A) {
    static const bool off = [] {  // KP_NO_LONG_ROWS=1: A/B switch (the pre-deferral schedules)
        const char *e = getenv("KP_NO_LONG_ROWS");
        return e && e[0] == '1';
    }();
    if (off) return INT64_MAX;
    int64_t t = INT64_MAX;
    if (kernel == KP_CSR_WM) {
        static const int64_t wm_m = [] {  // KP_WM_LONG_MULT overrides (A/B)
            const char *e = getenv("KP_WM_LONG_MULT");
            return e ? (int64_t)atoll(e) : (int64_t)64;
        }();
        t = wm_m * (int64_t)wm_group(A);
    }
    else if (kernel == KP_CSR_TM) {
        // a thread walking more than ~32 batches of 4 is the pitfall whatever the mean (dense
        // bands ran 120x behind BM).  A/B of the threshold (profiles/ab_tm_long_r02.txt, per
        // SpMV): 256 -> 128: C2 216 -> 174 us, band 300 108 -> 22 us, power-law 503 -> 443 us,
        // C3 / band 27 / stencils unchanged; 64 cost C3 1 %.  KP_TM_LONG overrides (A/B).
        static const int64_t tm_t = [] {
            const char *e = getenv("KP_TM_LONG");
            return e ? (int64_t)atoll(e) : (int64_t)128;
        }();
        t = tm_t;
    }
    return t < A->n_cols ? t : INT64_MAX;
}
// list capacity: rows past T (at most nnz / (T + 1)), then the huge rows past kLongCta
int64_t long_huge_at(int32_t kernel, const kp_csr *A) {
    const int64_t t = long_threshold(kernel, A);
    return t == INT64_MAX ? 0 : A->nnz / (t + 1) + 1;
}
int64_t long_giant_at(int32_t kernel, const kp_csr *A) {
    const int64_t h = long_huge_at(kernel, A);
    return h ? h + A->nnz / (kLongCta + 1) + 1 : 0;
}
int64_t long_slots(int32_t kernel, const kp_csr *A) {
    const int64_t g = long_giant_at(kernel, A);
    return g ? g + A->nnz / (kLongGiant + 1) + 1 : 0;
}

int64_t spmv_units(int32_t kernel, const kp_csr *A) {
    switch (kernel) {
        case KP_CSR_MP:
        case KP_CSR_WO: return merge_tiles(A);
        case KP_COO_WM: return coo_chunks(A);
        case KP_ADAPTIVE_CSR: return ad_units_max(A);
        default: return 0;
    }
}

template <typename V, typename O>
int prepare_t(int32_t kernel, const kp_csr *A, int64_t cap, unsigned char *buf, const Layout &L, kp_prepared *P,
              cudaStream_t s) {
    PrepHeader *hdr = reinterpret_cast<PrepHeader *>(buf);
    const O *off = reinterpret_cast<const O *>(A->row_offsets);
    const V *val = reinterpret_cast<const V *>(A->values);
    switch (kernel) {
        case KP_ELL_TM: {
            // header written by a kernel (no host-memory copy: plans capture this into a graph)
            k_prep_hdr<<<1, 1, 0, s>>>(hdr, kernel, cap);
            KP_LAUNCHED();
            KP_CUDA_TRY(cudaMemsetAsync(buf + L.red, 0, kRedWsBytes, s));
            int rc = launch_k1_stats_into(A->row_offsets, A->off_type, A->n_rows, hdr->stats, buf + L.red, s);
            if (rc) return rc;
            const int64_t g = (A->n_rows + 255) / 256;
            if (g > 0) {
                k_prep_ell<V, O><<<(unsigned)g, 256, 0, s>>>(hdr, off, A->col_indices, val,
                                                              reinterpret_cast<int32_t *>(buf + L.a),
                                                              reinterpret_cast<V *>(buf + L.b),
                                                              reinterpret_cast<int64_t *>(buf + L.c),
                                                              ell_tail_slots(A, cap), A->n_rows);
                KP_LAUNCHED();
            }
            P->n_units = 0;
            P->ell_cap = cap;
            break;
        }
        case KP_COO_WM: {
            const int64_t g = (A->nnz + kCooPrepItems - 1) / kCooPrepItems;
            if (g > 0) {
                int32_t *c0 = reinterpret_cast<int32_t *>(buf + L.b);
                k_prep_coo_starts<O><<<(unsigned)((A->n_rows + 255) / 256), 256, 0, s>>>(off, A->n_rows, c0);
                KP_LAUNCHED();
                k_prep_coo<O><<<(unsigned)g, 256, 0, s>>>(off, A->n_rows, A->nnz, c0,
                                                          reinterpret_cast<int32_t *>(buf + L.a));
                KP_LAUNCHED();
            }
            P->n_units = coo_chunks(A);
            break;
        }
        case KP_CSR_MP: {
            const MergeGeom G = merge_geom<V, O>(A);
            const int64_t g = ((G.n_ranges + 1) * 32 + 255) / 256;
            k_prep_mp<O, 32 * kMergeIPT<V>><<<(unsigned)g, 256, 0, s>>>(off, A->n_rows, A->nnz, G.upw, G.n_ranges,
                                                      reinterpret_cast<int64_t *>(buf + L.a));
            KP_LAUNCHED();
            P->n_units = G.n_ranges;
            break;
        }
        case KP_ADAPTIVE_CSR: {
            const int64_t nb = ad_scan_blocks(A);
            int64_t *bsum = reinterpret_cast<int64_t *>(buf + L.c);
            if (nb > 0) {
                k_ad_count<O><<<(unsigned)nb, 256, 0, s>>>(off, A->n_rows, bsum);
                KP_LAUNCHED();
            }
            k_scan_bsum<<<1, 1024, 0, s>>>(bsum, nb, &hdr->n_units);
            KP_LAUNCHED();
            if (nb > 0) {
                k_ad_write<O><<<(unsigned)nb, 256, 0, s>>>(off, A->n_rows, bsum, reinterpret_cast<int32_t *>(buf + L.a),
                                                            reinterpret_cast<int32_t *>(buf + L.b));
                KP_LAUNCHED();
            }
            P->n_units = ad_units_max(A);
            break;
        }
        default: P->n_units = 0; break;
    }
    return KP_OK;
}

// Opt-in shared memory for the TMA CSR,TM kernel (once per <V, O>; also called before a
// plan's graph capture so no attribute call happens inside a capture).
template <typename V, typename O>
int tm_attrs() {
    // the attribute is per device context: one bit per device (a process may drive several)
    static unsigned long long done = 0;
    int dev = 0;
    KP_CUDA_TRY(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (done & bit) return KP_OK;
    const int smem = (int)(kTmStages * TmCfg<V, O>::stage_bytes(TmCfg<V, O>::kCapMax));
    KP_CUDA_TRY(cudaFuncSetAttribute(k_csr_tm<V, O, true, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    KP_CUDA_TRY(cudaFuncSetAttribute(k_csr_tm<V, O, false, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    KP_CUDA_TRY(cudaFuncSetAttribute(k_csr_tm<V, O, true, kTmUWide, kTmSplitWide>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    KP_CUDA_TRY(cudaFuncSetAttribute(k_csr_tm<V, O, false, kTmUWide, kTmSplitWide>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    done |= bit;
    return KP_OK;
}

// PDL tail behind a row-mapped sweep (DeferWs); nothing when no row can be long.
template <typename V, typename O>
int launch_long_rows(int32_t kernel, const kp_csr *A, DeferWs *dw, const O *off, const int32_t *col, const V *val,
                     const V *x, V *y, cudaStream_t s) {
    const int64_t slots = long_slots(kernel, A);
    if (!slots) return KP_OK;
    // enough warps for many medium-long rows (power-law: C2 WM 333 -> 165 us with 2 x SMs
    // instead of 1 x), fewer when at most a handful of rows can be listed
    int64_t ctas = std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms() * 2, (long_huge_at(kernel, A) + 7) / 8));
    ctas = (ctas + kLongCluster - 1) / kLongCluster * kLongCluster;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3(kLongThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = kLongCluster;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    KP_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_long_rows<V, O>, dw, off, col, val, x, y, long_huge_at(kernel, A),
                                   long_giant_at(kernel, A)));
    KP_LAUNCHED();
    return KP_OK;
}

template <typename V, typename O>
int spmv_t(int32_t kernel, const kp_csr *A, const kp_prepared *P, const V *x, V *y, unsigned char *ws,
           cudaStream_t s, const kp_peers *peers = nullptr, const V *acc = nullptr,
           const int32_t *rid = nullptr) {
    const O *off = reinterpret_cast<const O *>(A->row_offsets);
    const int32_t *col = A->col_indices;
    const V *val = reinterpret_cast<const V *>(A->values);
    const int64_t R = A->n_rows, Z = A->nnz;
    const int sms = num_sms();
    // carries live in the workspace: [int32 rows | V vals]
    const int64_t nu = spmv_units(kernel, A);
    int32_t *crow = reinterpret_cast<int32_t *>(ws);
    V *cval = reinterpret_cast<V *>(ws + align_up((size_t)nu * sizeof(int32_t) + 16));
    switch (kernel) {
        case KP_CSR_WM: {
            const int G = P && P->group ? P->group : wm_group(A);
            const int64_t g = (R * G + 255) / 256;
            const int64_t lt = long_threshold(kernel, A), ha = long_huge_at(kernel, A), ga = long_giant_at(kernel, A);
            DeferWs *dw = reinterpret_cast<DeferWs *>(ws);
            switch (G) {
                case 2: k_csr_wm<V, O, 2><<<(unsigned)g, 256, 0, s>>>(off, col, val, x, y, R, dw, lt, ha, ga); break;
                case 4: k_csr_wm<V, O, 4><<<(unsigned)g, 256, 0, s>>>(off, col, val, x, y, R, dw, lt, ha, ga); break;
                case 8: k_csr_wm<V, O, 8><<<(unsigned)g, 256, 0, s>>>(off, col, val, x, y, R, dw, lt, ha, ga); break;
                case 16: k_csr_wm<V, O, 16><<<(unsigned)g, 256, 0, s>>>(off, col, val, x, y, R, dw, lt, ha, ga); break;
                default: k_csr_wm<V, O, 32><<<(unsigned)g, 256, 0, s>>>(off, col, val, x, y, R, dw, lt, ha, ga); break;
            }
            KP_LAUNCHED();
            return launch_long_rows<V, O>(kernel, A, dw, off, col, val, x, y, s);
        }
        case KP_CSR_BM: {
            static const double tiny = [] {  // KP_BM_TINY_MEAN / KP_BM_THREAD: A/B overrides
                const char *e = getenv("KP_BM_TINY_MEAN");
                return e ? atof(e) : kBmTinyMean;
            }();
            static const int64_t thr = [] {
                const char *e = getenv("KP_BM_THREAD");
                return e ? (int64_t)atoll(e) : kBmThread;
            }();
            if ((double)Z <= tiny * (double)R) {  // short known mean: thread-per-row tier
                const int64_t blocks = (R + kBmThreads - 1) / kBmThreads;
                const int64_t g = blocks < (int64_t)sms * 16 ? blocks : (int64_t)sms * 16;  // one resident wave
                k_csr_bm_short<V, O><<<(unsigned)g, kBmThreads, 0, s>>>(off, col, val, x, y, R, thr);
            } else {
                const int64_t groups = (R + 3) / 4;
                const int64_t g = groups < (int64_t)sms * 512 ? groups : (int64_t)sms * 512;
                k_csr_bm<V, O><<<(unsigned)g, 128, 0, s>>>(off, col, val, x, y, R);
            }
            KP_LAUNCHED();
            return KP_OK;
        }
        case KP_CSR_TM: {
            using Cfg = TmCfg<V, O>;
            const int cap = tm_capacity<V, O>(A);
            const size_t smem = kTmStages * Cfg::stage_bytes(cap);
            const bool aligned = (((uintptr_t)col | (uintptr_t)val | (uintptr_t)off) & 15) == 0;
            const bool wide = cap > Cfg::kCap;  // medium rows: enlarged stages, split rows, 1 row / thread
            const int rpt = wide ? 1 : tm_rows_per_thread(A, cap);
            const int64_t tiles = (R + (int64_t)kTmRows * rpt - 1) / ((int64_t)kTmRows * rpt);
            const int per_sm = (int)((227 * 1024) / (smem + 1024));
            const int64_t g = tiles < (int64_t)sms * per_sm ? tiles : (int64_t)sms * per_sm;
            {
                const int rc = tm_attrs<V, O>();
                if (rc) return rc;
            }
            constexpr unsigned bw = kTmRows * kTmSplitWide + 32, bn = kTmRows + 32;
            const int64_t lt = long_threshold(kernel, A), ha = long_huge_at(kernel, A), ga = long_giant_at(kernel, A);
            DeferWs *dw = reinterpret_cast<DeferWs *>(ws);
            if (aligned && wide)
                k_csr_tm<V, O, true, kTmUWide, kTmSplitWide><<<(unsigned)g, bw, smem, s>>>(off, col, val, x, y, R, 1, cap, dw, lt, ha, ga);
            else if (aligned)
                k_csr_tm<V, O, true, 4, 1><<<(unsigned)g, bn, smem, s>>>(off, col, val, x, y, R, rpt, cap, dw, lt, ha, ga);
            else if (wide)
                k_csr_tm<V, O, false, kTmUWide, kTmSplitWide><<<(unsigned)g, bw, smem, s>>>(off, col, val, x, y, R, 1, cap, dw, lt, ha, ga);
            else
                k_csr_tm<V, O, false, 4, 1><<<(unsigned)g, bn, smem, s>>>(off, col, val, x, y, R, rpt, cap, dw, lt, ha, ga);
            KP_LAUNCHED();
            return launch_long_rows<V, O>(kernel, A, dw, off, col, val, x, y, s);
        }
        case KP_ELL_TM: {
            if (!P || !P->buf) return KP_EINVAL;
            const Layout L = prep_layout(KP_ELL_TM, A, P->ell_cap);
            unsigned char *b = reinterpret_cast<unsigned char *>(P->buf);
            const int64_t g = (R + 255) / 256;
            const PrepHeader *hdr = reinterpret_cast<const PrepHeader *>(b);
            k_ell_tm<V, O><<<(unsigned)g, 256, 0, s>>>(hdr, reinterpret_cast<const int32_t *>(b + L.a),
                                                       reinterpret_cast<const V *>(b + L.b), x, y, R);
            KP_LAUNCHED();
            // tail warps: enough for the longest rows to spread over every SM (at most
            // nnz / (cap + 1) rows can be listed)
            const int64_t slots = ell_tail_slots(A, P->ell_cap);
            const int64_t tail_ctas = std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * 2, (slots + 15) / 16));
            KP_CUDA_TRY(launch_pdl(k_ell_tail<V, O>, (unsigned)tail_ctas, kEllTailThreads, s, hdr,
                                   reinterpret_cast<const int64_t *>(b + L.c), slots, off, col, val, x, y));
            KP_LAUNCHED();
            return KP_OK;
        }
        case KP_COO_WM: {
            if (!P || !P->buf) return KP_EINVAL;
            const Layout L = prep_layout(KP_COO_WM, A, 0);
            const MergeGeom G = coo_geom<V>(A);
            const int64_t g = (G.n_ranges * 32 + 255) / 256;
            // 32-byte vector loads need 16-byte aligned col / val (row ids: our buffer)
            const int32_t *rid = reinterpret_cast<const int32_t *>((unsigned char *)P->buf + L.a);
            if ((((uintptr_t)col | (uintptr_t)val) & 15) == 0)
                k_coo_wm<V, true><<<(unsigned)g, 256, 0, s>>>(rid, col, val, x, y, R, Z, G.n_units, G.upw, G.n_ranges,
                                                              crow, cval);
            else
                k_coo_wm<V, false><<<(unsigned)g, 256, 0, s>>>(rid, col, val, x, y, R, Z, G.n_units, G.upw, G.n_ranges,
                                                               crow, cval);
            KP_LAUNCHED();
            KP_CUDA_TRY(launch_pdl(k_carry_fixup<V, false>, (unsigned)((G.n_ranges * 32 + 255) / 256), 256, s, crow,
                                   cval, (const int64_t *)nullptr, G.n_ranges, y, YDst<V>{}));
            KP_LAUNCHED();
            return KP_OK;
        }
        case KP_CSR_MP:
        case KP_CSR_WO: {
            const MergeGeom G = merge_geom<V, O>(A);
            const unsigned g = (unsigned)((G.n_ranges + kMergeWarps - 1) / kMergeWarps);
            if (peers) {  // fused exchange: y stores to every rank's next-x slice
                YDst<V> d{};
                for (int p = 0; p < peers->n; ++p) d.y[p] = reinterpret_cast<V *>(peers->y[p]);
                d.n = peers->n;
                d.self = peers->self;
                d.acc = acc;
                d.rid = rid;
                const int64_t *part = nullptr;
                if (kernel == KP_CSR_MP) {
                    if (!P || !P->buf) return KP_EINVAL;
                    part = reinterpret_cast<const int64_t *>((unsigned char *)P->buf + prep_layout(KP_CSR_MP, A, 0).a);
                    k_csr_merge<V, O, true, true><<<g, kMergeWarps * 32, 0, s>>>(
                        off, col, val, x, d.y[d.self], R, Z, G.n_units, G.upw, G.n_ranges, part, crow, cval, d);
                } else {
                    k_csr_merge<V, O, false, true><<<g, kMergeWarps * 32, 0, s>>>(
                        off, col, val, x, d.y[d.self], R, Z, G.n_units, G.upw, G.n_ranges, nullptr, crow, cval, d);
                }
                KP_LAUNCHED();
                k_carry_fixup<V, true><<<(unsigned)((G.n_ranges * 32 + 255) / 256), 256, 0, s>>>(
                    crow, cval, nullptr, G.n_ranges, d.y[d.self], d);
                KP_LAUNCHED();
                return KP_OK;
            }
            if (kernel == KP_CSR_MP) {
                if (!P || !P->buf) return KP_EINVAL;
                const Layout L = prep_layout(KP_CSR_MP, A, 0);
                k_csr_merge<V, O, true><<<g, kMergeWarps * 32, 0, s>>>(
                    off, col, val, x, y, R, Z, G.n_units, G.upw, G.n_ranges,
                    reinterpret_cast<const int64_t *>((unsigned char *)P->buf + L.a), crow, cval);
            } else {
                k_csr_merge<V, O, false><<<g, kMergeWarps * 32, 0, s>>>(off, col, val, x, y, R, Z, G.n_units, G.upw,
                                                                         G.n_ranges, nullptr, crow, cval);
            }
            KP_LAUNCHED();
            KP_CUDA_TRY(launch_pdl(k_carry_fixup<V, false>, (unsigned)((G.n_ranges * 32 + 255) / 256), 256, s, crow,
                                   cval, (const int64_t *)nullptr, G.n_ranges, y, YDst<V>{}));
            KP_LAUNCHED();
            return KP_OK;
        }
        case KP_ADAPTIVE_CSR: {
            if (!P || !P->buf) return KP_EINVAL;
            const Layout L = prep_layout(KP_ADAPTIVE_CSR, A, 0);
            unsigned char *b = reinterpret_cast<unsigned char *>(P->buf);
            const int64_t *U = &reinterpret_cast<const PrepHeader *>(b)->n_units;
            const int per_sm = sizeof(V) == 4 ? 8 : 6;
            k_adaptive<V, O><<<(unsigned)(sms * per_sm), 256, 0, s>>>(
                off, col, val, x, y, R, reinterpret_cast<const int32_t *>(b + L.a),
                reinterpret_cast<const int32_t *>(b + L.b), U, crow, cval);
            KP_LAUNCHED();
            const int64_t umax = ad_units_max(A);
            const int64_t fg = (umax * 32 + 255) / 256 < (int64_t)sms * 16 ? (umax * 32 + 255) / 256 : (int64_t)sms * 16;
            k_carry_fixup<V><<<(unsigned)fg, 256, 0, s>>>(crow, cval, U, 0, y);
            KP_LAUNCHED();
            return KP_OK;
        }
        default: return KP_EINVAL;
    }
}

}  // namespace

// K1 stats into a caller pointer (used by the ELL prep); defined here to keep the
// reduction kernels private to kp_reduce.cu via its public C entry.
}  // namespace kp

using namespace kp;

extern "C" int kp_length_stats(const void *, int32_t, int64_t, int64_t *, void *, void *);

int kp::ensure_kernel_attrs() {
    int rc = tm_attrs<float, int32_t>();
    if (!rc) rc = tm_attrs<float, int64_t>();
    if (!rc) rc = tm_attrs<double, int32_t>();
    if (!rc) rc = tm_attrs<double, int64_t>();
    // occupancy queries cached outside any graph capture
    kp_csr dummy = {};
    coo_geom<float>(&dummy);
    coo_geom<double>(&dummy);
    merge_warps_per_sm<float, int32_t>();
    merge_warps_per_sm<float, int64_t>();
    merge_warps_per_sm<double, int32_t>();
    merge_warps_per_sm<double, int64_t>();
    return rc;
}

int kp::launch_k1_stats_into(const void *off, int32_t off_type, int64_t n_rows, int64_t *out4, void *ws,
                             cudaStream_t s) {
    return kp_length_stats(off, off_type, n_rows + 1, out4, ws, s);
}

extern "C" {

int kp_prepare_bytes(int32_t kernel, const kp_csr *A, int64_t ell_cap, size_t *bytes) {
    if (!valid_csr(A) || !bytes || kernel < 0 || kernel >= KP_NUM_KERNELS) return KP_EINVAL;
    if (kernel == KP_ELL_TM && ell_cap < 1) return KP_EINVAL;
    *bytes = prep_layout(kernel, A, kernel == KP_ELL_TM ? ell_cap : 0).total;
    return KP_OK;
}

int kp_prepare(int32_t kernel, const kp_csr *A, int64_t ell_cap, void *d_buf, size_t bytes, kp_prepared *out,
               void *stream) {
    KP_NVTX("kp_prepare");
    if (!valid_csr(A) || !out || kernel < 0 || kernel >= KP_NUM_KERNELS) return KP_EINVAL;
    if (kernel == KP_ELL_TM && ell_cap < 1) return KP_EINVAL;
    const Layout L = prep_layout(kernel, A, kernel == KP_ELL_TM ? ell_cap : 0);
    if (bytes < L.total || !d_buf) return KP_ENOMEM;
    if (((uintptr_t)d_buf & (kAlign - 1)) != 0) return KP_EINVAL;
    out->kernel = kernel;
    out->group = wm_group(A);
    out->n_units = 0;
    out->ell_cap = kernel == KP_ELL_TM ? ell_cap : 0;
    out->buf = d_buf;
    out->bytes = bytes;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned char *b = reinterpret_cast<unsigned char *>(d_buf);
    if (A->val_type == KP_F32) {
        return A->off_type == KP_I32 ? prepare_t<float, int32_t>(kernel, A, ell_cap, b, L, out, s)
                                     : prepare_t<float, int64_t>(kernel, A, ell_cap, b, L, out, s);
    }
    return A->off_type == KP_I32 ? prepare_t<double, int32_t>(kernel, A, ell_cap, b, L, out, s)
                                 : prepare_t<double, int64_t>(kernel, A, ell_cap, b, L, out, s);
}

int kp_spmv_workspace_bytes(int32_t kernel, const kp_csr *A, size_t *bytes) {
    if (!valid_csr(A) || !bytes || kernel < 0 || kernel >= KP_NUM_KERNELS) return KP_EINVAL;
    const int64_t nu = spmv_units(kernel, A), nl = long_slots(kernel, A);
    *bytes = nu ? align_up((size_t)nu * sizeof(int32_t) + 16) + align_up((size_t)nu * val_bytes(A))
                : (nl ? align_up(offsetof(DeferWs, rows) + (size_t)nl * sizeof(int64_t)) : 0);
    return KP_OK;
}

int kp_spmv(int32_t kernel, const kp_csr *A, const kp_prepared *P, const void *d_x, void *d_y, void *d_ws,
            size_t ws_bytes, void *stream) {
    KP_NVTX(::kp::kernel_label(kernel));
    if (!valid_csr(A) || kernel < 0 || kernel >= KP_NUM_KERNELS || !d_y || (A->n_cols > 0 && !d_x)) return KP_EINVAL;
    size_t need = 0;
    kp_spmv_workspace_bytes(kernel, A, &need);
    if (ws_bytes < need || (need && !d_ws)) return KP_ENOMEM;
    if (P && P->buf && P->kernel != kernel) return KP_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    if (A->n_rows == 0) return KP_OK;
    if (A->nnz == 0) {
        KP_CUDA_TRY(cudaMemsetAsync(d_y, 0, (size_t)A->n_rows * val_bytes(A), s));
        return KP_OK;
    }
    unsigned char *ws = reinterpret_cast<unsigned char *>(d_ws);
    if (A->val_type == KP_F32) {
        return A->off_type == KP_I32
                   ? spmv_t<float, int32_t>(kernel, A, P, (const float *)d_x, (float *)d_y, ws, s)
                   : spmv_t<float, int64_t>(kernel, A, P, (const float *)d_x, (float *)d_y, ws, s);
    }
    return A->off_type == KP_I32 ? spmv_t<double, int32_t>(kernel, A, P, (const double *)d_x, (double *)d_y, ws, s)
                                 : spmv_t<double, int64_t>(kernel, A, P, (const double *)d_x, (double *)d_y, ws, s);
}

int64_t kp_debug_set_wave_warps(int64_t warps) {
    const int64_t prev = g_wave_warps;
    g_wave_warps = warps > 0 ? warps : 0;
    return prev;
}

int kp_spmv_bcast(int32_t kernel, const kp_csr *A, const kp_prepared *P, const void *d_x, const kp_peers *peers,
                  void *d_ws, size_t ws_bytes, void *stream) {
    return kp_spmv_bcast_acc(kernel, A, P, d_x, nullptr, nullptr, peers, d_ws, ws_bytes, stream);
}

int kp_spmv_bcast_acc(int32_t kernel, const kp_csr *A, const kp_prepared *P, const void *d_x, const void *d_acc,
                      const int32_t *d_rows, const kp_peers *peers, void *d_ws, size_t ws_bytes, void *stream) {
    KP_NVTX("kp_spmv_bcast");
    if (!valid_csr(A) || !peers || peers->n < 1 || peers->n > KP_MAX_PEERS || peers->self < 0 ||
        peers->self >= peers->n || (kernel != KP_CSR_MP && kernel != KP_CSR_WO) || (A->n_cols > 0 && !d_x))
        return KP_EINVAL;
    for (int p = 0; p < peers->n; ++p)
        if (!peers->y[p]) return KP_EINVAL;
    size_t need = 0;
    kp_spmv_workspace_bytes(kernel, A, &need);
    if (ws_bytes < need || (need && !d_ws)) return KP_ENOMEM;
    if (P && P->buf && P->kernel != kernel) return KP_EINVAL;
    // a row map scatters into ONE destination, accumulating in place (or overwriting)
    if (d_rows && (peers->n != 1 || (d_acc && d_acc != peers->y[0]))) return KP_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    if (A->n_rows == 0) return KP_OK;
    const size_t yb = (size_t)A->n_rows * val_bytes(A);
    if (A->nnz == 0 && d_rows) return d_acc ? KP_OK : KP_EINVAL;  // mapped rows += 0: nothing to do
    if (A->nnz == 0) {  // y = acc (or 0) everywhere
        for (int p = 0; p < peers->n; ++p) {
            if (!d_acc) KP_CUDA_TRY(cudaMemsetAsync(peers->y[p], 0, yb, s));
            else if (peers->y[p] != d_acc) KP_CUDA_TRY(cudaMemcpyAsync(peers->y[p], d_acc, yb, cudaMemcpyDefault, s));
        }
        return KP_OK;
    }
    unsigned char *ws = reinterpret_cast<unsigned char *>(d_ws);
    if (A->val_type == KP_F32) {
        const float *acc = (const float *)d_acc;
        return A->off_type == KP_I32
                   ? spmv_t<float, int32_t>(kernel, A, P, (const float *)d_x, nullptr, ws, s, peers, acc, d_rows)
                   : spmv_t<float, int64_t>(kernel, A, P, (const float *)d_x, nullptr, ws, s, peers, acc, d_rows);
    }
    const double *acc = (const double *)d_acc;
    return A->off_type == KP_I32
               ? spmv_t<double, int32_t>(kernel, A, P, (const double *)d_x, nullptr, ws, s, peers, acc, d_rows)
               : spmv_t<double, int64_t>(kernel, A, P, (const double *)d_x, nullptr, ws, s, peers, acc, d_rows);
}

int kp_shard_partition(const void *d_off, int32_t off_type, int64_t n_rows, int32_t parts, int64_t *d_cuts,
                       void *stream) {
    KP_NVTX("kp_shard_partition");
    if (!d_off || !d_cuts || parts < 1 || n_rows < 0) return KP_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned g = (unsigned)((parts + 1 + 255) / 256);
    if (off_type == KP_I32) k_shard_partition<int32_t><<<g, 256, 0, s>>>((const int32_t *)d_off, n_rows, parts, d_cuts);
    else if (off_type == KP_I64) k_shard_partition<int64_t><<<g, 256, 0, s>>>((const int64_t *)d_off, n_rows, parts, d_cuts);
    else return KP_EINVAL;
    KP_LAUNCHED();
    return KP_OK;
}

}  // extern "C"
