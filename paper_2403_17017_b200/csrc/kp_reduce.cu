// kp_reduce.cu -- K1 row_stats (+ bit-exact fp64 epilogue + device tree eval),
// K2 wave_ceil_max_sum, dtree.predict batch, fused seer_select (K15).
//
// Reference counterparts:
//   K1  _kernels.length_stats     /root/reference/pkg/src/kernelpick/_kernels/_core.pyx:15-33
//   K1e gather_features epilogue  features.py:74-85 (compiled with -fmad=false AND explicit
//       __d*_rn intrinsics: Python float math never contracts to FMA)
//   K2  wave_ceil_max_sum         _core.pyx:36-56
//   predict                       SPEC.md:296-301 ; infer SPEC.md:376-384
//
// One pass over row_offsets: every CTA streams 16-byte vectors (4 x int32 or 2 x int64
// offsets per lane, neighbour offset via shuffle), reduces (min, max, sum of squares)
// in registers -> warp -> CTA, writes one partial; the last CTA to finish (ticket
// counter) folds the partials in fixed order, runs the epilogue and the tree, and
// resets the ticket so the workspace is reusable without a memset.  Integer sums are
// uint64 (wrap exactly like the reference's int64); sum = off[n] - off[0] telescopes.
#include "kp_internal.cuh"
#include "../../include/kp_seer_trees.h"

#include <string.h>

namespace kp {

unsigned long long g_launches = 0;

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = kNumSMs;
    }
    return n;
}

namespace {

constexpr int kRedThreads = 256;
// int32 offsets: 4 CTAs/SM (64 registers; 67 M rows 67 -> 59 us); int64 keeps the
// compiler's own allocation (0 = no minimum), which measured faster than any forced budget
template <typename O>
constexpr int kK1MinBlocks = sizeof(O) == 4 ? 4 : 0;
constexpr int kMaxRedBlocks = 148 * 8;

struct Partial {
    int64_t lo, hi;
    uint64_t s2, aux;
};
struct RedWorkspace {
    unsigned int ticket;
    unsigned int pad[3];
    Partial part[kMaxRedBlocks];
};

enum Mode : int { kModeStats = 0, kModeFeatures = 1, kModeSeer = 2 };

// ------------------------------------------------------------------ trees in smem
constexpr int kMaxTreeNodes = 255;  // staged in smem (depth <= 7); larger trees are walked in global memory

struct SmemTree {
    int32_t n;
    const void *src;
    kp_tree_node node[kMaxTreeNodes];
};

__device__ __forceinline__ void load_tree(SmemTree &t, const void *d_tree) {
    const kp_tree_header *h = reinterpret_cast<const kp_tree_header *>(d_tree);
    const kp_tree_node *src = reinterpret_cast<const kp_tree_node *>(h + 1);
    const int n = h->n_nodes;
    if (threadIdx.x == 0) {
        t.n = n;
        t.src = d_tree;
    }
    if (n <= kMaxTreeNodes)
        for (int i = threadIdx.x; i < n; i += blockDim.x) t.node[i] = src[i];
}

__device__ __forceinline__ int32_t predict_global(const void *d_tree, const double *x) {
    const kp_tree_node *nd = reinterpret_cast<const kp_tree_node *>(
        reinterpret_cast<const kp_tree_header *>(d_tree) + 1);
    int32_t i = 0;
    for (;;) {
        kp_tree_node v = nd[i];
        if (v.feature < 0) return v.value;
        i = (x[v.feature] <= v.threshold) ? v.left : v.right;
    }
}

// root-to-leaf, x[f] <= thr goes left.
__device__ __forceinline__ int32_t predict_smem(const SmemTree &t, const double *x) {
    if (t.n > kMaxTreeNodes) return predict_global(t.src, x);
    int32_t i = 0;
    while (t.node[i].feature >= 0) i = (x[t.node[i].feature] <= t.node[i].threshold) ? t.node[i].left : t.node[i].right;
    return t.node[i].value;
}

// ------------------------------------------------------------------ fp64 epilogue
// features.py:74-85 restated with explicit round-to-nearest intrinsics (no FMA).
constexpr int64_t kExact53 = (int64_t)1 << 53;

__device__ void epilogue(int64_t lo, int64_t hi, int64_t s1, int64_t s2, int64_t n, int64_t c,
                         kp_outcome *o) {
    o->lo = lo; o->hi = hi; o->s1 = s1; o->s2 = s2;
    // Python int/int true division is the single correctly-rounded double division
    // only while both operands are <= 2**53 (CPython long_true_divide fast path).
    bool exact = (c <= kExact53) && (hi <= kExact53) && (hi >= -kExact53) &&
                 (lo <= kExact53) && (lo >= -kExact53);
    double dc = __ll2double_rn(c);
    double max_d = __ddiv_rn(__ll2double_rn(hi), dc);
    double min_d = __ddiv_rn(__ll2double_rn(lo), dc);
    double denom = __dmul_rn(__ll2double_rn(n), dc);
    double mean_d = __ddiv_rn(__ll2double_rn(s1), denom);
    double var_d;
    if (hi == lo) {
        var_d = 0.0;
    } else {
        var_d = __dsub_rn(__ddiv_rn(__ll2double_rn(s2), __dmul_rn(denom, dc)), __dmul_rn(mean_d, mean_d));
        if (var_d < 0.0) var_d = 0.0;
    }
    o->max_d = max_d; o->min_d = min_d; o->mean_d = mean_d; o->var_d = var_d;
    o->status = exact ? KP_OK : KP_ERANGE;
}

// ------------------------------------------------------------------ K1 body
template <typename O>
struct Vec16;
template <>
struct Vec16<int64_t> {
    static constexpr int V = 2;
    __device__ static void load(const int64_t *p, int64_t (&o)[2]) {
        longlong2 v = ld_stream2ll(reinterpret_cast<const longlong2 *>(p));
        o[0] = v.x; o[1] = v.y;
    }
};

__device__ __forceinline__ void acc_len(int64_t a, int64_t b, int64_t &lo, int64_t &hi, uint64_t &s2) {
    uint64_t u = (uint64_t)b - (uint64_t)a;
    int64_t ln = (int64_t)u;
    lo = ln < lo ? ln : lo;
    hi = ln > hi ? ln : hi;
    s2 += u * u;
}

// Accumulates rows [0, n_rows) handled by this thread (grid-wide distribution).
template <typename O, bool kVec>
__device__ __forceinline__ void stats_accum(const O *__restrict__ off, int64_t n_rows,
                                            int64_t &lo, int64_t &hi, uint64_t &s2) {
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if constexpr (kVec && sizeof(O) == 4) {
        // int32 offsets (nnz < 2^31): lengths in 32 bits, Σlen² via one IMAD.WIDE.U32 per
        // row; kH independent accumulator sets so no chain serialises the 16 rows of a trip
        const int64_t nvec = n_rows / 4;
        constexpr int kH = 4;
        uint32_t l32[kH], h32[kH];
        uint64_t q[kH];
#pragma unroll
        for (int h = 0; h < kH; ++h) { l32[h] = 0xffffffffu; h32[h] = 0; q[h] = 0; }
        for (int64_t base = gwarp * (32 * kH); base < nvec; base += nwarps * (32 * kH)) {
            int4 e[kH];
            int32_t nx[kH];
#pragma unroll
            for (int h = 0; h < kH; ++h) {
                const int64_t v = base + h * 32 + lane;
                e[h] = v < nvec ? ld_stream4(reinterpret_cast<const int4 *>(off) + v) : make_int4(0, 0, 0, 0);
                nx[h] = (v < nvec && (lane == 31 || v + 1 >= nvec)) ? __ldg(reinterpret_cast<const int32_t *>(off) + (v + 1) * 4) : 0;
            }
#pragma unroll
            for (int h = 0; h < kH; ++h) {
                const int64_t v = base + h * 32 + lane;
                int32_t nxt = __shfl_down_sync(0xffffffffu, e[h].x, 1);
                if (lane == 31 || v + 1 >= nvec) nxt = nx[h];
                if (v < nvec) {
                    if (e[h].y >= e[h].x && e[h].z >= e[h].y && e[h].w >= e[h].z && nxt >= e[h].w) {
                        // non-decreasing (every valid CSR): lengths are exact as uint32
                        const uint32_t u0 = (uint32_t)e[h].y - (uint32_t)e[h].x, u1 = (uint32_t)e[h].z - (uint32_t)e[h].y,
                                       u2 = (uint32_t)e[h].w - (uint32_t)e[h].z, u3 = (uint32_t)nxt - (uint32_t)e[h].w;
                        l32[h] = min(min(l32[h], u0), min(min(u1, u2), u3));
                        h32[h] = max(max(h32[h], u0), max(max(u1, u2), u3));
                        q[h] += (uint64_t)u0 * u0 + (uint64_t)u1 * u1 + (uint64_t)u2 * u2 + (uint64_t)u3 * u3;
                    } else {  // arbitrary int32 arrays (the C-ABI accepts them): signed 64-bit lengths
                        acc_len(e[h].x, e[h].y, lo, hi, s2);
                        acc_len(e[h].y, e[h].z, lo, hi, s2);
                        acc_len(e[h].z, e[h].w, lo, hi, s2);
                        acc_len(e[h].w, nxt, lo, hi, s2);
                    }
                }
            }
        }
#pragma unroll
        for (int h = 0; h < kH; ++h) {
            if (l32[h] != 0xffffffffu || h32[h] != 0 || q[h] != 0) {
                lo = (int64_t)l32[h] < lo ? (int64_t)l32[h] : lo;
                hi = (int64_t)h32[h] > hi ? (int64_t)h32[h] : hi;
            }
            s2 += q[h];
        }
        // scalar tail rows [nvec*4, n_rows)
        const int64_t t0 = nvec * 4;
        const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (gt < n_rows - t0) acc_len(ldo(off + t0 + gt), ldo(off + t0 + gt + 1), lo, hi, s2);
    } else if constexpr (kVec) {
        constexpr int V = Vec16<O>::V;
        const int64_t nvec = n_rows / V;  // vector v covers rows v*V .. v*V+V-1
        // kH independent 16-byte vectors per lane per iteration, plus (lane 31 / the last
        // vector) the following offset, all issued before any use
        constexpr int kH = 4;
        for (int64_t base = gwarp * (32 * kH); base < nvec; base += nwarps * (32 * kH)) {
            int64_t e[kH][V];
            int64_t nx[kH];
#pragma unroll
            for (int h = 0; h < kH; ++h) {
                const int64_t v = base + h * 32 + lane;
                if (v < nvec) Vec16<O>::load(off + v * V, e[h]);
                else {
#pragma unroll
                    for (int k = 0; k < V; ++k) e[h][k] = 0;
                }
                nx[h] = (v < nvec && (lane == 31 || v + 1 >= nvec)) ? ldo(off + (v + 1) * V) : 0;
            }
#pragma unroll
            for (int h = 0; h < kH; ++h) {
                const int64_t v = base + h * 32 + lane;
                const bool act = v < nvec;
                int64_t nxt = __shfl_down_sync(0xffffffffu, e[h][0], 1);
                if (act && (lane == 31 || v + 1 >= nvec)) nxt = nx[h];
                if (act) {
#pragma unroll
                    for (int k = 0; k < V - 1; ++k) acc_len(e[h][k], e[h][k + 1], lo, hi, s2);
                    acc_len(e[h][V - 1], nxt, lo, hi, s2);
                }
            }
        }
        // scalar tail rows [nvec*V, n_rows)
        const int64_t t0 = nvec * V;
        const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (gt < n_rows - t0) acc_len(ldo(off + t0 + gt), ldo(off + t0 + gt + 1), lo, hi, s2);
    } else {
        const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const int64_t st = (int64_t)gridDim.x * blockDim.x;
        for (int64_t i = gt; i < n_rows; i += st) acc_len(ldo(off + i), ldo(off + i + 1), lo, hi, s2);
    }
}

template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) { T w = __shfl_xor_sync(0xffffffffu, v, o); v = w < v ? w : v; }
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) { T w = __shfl_xor_sync(0xffffffffu, v, o); v = w > v ? w : v; }
    return v;
}
__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-reduce (lo, hi, s2) into thread 0.
__device__ __forceinline__ void block_reduce(int64_t &lo, int64_t &hi, uint64_t &s2) {
    __shared__ int64_t slo[32], shi[32];
    __shared__ uint64_t ss2[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    lo = warp_min(lo); hi = warp_max(hi); s2 = warp_sum_u64(s2);
    if (lane == 0) { slo[w] = lo; shi[w] = hi; ss2[w] = s2; }
    __syncthreads();
    if (w == 0) {
        lo = lane < nw ? slo[lane] : INT64_MAX;
        hi = lane < nw ? shi[lane] : INT64_MIN;
        s2 = lane < nw ? ss2[lane] : 0;
        lo = warp_min(lo); hi = warp_max(hi); s2 = warp_sum_u64(s2);
    }
}

// Shared state of the fused K1 / K15 kernel.
struct K1Args {
    const void *off;
    int64_t n_rows, n_cols, nnz, iters;
    int mode;
    int64_t *out4;          // kModeStats
    kp_outcome *out;        // kModeFeatures / kModeSeer
    const void *sel, *known, *gath;
    RedWorkspace *ws;
};

// Grid-wide (min, max, sum of squares) of row lengths; returns true in the LAST CTA to
// finish (valid in thread 0), which has folded all CTA partials in fixed order and reset
// the ticket so the workspace is reusable without a memset.
template <typename O, bool kVec>
__device__ __forceinline__ bool k1_pass(const K1Args &a, const O *off, int64_t &lo, int64_t &hi, uint64_t &s2) {
    __shared__ bool s_last;
    lo = INT64_MAX; hi = INT64_MIN; s2 = 0;
    stats_accum<O, kVec>(off, a.n_rows, lo, hi, s2);
    block_reduce(lo, hi, s2);
    if (threadIdx.x == 0) {
        a.ws->part[blockIdx.x] = Partial{lo, hi, s2, 0};
        __threadfence();
        unsigned t = atomicAdd(&a.ws->ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    lo = INT64_MAX; hi = INT64_MIN; s2 = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
        const Partial *p = &a.ws->part[i];
        const int64_t plo = __ldcg(&p->lo), phi = __ldcg(&p->hi);
        lo = plo < lo ? plo : lo;
        hi = phi > hi ? phi : hi;
        s2 += (uint64_t)__ldcg((const unsigned long long *)&p->s2);
    }
    __syncthreads();
    block_reduce(lo, hi, s2);
    if (threadIdx.x == 0) {
        a.ws->ticket = 0;
        if (a.n_rows <= 0) { lo = hi = 0; s2 = 0; }
    }
    return true;
}

template <typename O, bool kVec>
__global__ void __launch_bounds__(kRedThreads, kK1MinBlocks<O>) k_row_stats(K1Args a) {
    __shared__ SmemTree tree;
    __shared__ int s_path;
    const O *off = reinterpret_cast<const O *>(a.off);

    if (a.mode == kModeSeer) {
        // Selector on the known schema (rows, cols, nnz, iterations).
        load_tree(tree, a.sel);
        __syncthreads();
        if (threadIdx.x == 0) {
            double xk[4] = {(double)a.n_rows, (double)a.n_cols, (double)a.nnz, (double)a.iters};
            s_path = predict_smem(tree, xk);
        }
        __syncthreads();
        if (s_path == KP_USE_KNOWN) {
            // Known path never reads the matrix (SPEC.md:388 purity): CTA 0 answers.
            if (blockIdx.x != 0) return;
            __syncthreads();
            load_tree(tree, a.known);
            __syncthreads();
            if (threadIdx.x == 0) {
                double xk[4] = {(double)a.n_rows, (double)a.n_cols, (double)a.nnz, (double)a.iters};
                kp_outcome o = {};
                o.kernel = predict_smem(tree, xk);
                o.path = KP_USE_KNOWN;
                o.status = KP_OK;
                *a.out = o;
            }
            return;
        }
        // gathered path: prefetch the gathered tree now (overlaps the offsets stream), so
        // the last CTA evaluates it without two more round trips at the tail
        __syncthreads();
        load_tree(tree, a.gath);
    }

    int64_t lo, hi;
    uint64_t s2;
    // sum = off[n] - off[0] telescopes; loaded up front so the last CTA's tail has no extra round trip
    const int64_t n = a.n_rows;
    const int64_t s1 = (threadIdx.x == 0 && n > 0) ? (int64_t)((uint64_t)ldo(off + n) - (uint64_t)ldo(off)) : 0;
    if (!k1_pass<O, kVec>(a, off, lo, hi, s2)) return;
    if (threadIdx.x == 0) {
        if (a.mode == kModeStats) {
            a.out4[0] = lo; a.out4[1] = hi; a.out4[2] = s1; a.out4[3] = (int64_t)s2;
        } else {
            kp_outcome o = {};
            epilogue(lo, hi, s1, (int64_t)s2, n, a.n_cols, &o);
            o.kernel = -1;
            o.path = KP_USE_GATHERED;
            if (a.mode == kModeSeer) {
                double xg[8] = {(double)a.n_rows, (double)a.n_cols, (double)a.nnz, (double)a.iters,
                                o.max_d, o.min_d, o.mean_d, o.var_d};
                o.kernel = predict_smem(tree, xg);
            }
            *a.out = o;
        }
    }
}

// ------------------------------------------------------------------ plan select (K15, graph)
// The graph flavour of kp_seer_select: the three trees travel BY VALUE in the kernel's
// parameter space (constant bank: every thread walks the selector with broadcast loads,
// no global / smem round trip), and the chosen kernel index steers the plan's SWITCH node
// directly (cudaGraphSetConditional) -- no separate set-switch launch.
__device__ __forceinline__ double feat(const double *x, int f, int nf) {
    double v = x[0];
#pragma unroll
    for (int i = 1; i < 8; ++i)
        if (i < nf && f == i) v = x[i];
    return v;
}
template <int NF>
__device__ __forceinline__ int32_t predict_param(const ParamTrees &T, int t, const double (&x)[NF]) {
    int32_t i = 0;
    while (T.node[t][i].feature >= 0)
        i = (feat(x, T.node[t][i].feature, NF) <= T.node[t][i].threshold) ? T.node[t][i].left : T.node[t][i].right;
    return T.node[t][i].value;
}

// Tree evaluators for the plan's selection kernel: the packed trees by value (any bundle)
// or the bundle's trees compiled in as nested conditionals (include/kp_seer_trees.h,
// emitted by tools/emit_trees.py) -- used only when the plan's
// trees equal the compiled ones byte for byte (emitted_trees_match).
struct ParamPred {
    const ParamTrees &T;
    template <int NF>
    __device__ __forceinline__ int32_t operator()(int t, const double (&x)[NF]) const { return predict_param(T, t, x); }
};
struct EmittedPred {
    template <int NF>
    __device__ __forceinline__ int32_t operator()(int t, const double (&x)[NF]) const {
        if constexpr (NF == 4) return t == 0 ? seer_selector(x) : seer_known(x);
        else return seer_gathered(x);
    }
};

template <typename O, bool kVec, typename Pred>
__device__ __forceinline__ void plan_select_body(const K1Args &a, const Pred &pred, cudaGraphConditionalHandle h) {
    const O *off = reinterpret_cast<const O *>(a.off);
    const double xk[4] = {(double)a.n_rows, (double)a.n_cols, (double)a.nnz, (double)a.iters};
    if (pred(0, xk) == KP_USE_KNOWN) {  // the matrix is never read
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            kp_outcome o = {};
            o.kernel = pred(1, xk);
            o.path = KP_USE_KNOWN;
            o.status = KP_OK;
            *a.out = o;
            cudaGraphSetConditional(h, (o.kernel >= 0 && o.kernel < KP_NUM_KERNELS) ? (unsigned)o.kernel
                                                                                   : (unsigned)KP_NUM_KERNELS);
        }
        return;
    }
    int64_t lo, hi;
    uint64_t s2;
    const int64_t n = a.n_rows;
    const int64_t s1 = threadIdx.x == 0 ? (int64_t)((uint64_t)ldo(off + n) - (uint64_t)ldo(off)) : 0;
    if (!k1_pass<O, kVec>(a, off, lo, hi, s2)) return;
    if (threadIdx.x == 0) {
        kp_outcome o = {};
        epilogue(lo, hi, s1, (int64_t)s2, n, a.n_cols, &o);
        o.path = KP_USE_GATHERED;
        const double xg[8] = {(double)a.n_rows, (double)a.n_cols, (double)a.nnz, (double)a.iters,
                              o.max_d, o.min_d, o.mean_d, o.var_d};
        o.kernel = pred(2, xg);
        *a.out = o;
        cudaGraphSetConditional(h, (o.kernel >= 0 && o.kernel < KP_NUM_KERNELS) ? (unsigned)o.kernel
                                                                               : (unsigned)KP_NUM_KERNELS);
    }
}

template <typename O, bool kVec>
__global__ void __launch_bounds__(kRedThreads, kK1MinBlocks<O>) k_seer_plan_select(K1Args a, const __grid_constant__ ParamTrees T,
                                                                   cudaGraphConditionalHandle h) {
    plan_select_body<O, kVec>(a, ParamPred{T}, h);
}

template <typename O, bool kVec>
__global__ void __launch_bounds__(kRedThreads, kK1MinBlocks<O>) k_seer_plan_select_emitted(K1Args a,
                                                                   cudaGraphConditionalHandle h) {
    plan_select_body<O, kVec>(a, EmittedPred{}, h);
}

// batch evaluation of one compiled tree (tests: emitted == interpreted on 1e5 vectors)
__global__ void k_emitted_predict(int32_t which, const double *__restrict__ x, int64_t n, int32_t *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (which == 2) {
            double xv[8];
            for (int f = 0; f < 8; ++f) xv[f] = x[i * 8 + f];
            out[i] = seer_gathered(xv);
        } else {
            double xv[4];
            for (int f = 0; f < 4; ++f) xv[f] = x[i * 4 + f];
            out[i] = which == 0 ? seer_selector(xv) : seer_known(xv);
        }
    }
}

// ------------------------------------------------------------------ K2
// Small waves (<= 4096 rows): a group of G lanes owns whole waves, lanes stride the
// wave's rows; large waves: one CTA per wave.  Per-thread running sums of wave maxima
// -> partials -> last CTA.  units = (len + div - 1) / div in C semantics (_core.pyx:46).
template <typename O, int G>
__global__ void __launch_bounds__(kRedThreads) k_wave_small(const O *__restrict__ off, int64_t n_rows,
                                                            int64_t div, int64_t wave, int64_t *out,
                                                            RedWorkspace *ws) {
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    constexpr int kGpw = 32 / G;  // groups (waves) per warp
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t n_waves = (n_rows + wave - 1) / wave;
    uint64_t sum = 0;
    // warp-uniform outer loop: the full-mask shuffle below is executed by all lanes
    for (int64_t wb = gwarp * kGpw; wb < n_waves; wb += nwarps * kGpw) {
        const int64_t w = wb + lane / G;
        int64_t m = 0;
        if (w < n_waves) {
            const int64_t r0 = w * wave;
            int64_t r1 = r0 + wave;
            if (r1 > n_rows) r1 = n_rows;
            for (int64_t r = r0 + gl; r < r1; r += G) {
                int64_t u = (ldo(off + r + 1) - ldo(off + r) + div - 1) / div;
                m = u > m ? u : m;
            }
        }
#pragma unroll
        for (int o = G / 2; o; o >>= 1) {
            int64_t t = __shfl_xor_sync(0xffffffffu, m, o);
            m = t > m ? t : m;
        }
        if (gl == 0 && w < n_waves) sum += (uint64_t)m;
    }
    sum = warp_sum_u64(sum);
    __shared__ uint64_t sw[32];
    if (lane == 0) sw[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sw[i];
        ws->part[blockIdx.x] = Partial{0, 0, t, 0};
        __threadfence();
        s_last = atomicAdd(&ws->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int i = 0; i < (int)gridDim.x; ++i) t += ws->part[i].s2;
        *out = (int64_t)t;
        ws->ticket = 0;
    }
}

template <typename O>
__global__ void __launch_bounds__(1024) k_wave_large(const O *__restrict__ off, int64_t n_rows,
                                                     int64_t div, int64_t wave, int64_t *out,
                                                     RedWorkspace *ws) {
    __shared__ bool s_last;
    __shared__ int64_t sm[32];
    const int lane = threadIdx.x & 31;
    const int64_t n_waves = (n_rows + wave - 1) / wave;
    uint64_t sum = 0;
    for (int64_t w = blockIdx.x; w < n_waves; w += gridDim.x) {
        const int64_t r0 = w * wave;
        int64_t r1 = r0 + wave;
        if (r1 > n_rows) r1 = n_rows;
        int64_t m = 0;
        for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
            int64_t u = (ldo(off + r + 1) - ldo(off + r) + div - 1) / div;
            m = u > m ? u : m;
        }
        m = warp_max(m);
        if (lane == 0) sm[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t mm = 0;
            for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mm = sm[i] > mm ? sm[i] : mm;
            sum += (uint64_t)mm;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ws->part[blockIdx.x] = Partial{0, 0, sum, 0};
        __threadfence();
        s_last = atomicAdd(&ws->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    uint64_t t = 0;
    for (int i = 0; i < (int)gridDim.x; ++i) t += ws->part[i].s2;
    *out = (int64_t)t;
    ws->ticket = 0;
}

// ------------------------------------------------------------------ batch predict
__global__ void k_tree_predict(const void *tree, const double *__restrict__ x, int64_t n, int32_t nf,
                               int32_t *__restrict__ out) {
    __shared__ SmemTree t;
    load_tree(t, tree);
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double xv[16];
        for (int f = 0; f < nf && f < 16; ++f) xv[f] = x[i * nf + f];
        out[i] = predict_smem(t, xv);
    }
}

// ------------------------------------------------------------------ launch helpers
// `per_thread` rows per thread keeps the partials few on large inputs; small inputs get up
// to one CTA per SM at a quarter of that, so every offset load of the pass is in flight in
// the first trip instead of a chain of dependent trips in one CTA (latency, not bandwidth)
int grid_for(int64_t n_rows, int per_thread) {
    const int64_t per_cta = (int64_t)kRedThreads * per_thread, per_cta_lat = per_cta / 4;
    int64_t want = (n_rows + per_cta - 1) / per_cta;
    int64_t want_lat = (n_rows + per_cta_lat - 1) / per_cta_lat;
    if (want_lat > num_sms()) want_lat = num_sms();
    if (want < want_lat) want = want_lat;
    int cap = num_sms() * 8;  // full occupancy for large inputs (bytes in flight)
    if (cap > kMaxRedBlocks) cap = kMaxRedBlocks;
    if (want < 1) want = 1;
    return (int)(want < cap ? want : cap);
}

// Defensive reset of the last-CTA ticket before every host-dispatched pass: the kernels
// leave it zero, but a caller that shares one workspace between overlapping streams (or a
// grid that died mid-way) would otherwise poison every later pass.  16 bytes, async.
int reset_ticket(void *ws, cudaStream_t s) {
    KP_CUDA_TRY(cudaMemsetAsync(ws, 0, 16, s));
    return KP_OK;
}

int launch_k1(K1Args a, int32_t off_type, cudaStream_t s) {
    if (reset_ticket(a.ws, s)) return KP_ECUDA;
    const bool aligned = ((uintptr_t)a.off & 15) == 0;
    if (off_type == KP_I32) {
        int g = grid_for(a.n_rows, 64);
        if (aligned) k_row_stats<int32_t, true><<<g, kRedThreads, 0, s>>>(a);
        else k_row_stats<int32_t, false><<<g, kRedThreads, 0, s>>>(a);
    } else if (off_type == KP_I64) {
        int g = grid_for(a.n_rows, 32);
        if (aligned) k_row_stats<int64_t, true><<<g, kRedThreads, 0, s>>>(a);
        else k_row_stats<int64_t, false><<<g, kRedThreads, 0, s>>>(a);
    } else {
        return KP_EINVAL;
    }
    KP_LAUNCHED();
    return KP_OK;
}

template <typename O>
int launch_wave(const O *off, int64_t n_rows, int64_t div, int64_t wave, int64_t *out, RedWorkspace *ws,
                cudaStream_t s) {
    const int64_t n_waves = (n_rows + wave - 1) / wave;
    if (wave <= 4096) {
        int G = 1;
        while (G < wave && G < 32) G <<= 1;
        const int64_t groups_per_block = kRedThreads / G;
        int64_t want = (n_waves + groups_per_block - 1) / groups_per_block;
        int cap = num_sms() * 8 < kMaxRedBlocks ? num_sms() * 8 : kMaxRedBlocks;
        int g = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
        switch (G) {
            case 1: k_wave_small<O, 1><<<g, kRedThreads, 0, s>>>(off, n_rows, div, wave, out, ws); break;
            case 2: k_wave_small<O, 2><<<g, kRedThreads, 0, s>>>(off, n_rows, div, wave, out, ws); break;
            case 4: k_wave_small<O, 4><<<g, kRedThreads, 0, s>>>(off, n_rows, div, wave, out, ws); break;
            case 8: k_wave_small<O, 8><<<g, kRedThreads, 0, s>>>(off, n_rows, div, wave, out, ws); break;
            case 16: k_wave_small<O, 16><<<g, kRedThreads, 0, s>>>(off, n_rows, div, wave, out, ws); break;
            default: k_wave_small<O, 32><<<g, kRedThreads, 0, s>>>(off, n_rows, div, wave, out, ws); break;
        }
    } else {
        int cap = num_sms() * 2 < kMaxRedBlocks ? num_sms() * 2 : kMaxRedBlocks;
        int g = (int)(n_waves < cap ? n_waves : cap);
        k_wave_large<O><<<g, 1024, 0, s>>>(off, n_rows, div, wave, out, ws);
    }
    KP_LAUNCHED();
    return KP_OK;
}

// Multi-GPU K15: every rank holds the (lo, hi, s1, s2) partials of all ranks' row blocks
// (one 32-byte all-gather); combine exactly (min / max / wrapping sums = the single-matrix
// reduction, _core.pyx:25-32), then the same selector / epilogue / tree path as K1+K15.
__global__ void k_seer_select_partials(const int64_t *__restrict__ parts, int32_t n_parts, int64_t n_rows,
                                       int64_t n_cols, int64_t nnz, int64_t iters, const void *sel, const void *known,
                                       const void *gath, kp_outcome *out) {
    if (threadIdx.x != 0) return;
    const double xk[4] = {(double)n_rows, (double)n_cols, (double)nnz, (double)iters};
    double xkk[4] = {xk[0], xk[1], xk[2], xk[3]};
    kp_outcome o = {};
    if (predict_global(sel, xkk) == KP_USE_KNOWN) {
        o.kernel = predict_global(known, xkk);
        o.path = KP_USE_KNOWN;
        o.status = KP_OK;
        *out = o;
        return;
    }
    int64_t lo = INT64_MAX, hi = INT64_MIN;
    uint64_t s1 = 0, s2 = 0;
    for (int p = 0; p < n_parts; ++p) {
        const int64_t *q = parts + 4 * p;
        lo = q[0] < lo ? q[0] : lo;
        hi = q[1] > hi ? q[1] : hi;
        s1 += (uint64_t)q[2];
        s2 += (uint64_t)q[3];
    }
    if (n_rows <= 0) { lo = hi = 0; s1 = s2 = 0; }
    epilogue(lo, hi, (int64_t)s1, (int64_t)s2, n_rows, n_cols, &o);
    o.path = KP_USE_GATHERED;
    double xg[8] = {xk[0], xk[1], xk[2], xk[3], o.max_d, o.min_d, o.mean_d, o.var_d};
    o.kernel = predict_global(gath, xg);
    *out = o;
}

}  // namespace

// ---- plan select (graph flavour of K15): trees copied once to the host at plan creation
int plan_trees_load(const void *d_sel, const void *d_known, const void *d_gath, ParamTrees *T) {
    const void *src[3] = {d_sel, d_known, d_gath};
    *T = ParamTrees{};
    for (int t = 0; t < 3; ++t) {
        kp_tree_header h;
        KP_CUDA_TRY(cudaMemcpy(&h, src[t], sizeof(h), cudaMemcpyDeviceToHost));
        if (h.n_nodes < 1 || h.n_nodes > kParamTreeNodes) return KP_EINVAL;
        KP_CUDA_TRY(cudaMemcpy(T->node[t], reinterpret_cast<const kp_tree_header *>(src[t]) + 1,
                               (size_t)h.n_nodes * sizeof(kp_tree_node), cudaMemcpyDeviceToHost));
        for (int i = 0; i < h.n_nodes; ++i) {  // a malformed tree must not walk out of the table
            const kp_tree_node &nd = T->node[t][i];
            if (nd.feature >= 0 && (nd.left <= i || nd.right <= i || nd.left >= h.n_nodes || nd.right >= h.n_nodes ||
                                    nd.feature >= (t == 2 ? 8 : 4)))
                return KP_EINVAL;
        }
        T->n[t] = h.n_nodes;
    }
    return KP_OK;
}

bool emitted_trees_match(const ParamTrees &T) {
    const unsigned char *packed[3] = {kp_seer_packed_selector, kp_seer_packed_known, kp_seer_packed_gathered};
    const size_t bytes[3] = {sizeof(kp_seer_packed_selector), sizeof(kp_seer_packed_known),
                             sizeof(kp_seer_packed_gathered)};
    for (int t = 0; t < 3; ++t) {
        kp_tree_header h;
        memcpy(&h, packed[t], sizeof(h));
        if (h.n_nodes != T.n[t] || bytes[t] != sizeof(h) + (size_t)h.n_nodes * sizeof(kp_tree_node) ||
            memcmp(packed[t] + sizeof(h), T.node[t], (size_t)h.n_nodes * sizeof(kp_tree_node)) != 0)
            return false;
    }
    return true;
}

int launch_plan_select(const void *d_off, int32_t off_type, int64_t n_rows, int64_t n_cols, int64_t nnz,
                       int64_t iters, const ParamTrees &T, bool emitted, kp_outcome *d_out, void *d_ws,
                       cudaGraphConditionalHandle h, cudaStream_t s) {
    K1Args a = {};
    a.off = d_off; a.n_rows = n_rows; a.n_cols = n_cols; a.nnz = nnz; a.iters = iters;
    a.mode = kModeSeer; a.out = d_out; a.ws = (RedWorkspace *)d_ws;
    // launch-shape hint only: the kernel evaluates the selector on the device every run;
    // for a KNOWN-path plan (static shape) one CTA answers, else a full feature-pass grid
    const double xk[4] = {(double)n_rows, (double)n_cols, (double)nnz, (double)iters};
    int32_t i = 0;
    while (T.node[0][i].feature >= 0) i = (xk[T.node[0][i].feature] <= T.node[0][i].threshold) ? T.node[0][i].left : T.node[0][i].right;
    const bool known = T.node[0][i].value == KP_USE_KNOWN;
    const bool aligned = ((uintptr_t)d_off & 15) == 0;
    if (off_type == KP_I32) {
        const int g = known ? 1 : grid_for(n_rows, 64);
        if (emitted) {
            if (aligned) k_seer_plan_select_emitted<int32_t, true><<<g, kRedThreads, 0, s>>>(a, h);
            else k_seer_plan_select_emitted<int32_t, false><<<g, kRedThreads, 0, s>>>(a, h);
        } else if (aligned) k_seer_plan_select<int32_t, true><<<g, kRedThreads, 0, s>>>(a, T, h);
        else k_seer_plan_select<int32_t, false><<<g, kRedThreads, 0, s>>>(a, T, h);
    } else if (off_type == KP_I64) {
        const int g = known ? 1 : grid_for(n_rows, 32);
        if (emitted) {
            if (aligned) k_seer_plan_select_emitted<int64_t, true><<<g, kRedThreads, 0, s>>>(a, h);
            else k_seer_plan_select_emitted<int64_t, false><<<g, kRedThreads, 0, s>>>(a, h);
        } else if (aligned) k_seer_plan_select<int64_t, true><<<g, kRedThreads, 0, s>>>(a, T, h);
        else k_seer_plan_select<int64_t, false><<<g, kRedThreads, 0, s>>>(a, T, h);
    } else {
        return KP_EINVAL;
    }
    KP_LAUNCHED();
    return KP_OK;
}

}  // namespace kp

using namespace kp;

extern "C" {

size_t kp_reduce_workspace_bytes(void) { return sizeof(RedWorkspace); }

int kp_length_stats(const void *d_off, int32_t off_type, int64_t n_off, int64_t *d_out4, void *d_ws,
                    void *stream) {
    KP_NVTX("kp_length_stats");
    if (!d_out4 || !d_ws || n_off < 0 || (n_off > 0 && !d_off)) return KP_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = n_off - 1;
    if (n <= 0) {  // _core.pyx:21-22 / _pure.py:14-15
        KP_CUDA_TRY(cudaMemsetAsync(d_out4, 0, 4 * sizeof(int64_t), s));
        return KP_OK;
    }
    K1Args a = {};
    a.off = d_off; a.n_rows = n; a.mode = kModeStats; a.out4 = d_out4; a.ws = (RedWorkspace *)d_ws;
    return launch_k1(a, off_type, s);
}

int kp_gather_features(const void *d_off, int32_t off_type, int64_t n_rows, int64_t n_cols,
                       kp_outcome *d_out, void *d_ws, void *stream) {
    KP_NVTX("kp_gather_features");
    if (n_rows <= 0 || n_cols <= 0 || !d_off || !d_out || !d_ws) return KP_EINVAL;
    K1Args a = {};
    a.off = d_off; a.n_rows = n_rows; a.n_cols = n_cols; a.mode = kModeFeatures; a.out = d_out;
    a.ws = (RedWorkspace *)d_ws;
    return launch_k1(a, off_type, (cudaStream_t)stream);
}

int kp_seer_select(const void *d_off, int32_t off_type, int64_t n_rows, int64_t n_cols, int64_t nnz,
                   int64_t iterations, const void *d_selector, const void *d_known, const void *d_gathered,
                   kp_outcome *d_out, void *d_ws, void *stream) {
    KP_NVTX("kp_seer_select");
    if (n_rows <= 0 || n_cols <= 0 || !d_off || !d_out || !d_ws || !d_selector || !d_known || !d_gathered)
        return KP_EINVAL;
    K1Args a = {};
    a.off = d_off; a.n_rows = n_rows; a.n_cols = n_cols; a.nnz = nnz; a.iters = iterations;
    a.mode = kModeSeer; a.out = d_out; a.sel = d_selector; a.known = d_known; a.gath = d_gathered;
    a.ws = (RedWorkspace *)d_ws;
    return launch_k1(a, off_type, (cudaStream_t)stream);
}

int kp_wave_ceil_max_sum(const void *d_off, int32_t off_type, int64_t n_off, int64_t divisor,
                         int64_t wave_rows, int64_t *d_out1, void *d_ws, void *stream) {
    KP_NVTX("kp_wave_ceil_max_sum");
    if (divisor <= 0 || wave_rows <= 0 || !d_out1 || !d_ws || n_off < 0) return KP_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = n_off - 1;
    if (n <= 0) {
        KP_CUDA_TRY(cudaMemsetAsync(d_out1, 0, sizeof(int64_t), s));
        return KP_OK;
    }
    RedWorkspace *ws = (RedWorkspace *)d_ws;
    if (reset_ticket(ws, s)) return KP_ECUDA;
    if (off_type == KP_I32) return launch_wave((const int32_t *)d_off, n, divisor, wave_rows, d_out1, ws, s);
    if (off_type == KP_I64) return launch_wave((const int64_t *)d_off, n, divisor, wave_rows, d_out1, ws, s);
    return KP_EINVAL;
}

int kp_tree_predict(const void *d_tree, const double *d_x, int64_t n, int32_t n_feat, int32_t *d_out,
                    void *stream) {
    KP_NVTX("kp_tree_predict");
    if (!d_tree || n < 0 || n_feat <= 0 || n_feat > 16) return KP_EINVAL;
    if (n == 0) return KP_OK;
    int64_t want = (n + 255) / 256;
    int g = (int)(want < num_sms() * 8 ? want : num_sms() * 8);
    k_tree_predict<<<g, 256, 0, (cudaStream_t)stream>>>(d_tree, d_x, n, n_feat, d_out);
    KP_LAUNCHED();
    return KP_OK;
}

int kp_seer_select_partials(const int64_t *d_parts, int32_t n_parts, int64_t n_rows, int64_t n_cols, int64_t nnz,
                            int64_t iterations, const void *d_selector, const void *d_known, const void *d_gathered,
                            kp_outcome *d_out, void *stream) {
    KP_NVTX("kp_seer_select_partials");
    if (n_parts < 1 || n_rows <= 0 || n_cols <= 0 || !d_parts || !d_out || !d_selector || !d_known || !d_gathered)
        return KP_EINVAL;
    k_seer_select_partials<<<1, 32, 0, (cudaStream_t)stream>>>(d_parts, n_parts, n_rows, n_cols, nnz, iterations,
                                                               d_selector, d_known, d_gathered, d_out);
    KP_LAUNCHED();
    return KP_OK;
}

int kp_seer_emitted_predict(int32_t tree, const double *d_x, int64_t n, int32_t *d_out, void *stream) {
    KP_NVTX("kp_seer_emitted_predict");
    if (tree < 0 || tree > 2 || n < 0 || (n > 0 && (!d_x || !d_out))) return KP_EINVAL;
    if (n == 0) return KP_OK;
    int64_t want = (n + 255) / 256;
    int g = (int)(want < num_sms() * 8 ? want : num_sms() * 8);
    k_emitted_predict<<<g, 256, 0, (cudaStream_t)stream>>>(tree, d_x, n, d_out);
    KP_LAUNCHED();
    return KP_OK;
}

const char *kp_seer_emitted_sha256(void) { return KP_SEER_TREES_SHA256; }

uint64_t kp_launch_count(void) { return (uint64_t)kp::g_launches; }
const char *kp_version(void) { return "kpb200 0.1.0 sm_100a"; }

}  // extern "C"
