// kp_coo2csr.cu -- csr_from_coo (sparse.py:87-103) on the device: the canonicalisation step
// in front of the Seer path.
//
// Reference semantics, restated exactly:
//   order = np.lexsort((cols, rows))            -> STABLE sort by key = row * n_cols + col
//   v = np.add.reduceat(v[order], starts)       -> per duplicate run: v0 + pairwise_sum(rest)
//                                                  (numpy's reduce loop: 8-way unrolled blocks
//                                                  of <= 128, halving recursion above)
//   offsets = cumsum(bincount(rows))            -> offsets from the unique keys' rows
//
// B200 design: an LSD radix sort of the 64-bit keys (8-bit digits, only the digits the key
// range needs) carrying the original index as payload.  Per pass: a per-tile digit
// histogram, one exclusive scan of the digit-major histogram table, and a stable scatter in
// which each warp ranks its striped items step by step with __match_any_sync (lanes with the
// same digit) + per-warp smem digit counters, then a per-digit prefix over the CTA's warps.
// Duplicate runs are summed by one thread each, in input order, with numpy's pairwise
// algorithm, so values are bit-identical to the reference; offsets come from a lower_bound
// of every row over the unique rows.  No floating-point atomics.
#include "kp_internal.cuh"

namespace kp {
namespace {

constexpr int kRsThreads = 256;
constexpr int kRsIPT = 8;
constexpr int kRsTile = kRsThreads * kRsIPT;  // 2048 items per tile
constexpr int kRsDigits = 256;
constexpr int kScanChunk = 2048;

constexpr size_t al256(size_t v) { return (v + 255) / 256 * 256; }

__global__ void __launch_bounds__(256) k_coo_keys(const int64_t *__restrict__ rows, const int64_t *__restrict__ cols,
                                                  int64_t n, int64_t n_rows, int64_t n_cols, uint64_t *__restrict__ key,
                                                  int32_t *__restrict__ idx, unsigned long long *__restrict__ bad) {
    int64_t nbad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = rows[i], c = cols[i];
        const bool ok = r >= 0 && r < n_rows && c >= 0 && c < n_cols;
        key[i] = ok ? (uint64_t)r * (uint64_t)n_cols + (uint64_t)c : 0;
        idx[i] = (int32_t)i;
        nbad += !ok;
    }
    if (nbad) atomicAdd(bad, (unsigned long long)nbad);
}

__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const uint64_t *__restrict__ key, int64_t n, int shift,
                                                        int32_t *__restrict__ hist, int64_t n_tiles) {
    __shared__ int32_t cnt[kRsDigits];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t t0 = (int64_t)blockIdx.x * kRsTile;
#pragma unroll
    for (int j = 0; j < kRsIPT; ++j) {
        const int64_t e = t0 + j * kRsThreads + threadIdx.x;
        if (e < n) atomicAdd(&cnt[(int)((key[e] >> shift) & 255)], 1);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * n_tiles + blockIdx.x] = cnt[threadIdx.x];
}

// ---- exclusive scan of an int32 array (values and totals < 2^31), 3 kernels
__global__ void __launch_bounds__(256) k_scan_partials(const int32_t *__restrict__ a, int64_t m, int64_t *__restrict__ part) {
    __shared__ int64_t sw[8];
    const int64_t c0 = (int64_t)blockIdx.x * kScanChunk;
    int64_t s = 0;
    for (int j = threadIdx.x; j < kScanChunk; j += 256)
        if (c0 + j < m) s += a[c0 + j];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < 8; ++w) t += sw[w];
        part[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) k_scan_top(int64_t *__restrict__ part, int64_t np) {
    __shared__ int64_t sw[32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t b = 0; b < np; b += 1024) {
        const int64_t i = b + threadIdx.x;
        const int64_t v = i < np ? part[i] : 0;
        int64_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) sw[w] = inc;
        __syncthreads();
        if (w == 0) {
            int64_t x = sw[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t t = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += t;
            }
            sw[lane] = x;
        }
        __syncthreads();
        const int64_t excl = carry + (w > 0 ? sw[w - 1] : 0) + inc - v;
        if (i < np) part[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_scan_apply(int32_t *__restrict__ a, int64_t m, const int64_t *__restrict__ part) {
    // 256 threads x 8 consecutive items (blocked): thread-local scan + block scan
    __shared__ int64_t sw[8];
    const int64_t c0 = (int64_t)blockIdx.x * kScanChunk;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t v[8];
    int64_t s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int64_t e = c0 + threadIdx.x * 8 + j;
        v[j] = e < m ? a[e] : 0;
        s += v[j];
    }
    int64_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) sw[w] = inc;
    __syncthreads();
    int64_t run = part[blockIdx.x] + inc - s;
    for (int k = 0; k < w; ++k) run += sw[k];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int64_t e = c0 + threadIdx.x * 8 + j;
        if (e < m) a[e] = (int32_t)run;
        run += v[j];
    }
}

// ---- stable scatter of one radix pass
__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const uint64_t *__restrict__ key_in,
                                                           const int32_t *__restrict__ idx_in,
                                                           uint64_t *__restrict__ key_out, int32_t *__restrict__ idx_out,
                                                           int64_t n, int shift, const int32_t *__restrict__ hist,
                                                           int64_t n_tiles) {
    __shared__ int32_t wcnt[kRsThreads / 32][kRsDigits];
    __shared__ int32_t base[kRsDigits];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kRsThreads / 32; ++k) wcnt[k][threadIdx.x] = 0;
    base[threadIdx.x] = hist[(int64_t)threadIdx.x * n_tiles + blockIdx.x];
    __syncthreads();
    // warp w owns tile items [w*256, w*256+256), striped: step i -> item w*256 + i*32 + lane,
    // so (step, lane) order IS the input order and ranking lanes within a step keeps it stable
    const int64_t e0 = (int64_t)blockIdx.x * kRsTile + w * (kRsIPT * 32) + lane;
    uint64_t k[kRsIPT];
    int32_t v[kRsIPT], d[kRsIPT], rk[kRsIPT];
#pragma unroll
    for (int i = 0; i < kRsIPT; ++i) {
        const int64_t e = e0 + i * 32;
        k[i] = e < n ? key_in[e] : 0;
        v[i] = e < n ? idx_in[e] : 0;
        d[i] = e < n ? (int)((k[i] >> shift) & 255) : kRsDigits;
    }
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kRsIPT; ++i) {
        const unsigned m = __match_any_sync(0xffffffffu, d[i]);
        const int before = d[i] < kRsDigits ? wcnt[w][d[i]] : 0;
        rk[i] = before + __popc(m & lt);
        __syncwarp();
        if (d[i] < kRsDigits && (m & lt) == 0) wcnt[w][d[i]] = before + __popc(m);  // run leader
        __syncwarp();
    }
    __syncthreads();
    {   // per digit: exclusive prefix over the CTA's warps (warp w's items follow warps < w)
        int32_t acc = 0;
#pragma unroll
        for (int k2 = 0; k2 < kRsThreads / 32; ++k2) {
            const int32_t t = wcnt[k2][threadIdx.x];
            wcnt[k2][threadIdx.x] = acc;
            acc += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRsIPT; ++i) {
        if (d[i] < kRsDigits) {
            const int64_t pos = (int64_t)base[d[i]] + wcnt[w][d[i]] + rk[i];
            key_out[pos] = k[i];
            idx_out[pos] = v[i];
        }
    }
}

// numpy pairwise_sum (DOUBLE, contiguous): n < 8 sequential from 0.0; n <= 128 eight
// accumulators over 8-blocks + sequential remainder; above, split at n/2 rounded down to 8.
__device__ double np_pairwise(const double *__restrict__ val, const int32_t *__restrict__ idx, int64_t a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, val[idx[a + i]]);
        return r;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = val[idx[a + j]];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], val[idx[a + i + j]]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, val[idx[a + i]]);
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(np_pairwise(val, idx, a, n2), np_pairwise(val, idx, a + n2, n - n2));
}

// heads: flag[i] = 1 at the first element of each duplicate run (scanned afterwards)
__global__ void __launch_bounds__(256) k_coo_heads(const uint64_t *__restrict__ key, int64_t n, int32_t *__restrict__ flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// one thread per duplicate run: v0 + pairwise(rest) in input order (np.add.reduceat)
__global__ void __launch_bounds__(256) k_coo_reduce(const uint64_t *__restrict__ key, const int32_t *__restrict__ idx,
                                                    const int32_t *__restrict__ pos, const double *__restrict__ val,
                                                    int64_t n, int64_t n_cols, int32_t *__restrict__ col_out,
                                                    double *__restrict__ val_out, int32_t *__restrict__ row_out,
                                                    int64_t *__restrict__ nnz_out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t kk = key[i];
        if (i > 0 && key[i - 1] == kk) continue;
        int64_t j = i + 1;
        while (j < n && key[j] == kk) ++j;
        const double v0 = val[idx[i]];
        const double s = j - i > 1 ? __dadd_rn(v0, np_pairwise(val, idx, i + 1, j - i - 1)) : v0;
        const int64_t p = pos[i];
        col_out[p] = (int32_t)(kk % (uint64_t)n_cols);
        row_out[p] = (int32_t)(kk / (uint64_t)n_cols);
        val_out[p] = s;
        if (j == n) *nnz_out = p + 1;
    }
}

// off[r] = #unique entries with row < r (lower_bound over the sorted unique rows)
__global__ void __launch_bounds__(256) k_coo_offsets(const int32_t *__restrict__ urow, const int64_t *__restrict__ nnz_dev,
                                                     int64_t n_rows, int64_t *__restrict__ off) {
    const int64_t nnz = *nnz_dev;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)urow[mid] < r) lo = mid + 1;
            else hi = mid;
        }
        off[r] = lo;
    }
}

struct CooLayout {
    size_t key0, key1, idx0, idx1, hist, part, bad, total;
    int64_t n_tiles, hist_len, n_parts, passes;
};

int key_bits(int64_t n_rows, int64_t n_cols) {
    const unsigned __int128 span = (unsigned __int128)n_rows * (unsigned __int128)n_cols;
    int b = 0;
    while (b < 64 && ((unsigned __int128)1 << b) < span) ++b;
    return b;
}

CooLayout coo_layout(int64_t n, int64_t n_rows, int64_t n_cols) {
    CooLayout L{};
    L.n_tiles = (n + kRsTile - 1) / kRsTile;
    L.hist_len = L.n_tiles * kRsDigits;
    const int64_t m = L.hist_len > n ? L.hist_len : n;  // the scan also runs over the n head flags
    L.n_parts = (m + kScanChunk - 1) / kScanChunk;
    L.passes = (key_bits(n_rows, n_cols) + 7) / 8;
    size_t o = 0;
    L.key0 = o; o += al256((size_t)n * 8);
    L.key1 = o; o += al256((size_t)n * 8);
    L.idx0 = o; o += al256((size_t)n * 4);
    L.idx1 = o; o += al256((size_t)n * 4);
    L.hist = o; o += al256((size_t)L.hist_len * 4);
    L.part = o; o += al256((size_t)(L.n_parts + 1) * 8);
    L.bad = o; o += 256;
    L.total = o;
    return L;
}

int scan_exclusive(int32_t *a, int64_t m, int64_t *part, cudaStream_t s) {
    if (m <= 0) return KP_OK;
    const int64_t np = (m + kScanChunk - 1) / kScanChunk;
    k_scan_partials<<<(unsigned)np, 256, 0, s>>>(a, m, part);
    KP_LAUNCHED();
    k_scan_top<<<1, 1024, 0, s>>>(part, np);
    KP_LAUNCHED();
    k_scan_apply<<<(unsigned)np, 256, 0, s>>>(a, m, part);
    KP_LAUNCHED();
    return KP_OK;
}

}  // namespace
}  // namespace kp

using namespace kp;

extern "C" {

int kp_coo_workspace_bytes(int64_t n, int64_t n_rows, int64_t n_cols, size_t *bytes) {
    if (!bytes || n < 0 || n_rows < 0 || n_cols < 0 || n >= INT32_MAX) return KP_EINVAL;
    *bytes = coo_layout(n, n_rows, n_cols).total;
    return KP_OK;
}

int kp_csr_from_coo(int64_t n_rows, int64_t n_cols, const int64_t *d_rows, const int64_t *d_cols,
                    const double *d_vals, int64_t n, int64_t *d_off, int32_t *d_col, double *d_val,
                    int64_t *d_out2, void *d_ws, size_t ws_bytes, void *stream) {
    KP_NVTX("kp_csr_from_coo");
    if (n < 0 || n >= INT32_MAX || n_rows < 0 || n_rows >= INT32_MAX || n_cols < 0 || n_cols > INT32_MAX ||
        !d_off || !d_out2 || (n > 0 && (!d_rows || !d_cols || !d_vals || !d_col || !d_val)))
        return KP_EINVAL;
    const CooLayout L = coo_layout(n, n_rows, n_cols);
    if (n > 0 && (ws_bytes < L.total || !d_ws)) return KP_ENOMEM;
    cudaStream_t s = (cudaStream_t)stream;
    KP_CUDA_TRY(cudaMemsetAsync(d_out2, 0, 2 * sizeof(int64_t), s));
    const int sms = num_sms();
    if (n == 0) {
        KP_CUDA_TRY(cudaMemsetAsync(d_off, 0, (size_t)(n_rows + 1) * sizeof(int64_t), s));
        return KP_OK;
    }
    unsigned char *w = reinterpret_cast<unsigned char *>(d_ws);
    uint64_t *key[2] = {reinterpret_cast<uint64_t *>(w + L.key0), reinterpret_cast<uint64_t *>(w + L.key1)};
    int32_t *idx[2] = {reinterpret_cast<int32_t *>(w + L.idx0), reinterpret_cast<int32_t *>(w + L.idx1)};
    int32_t *hist = reinterpret_cast<int32_t *>(w + L.hist);
    int64_t *part = reinterpret_cast<int64_t *>(w + L.part);
    const unsigned gs = (unsigned)(sms * 8);
    k_coo_keys<<<gs, 256, 0, s>>>(d_rows, d_cols, n, n_rows, n_cols, key[0], idx[0],
                                  reinterpret_cast<unsigned long long *>(d_out2 + 1));
    KP_LAUNCHED();
    int cur = 0;
    for (int64_t p = 0; p < L.passes; ++p) {
        const int shift = (int)(8 * p);
        k_rs_hist<<<(unsigned)L.n_tiles, kRsThreads, 0, s>>>(key[cur], n, shift, hist, L.n_tiles);
        KP_LAUNCHED();
        int rc = scan_exclusive(hist, L.hist_len, part, s);
        if (rc) return rc;
        k_rs_scatter<<<(unsigned)L.n_tiles, kRsThreads, 0, s>>>(key[cur], idx[cur], key[1 - cur], idx[1 - cur], n, shift,
                                                              hist, L.n_tiles);
        KP_LAUNCHED();
        cur = 1 - cur;
    }
    // duplicate runs: head flags -> exclusive scan = output position of each run
    int32_t *pos = idx[1 - cur];
    k_coo_heads<<<gs, 256, 0, s>>>(key[cur], n, pos);
    KP_LAUNCHED();
    int rc = scan_exclusive(pos, n, part, s);
    if (rc) return rc;
    int32_t *urow = reinterpret_cast<int32_t *>(key[1 - cur]);  // n int32 fit in the spare key buffer
    k_coo_reduce<<<gs, 256, 0, s>>>(key[cur], idx[cur], pos, d_vals, n, n_cols, d_col, d_val, urow, d_out2);
    KP_LAUNCHED();
    k_coo_offsets<<<(unsigned)((n_rows + 1 + 255) / 256 < sms * 16 ? (n_rows + 1 + 255) / 256 : sms * 16), 256, 0, s>>>(
        urow, d_out2, n_rows, d_off);
    KP_LAUNCHED();
    return KP_OK;
}

}  // extern "C"
