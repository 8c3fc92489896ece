// kp_pack.cu -- the compact host->device transfer format of a CSR matrix's column indices.
//
// A single SpMV of a host-resident matrix is bound by PCIe (C2: 137 MB per step at ~50-55
// GB/s against 84 us of SpMV), and half of those bytes are column indices that need only
// ceil(log2(n_cols)) bits (C2: 20 of 32).  The host side (kp_pack_cols, OpenMP, kp_hostpack
// in this file's host half) writes them as one little-endian bitstream of 32-bit words --
// column i occupies bits [i*b, (i+1)*b) -- once, when the matrix is loaded; every step then
// moves the packed stream (C2: 40 MB instead of 64 MB) and k_unpack_cols restores the int32
// array the SpMV kernels read, in HBM at ~6 TB/s (~15 us for C2).  Lossless; values, offsets
// and x travel unchanged.
#include <omp.h>

#include "kp_internal.cuh"

namespace kp {
namespace {

// 4 columns per thread: bit offset i*b, word w = off >> 5, shift s = off & 31; a column
// spans at most two words (b <= 32), read as an unaligned 64-bit funnel of words w, w+1.
__global__ void __launch_bounds__(256) k_unpack_cols(const uint32_t *__restrict__ packed, int64_t n_words,
                                                     int64_t n, int32_t b, int32_t *__restrict__ cols) {
    const uint32_t mask = b == 32 ? 0xffffffffu : ((1u << b) - 1u);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
    for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i0 < n; i0 += stride) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t i = i0 + q;
            if (i >= n) break;
            const int64_t bit = i * b;
            const int64_t w = bit >> 5;
            const uint32_t lo = __ldg(packed + w);
            const uint32_t hi = w + 1 < n_words ? __ldg(packed + w + 1) : 0u;
            cols[i] = (int32_t)(__funnelshift_r(lo, hi, (uint32_t)(bit & 31)) & mask);
        }
    }
}

}  // namespace
}  // namespace kp

using namespace kp;

extern "C" {

int32_t kp_pack_bits(int64_t n_cols) {
    int32_t b = 1;
    while (b < 32 && ((int64_t)1 << b) < n_cols) ++b;
    return b;
}

size_t kp_pack_cols_bytes(int64_t n, int64_t n_cols) {
    const int64_t b = kp_pack_bits(n_cols);
    return (size_t)(((n * b + 31) >> 5) + 1) * sizeof(uint32_t);  // +1 word: the funnel's w+1
}

int kp_pack_cols(const int32_t *h_cols, int64_t n, int64_t n_cols, uint32_t *h_out, int32_t n_threads) {
    KP_NVTX("kp_pack_cols");
    if (n < 0 || n_cols < 1 || (n > 0 && (!h_cols || !h_out))) return KP_EINVAL;
    const int32_t b = kp_pack_bits(n_cols);
    const int64_t n_words = ((n * b + 31) >> 5) + 1;
    // word-parallel: word w holds the bits of columns floor(32w / b) .. floor((32w + 31) / b)
    int bad = 0;
#pragma omp parallel for schedule(static) num_threads(n_threads > 0 ? n_threads : omp_get_max_threads()) reduction(| : bad)
    for (int64_t w = 0; w < n_words; ++w) {
        uint64_t acc = 0;
        const int64_t bit0 = w * 32;
        int64_t i = bit0 / b;
        for (; i < n && i * b < bit0 + 32; ++i) {
            const int32_t c = h_cols[i];
            bad |= (c < 0 || (int64_t)c >= n_cols);
            const int64_t sh = i * b - bit0;  // may be negative for the column straddling in
            const uint64_t v = (uint64_t)(uint32_t)c;
            acc |= sh >= 0 ? (v << sh) : (v >> -sh);
        }
        h_out[w] = (uint32_t)acc;
    }
    return bad ? KP_ERANGE : KP_OK;
}

int kp_unpack_cols(const uint32_t *d_packed, int64_t n, int64_t n_cols, int32_t *d_cols, void *stream) {
    KP_NVTX("kp_unpack_cols");
    if (n < 0 || n_cols < 1 || (n > 0 && (!d_packed || !d_cols))) return KP_EINVAL;
    if (n == 0) return KP_OK;
    const int32_t b = kp_pack_bits(n_cols);
    const int64_t n_words = ((n * b + 31) >> 5) + 1;
    const int64_t want = (n + 1023) / 1024;
    const int g = (int)(want < (int64_t)num_sms() * 16 ? want : (int64_t)num_sms() * 16);
    k_unpack_cols<<<g, 256, 0, (cudaStream_t)stream>>>(d_packed, n_words, n, b, d_cols);
    KP_LAUNCHED();
    return KP_OK;
}

}  // extern "C"
