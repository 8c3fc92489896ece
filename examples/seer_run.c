/* seer_run.c -- the Seer pipeline from plain C over the C-ABI (no Python, no torch):
 *
 *   Matrix Market text --kp_mm_parse--> triples --kp_csr_from_coo (GPU)--> CSR in HBM
 *   --kp_seer_plan_create / _launch--> selection + chosen preprocessing + k SpMVs (one graph)
 *
 * what a non-Python host of the reference's path (a cgo / JNI / N-API binding) would do.
 *
 *   ./seer_run matrix.mtx seer_b200.trees [iterations]
 * prints: kernel=<idx> path=<0 known|1 gathered> nnz=<n> us_per_launch=<t> y0=<y[0]>
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "kernelpick_b200.h"

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            return 2;                                                          \
        }                                                                      \
    } while (0)
#define KP(x)                                                                  \
    do {                                                                       \
        int rc_ = (x);                                                         \
        if (rc_ != KP_OK) {                                                    \
            fprintf(stderr, "%s:%d %s -> %d\n", __FILE__, __LINE__, #x, rc_);  \
            return 3;                                                          \
        }                                                                      \
    } while (0)

static char *slurp(const char *path, size_t *len) {
    FILE *f = fopen(path, "rb");
    if (!f) return NULL;
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    char *b = (char *)malloc((size_t)n + 1);
    if (b && fread(b, 1, (size_t)n, f) != (size_t)n) { free(b); b = NULL; }
    fclose(f);
    *len = (size_t)n;
    return b;
}

int main(int argc, char **argv) {
    if (argc < 3) {
        fprintf(stderr, "usage: %s matrix.mtx seer.trees [iterations]\n", argv[0]);
        return 1;
    }
    const int64_t iters = argc > 3 ? atoll(argv[3]) : 1;
    size_t mlen = 0, tlen = 0;
    char *mtx = slurp(argv[1], &mlen), *trees = slurp(argv[2], &tlen);
    if (!mtx || !trees || tlen < 4 || memcmp(trees, "KPT1", 4) != 0) {
        fprintf(stderr, "cannot read inputs\n");
        return 1;
    }
    /* 1) parse (host, parallel) */
    kp_mm_info info;
    int rc = kp_mm_header(mtx, mlen, &info);
    if (rc == KP_EPARSE) { fprintf(stderr, "ParseError: %s\n", info.err); return 4; }
    KP(rc);
    int64_t cap = info.n_entries * (info.symmetry ? 2 : 1);
    int64_t *rows = (int64_t *)malloc((size_t)(cap ? cap : 1) * 8), *cols = (int64_t *)malloc((size_t)(cap ? cap : 1) * 8);
    double *vals = (double *)malloc((size_t)(cap ? cap : 1) * 8);
    rc = kp_mm_parse(mtx, mlen, rows, cols, vals, cap, 0, &info);
    if (rc == KP_EPARSE) { fprintf(stderr, "ParseError: %s\n", info.err); return 4; }
    KP(rc);
    const int64_t n = info.n_triples, R = info.n_rows, C = info.n_cols;
    /* 2) canonical CSR on the GPU */
    int64_t *d_r, *d_c, *d_off, *d_out2;
    double *d_v, *d_val;
    int32_t *d_col;
    void *d_ws;
    size_t ws = 0;
    KP(kp_coo_workspace_bytes(n, R, C, &ws));
    CK(cudaMalloc((void **)&d_r, (size_t)(n ? n : 1) * 8));
    CK(cudaMalloc((void **)&d_c, (size_t)(n ? n : 1) * 8));
    CK(cudaMalloc((void **)&d_v, (size_t)(n ? n : 1) * 8));
    CK(cudaMalloc((void **)&d_off, (size_t)(R + 1) * 8));
    CK(cudaMalloc((void **)&d_col, (size_t)(n ? n : 1) * 4));
    CK(cudaMalloc((void **)&d_val, (size_t)(n ? n : 1) * 8));
    CK(cudaMalloc((void **)&d_out2, 16));
    CK(cudaMalloc(&d_ws, ws ? ws : 256));
    CK(cudaMemcpy(d_r, rows, (size_t)n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_c, cols, (size_t)n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_v, vals, (size_t)n * 8, cudaMemcpyHostToDevice));
    KP(kp_csr_from_coo(R, C, d_r, d_c, d_v, n, d_off, d_col, d_val, d_out2, d_ws, ws, NULL));
    int64_t out2[2];
    CK(cudaMemcpy(out2, d_out2, 16, cudaMemcpyDeviceToHost));
    if (out2[1]) { fprintf(stderr, "%lld out-of-range triples\n", (long long)out2[1]); return 5; }
    kp_csr A = {R, C, out2[0], KP_I64, KP_F64, d_off, d_col, d_val};
    /* 3) trees (packed) -> device */
    const void *d_tree[3];
    size_t at = 4;
    for (int t = 0; t < 3; ++t) {
        uint32_t nb;
        memcpy(&nb, trees + at, 4);
        at += 4;
        void *p;
        CK(cudaMalloc(&p, nb));
        CK(cudaMemcpy(p, trees + at, nb, cudaMemcpyHostToDevice));
        d_tree[t] = p;
        at += nb;
    }
    /* 4) the Seer plan: select -> chosen preprocessing -> iters SpMVs, one CUDA graph */
    double *d_x, *d_y;
    CK(cudaMalloc((void **)&d_x, (size_t)(C ? C : 1) * 8));
    CK(cudaMalloc((void **)&d_y, (size_t)(R ? R : 1) * 8));
    double *hx = (double *)malloc((size_t)(C ? C : 1) * 8);
    for (int64_t j = 0; j < C; ++j) hx[j] = 1.0;
    CK(cudaMemcpy(d_x, hx, (size_t)C * 8, cudaMemcpyHostToDevice));
    const int64_t ell_cap = (R ? 2 * (out2[0] / R) : 0) + 8;
    size_t pb = 0;
    KP(kp_seer_plan_bytes(&A, ell_cap, &pb));
    void *d_buf, *d_red;
    kp_outcome *d_outc;
    CK(cudaMalloc(&d_buf, pb ? pb : 256));
    const size_t red = kp_reduce_workspace_bytes();
    CK(cudaMalloc(&d_red, red));
    CK(cudaMemset(d_red, 0, red));
    CK(cudaMalloc((void **)&d_outc, sizeof(kp_outcome)));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    kp_seer_plan *plan = NULL;
    KP(kp_seer_plan_create(&A, iters, ell_cap, d_tree[0], d_tree[1], d_tree[2], d_x, d_y, d_buf, pb, d_red, d_outc,
                           &plan, s));
    KP(kp_seer_plan_launch(plan, s));
    CK(cudaStreamSynchronize(s));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int reps = 10;
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < reps; ++i) KP(kp_seer_plan_launch(plan, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    kp_outcome o;
    double y0 = 0;
    CK(cudaMemcpy(&o, d_outc, sizeof(o), cudaMemcpyDeviceToHost));
    if (R) CK(cudaMemcpy(&y0, d_y, 8, cudaMemcpyDeviceToHost));
    printf("kernel=%d path=%d nnz=%lld us_per_launch=%.2f y0=%.17g\n", o.kernel, o.path, (long long)out2[0],
           1000.0 * ms / reps, y0);
    KP(kp_seer_plan_destroy(plan));
    return 0;
}
