/*
 * kernelpick_b200.h -- C-ABI of the B200-native Seer hot path (libkpb200.so).
 *
 * Drop-in boundary for the reference's `kernelpick._kernels` backend
 * (/root/reference/pkg/src/kernelpick/_kernels/__init__.py:1-28) plus the SPEC-only
 * surfaces on the north-star path (dtree.predict, seer-core.infer, the SpMV kernel
 * family of PAPER.md:263-273 and its preprocessing).
 *
 * Conventions (all entry points):
 *   - return int status: KP_OK (0) or a negative KP_E* code; no exceptions cross the ABI;
 *   - every buffer argument named d_* is a DEVICE pointer owned by the caller;
 *   - work is enqueued asynchronously on `stream` (a cudaStream_t; NULL = legacy default);
 *   - no host synchronisation happens inside any call below;
 *   - scratch memory comes from the caller through *_workspace_bytes() queries.
 *
 * Offset arrays may be int32 (KP_I32, valid while nnz < 2^31) or int64 (KP_I64, the
 * reference layout, sparse.py:37); column indices are int32; values / x / y are fp32
 * (KP_F32) or fp64 (KP_F64).
 */
#ifndef KERNELPICK_B200_H
#define KERNELPICK_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define KP_API __attribute__((visibility("default")))
#else
#define KP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status codes */
#define KP_OK 0
#define KP_EINVAL (-1)      /* bad argument (reference: ValueError)                */
#define KP_ECUDA (-2)       /* a CUDA launch / runtime call failed                  */
#define KP_ENOMEM (-3)      /* caller workspace too small                           */
#define KP_EUNSUPPORTED (-4)
#define KP_ERANGE (-5)      /* value outside the exactly-representable range        */
#define KP_EPARSE (-6)      /* malformed input text (reference: ParseError)           */

/* ---------------------------------------------------------------- type codes   */
#define KP_I32 0
#define KP_I64 1
#define KP_F32 0
#define KP_F64 1

/* Kernel vocabulary, fixed order = PAPER.md Table III (:311-318); tree class indices
 * and lowest-index tie-breaks depend on it.  Never reorder. */
#define KP_ADAPTIVE_CSR 0
#define KP_CSR_BM 1
#define KP_CSR_MP 2
#define KP_CSR_WM 3
#define KP_CSR_WO 4
#define KP_CSR_TM 5
#define KP_COO_WM 6
#define KP_ELL_TM 7
#define KP_NUM_KERNELS 8
#define KP_MAX_PEERS 8

/* Seer path. */
#define KP_USE_KNOWN 0
#define KP_USE_GATHERED 1

/* Device CSR view (host struct holding device pointers).  Mirrors SparseMatrixCSR
 * (sparse.py:33-39) with device-width index/value types. */
typedef struct kp_csr {
    int64_t n_rows, n_cols, nnz;
    int32_t off_type;          /* KP_I32 | KP_I64 */
    int32_t val_type;          /* KP_F32 | KP_F64 */
    const void *row_offsets;   /* [n_rows + 1] */
    const int32_t *col_indices;/* [nnz] */
    const void *values;        /* [nnz] */
} kp_csr;

/* Result of the fused feature pass / selection, written to DEVICE memory.
 * lo/hi/s1/s2 = _kernels.length_stats (_core.pyx:15-33, wrapping int64);
 * max/min/mean/var = GatheredFeatures.as_vector() (features.py:46-52, 74-85). */
typedef struct kp_outcome {
    int64_t lo, hi, s1, s2;
    double max_d, min_d, mean_d, var_d;
    int32_t kernel;            /* chosen kernel index (seer) or -1            */
    int32_t path;              /* KP_USE_KNOWN / KP_USE_GATHERED              */
    int32_t status;            /* KP_OK or KP_ERANGE from the epilogue guard  */
    int32_t reserved;
} kp_outcome;

/* Packed decision tree, DEVICE memory, 8-byte aligned:
 *   kp_tree_header followed by n_nodes kp_tree_node records.
 * feature < 0 marks a leaf whose class is `value`. Left iff x[feature] <= threshold. */
typedef struct kp_tree_header {
    int32_t n_nodes, n_features, n_classes, max_depth;
} kp_tree_header;
typedef struct kp_tree_node {
    double threshold;
    int32_t feature, left, right, value;
} kp_tree_node;

/* Prepared-format view produced by kp_prepare() inside a caller buffer. */
typedef struct kp_prepared {
    int32_t kernel;            /* KP_* kernel id this preparation serves            */
    int32_t group;             /* CSR,WM lanes per row (2..32), chosen from nnz/rows */
    int64_t n_units;           /* MP tiles / adaptive units / COO chunks            */
    int64_t ell_cap;           /* ELL: allocated width (columns)                    */
    void *buf;                 /* base of the caller buffer                         */
    size_t bytes;
} kp_prepared;

/* ------------------------------------------------------- drop-in backend (K1, K2) */
/* Scratch for every reduction entry point; must be zeroed ONCE at allocation
 * (cudaMemset); the kernels leave it zeroed again after each call, and every entry point
 * below also re-zeroes its 16-byte ticket (async) before launching.  One workspace per
 * stream: two passes that may overlap must not share one. */
KP_API size_t kp_reduce_workspace_bytes(void);

/* _kernels.length_stats (_core.pyx:15-33 / _pure.py:11-21):
 * d_out4 <- (min, max, sum, sum of squares) of diff(row_offsets), int64 wrapping.
 * n_off = len(row_offsets); n_off <= 1 gives (0, 0, 0, 0). */
KP_API int kp_length_stats(const void *d_off, int32_t off_type, int64_t n_off,
                    int64_t *d_out4, void *d_ws, void *stream);

/* _kernels.wave_ceil_max_sum (_core.pyx:36-56 / _pure.py:24-38):
 * d_out1 <- sum over consecutive waves of `wave_rows` rows of max ceil(len/divisor).
 * divisor <= 0 or wave_rows <= 0 -> KP_EINVAL (the reference backends diverge). */
KP_API int kp_wave_ceil_max_sum(const void *d_off, int32_t off_type, int64_t n_off,
                         int64_t divisor, int64_t wave_rows, int64_t *d_out1,
                         void *d_ws, void *stream);

/* features.gather_features (features.py:64-87) minus the clock: the integer pass
 * and the bit-exact fp64 epilogue in one launch.  n_rows == 0 or n_cols == 0 ->
 * KP_EINVAL (features.py:67-70). */
KP_API int kp_gather_features(const void *d_off, int32_t off_type, int64_t n_rows,
                       int64_t n_cols, kp_outcome *d_out, void *d_ws, void *stream);

/* ------------------------------------------------------------ trees / selection */
/* dtree.predict over a batch: d_out[i] = predict(tree, d_x[i*n_feat:]). */
KP_API int kp_tree_predict(const void *d_tree, const double *d_x, int64_t n, int32_t n_feat,
                    int32_t *d_out, void *stream);

/* seer-core.infer fused on device: selector tree on
 * (rows, cols, nnz, iterations) -> USE_KNOWN: known tree; USE_GATHERED: the
 * gather_features pass + gathered tree on known + (max, min, mean, var).
 * Writes the kp_outcome (kernel, path, features) to d_out; no host sync. */
KP_API int kp_seer_select(const void *d_off, int32_t off_type, int64_t n_rows, int64_t n_cols,
                   int64_t nnz, int64_t iterations, const void *d_selector,
                   const void *d_known, const void *d_gathered, kp_outcome *d_out,
                   void *d_ws, void *stream);

/* Row-sharded seer-core.infer (multi-GPU): d_parts holds n_parts rows of
 * (lo, hi, s1, s2) = kp_length_stats of each rank's row block (one 32-byte all-gather);
 * they combine exactly (min, max, wrapping sums) into the single-matrix reduction, so the
 * outcome equals kp_seer_select on the whole matrix.  n_rows / n_cols / nnz are GLOBAL. */
KP_API int kp_seer_select_partials(const int64_t *d_parts, int32_t n_parts, int64_t n_rows,
                                   int64_t n_cols, int64_t nnz, int64_t iterations,
                                   const void *d_selector, const void *d_known,
                                   const void *d_gathered, kp_outcome *d_out, void *stream);

/* ------------------------------------------------------------ preprocessing */
/* Bytes the caller must provide for kp_prepare(kernel, A).  ell_cap (ELL only) is
 * the width reserved for the padded part; rows longer than the actual width
 * continue from CSR (hybrid tail), so any cap >= 1 is correct. */
KP_API int kp_prepare_bytes(int32_t kernel, const kp_csr *A, int64_t ell_cap, size_t *bytes);
/* Builds the kernel's preprocessed format (MP partition K10, COO row ids K11,
 * ELL K12, adaptive row blocks K13) into d_buf.  Kernels without preprocessing
 * (BM, WM, WO, TM) just fill *out.  The prepared data stays valid while A lives. */
KP_API int kp_prepare(int32_t kernel, const kp_csr *A, int64_t ell_cap, void *d_buf, size_t bytes,
               kp_prepared *out, void *stream);

/* ------------------------------------------------------------ SpMV */
/* Scratch of kp_spmv / kp_spmv_bcast for this kernel and matrix (0 = none): carries of the
 * split-row schedules, the long-row list of CSR,WM / CSR,TM.  Zero it ONCE at allocation
 * (cudaMemset); the kernels leave it zeroed.  One workspace per stream. */
KP_API int kp_spmv_workspace_bytes(int32_t kernel, const kp_csr *A, size_t *bytes);
/* y = A . x with kernel `kernel` (KP_*).  d_x has n_cols entries, d_y n_rows, both of
 * A->val_type.  Deterministic: no floating-point atomics; repeated calls give
 * identical bits. */
KP_API int kp_spmv(int32_t kernel, const kp_csr *A, const kp_prepared *P, const void *d_x,
            void *d_y, void *d_ws, size_t ws_bytes, void *stream);

/* Fused row-sharded exchange: destinations of a rank's y slice.  y[p] = this rank's slice
 * inside rank p's next-x buffer (device pointers valid in this process: NVLink peer / NVLS
 * mappings of a symmetric allocation, or plain local buffers); y[self] is this rank's own
 * copy.  n <= KP_MAX_PEERS. */
typedef struct kp_peers {
    void *y[KP_MAX_PEERS];
    int32_t n, self;
} kp_peers;
/* kp_spmv whose y stores go to every destination in `peers` from the kernel's own epilogue
 * (and its carry fix-up), replacing the y all-gather of a row-sharded iteration (SURVEY
 * 8e) -- the transfer overlaps the SpMV tile by tile.  The caller orders the next read of x
 * after a cross-rank barrier.  Merge-path kernels (KP_CSR_MP, KP_CSR_WO); other kernels
 * return KP_EINVAL (use kp_spmv + an all-gather). */
KP_API int kp_spmv_bcast(int32_t kernel, const kp_csr *A, const kp_prepared *P, const void *d_x,
                         const kp_peers *peers, void *d_ws, size_t ws_bytes, void *stream);
/* kp_spmv_bcast with accumulation: every destination receives acc + A . x (d_acc: n_rows
 * entries of A->val_type, or NULL = kp_spmv_bcast).  d_acc may be the same buffer as
 * peers->y[peers->self].  d_rows (int32, A->n_rows entries, or NULL = identity): row r of A
 * is row d_rows[r] of the destination and of acc -- a compressed-row block (only its
 * non-empty rows) accumulating in place; requires one destination and d_acc == NULL or
 * == that destination; rows not listed are left untouched.  The column-blocked iteration
 * of a row shard whose x does not fit in L2 (dist.ShardedSeer): A split into column
 * slices, y = A_0 x + ... + A_{S-1} x accumulated block by block, the last block's stores
 * going to every rank.  Not part of the reference interface (a B200 layout choice of the
 * multi-GPU executor). */
KP_API int kp_spmv_bcast_acc(int32_t kernel, const kp_csr *A, const kp_prepared *P, const void *d_x,
                             const void *d_acc, const int32_t *d_rows, const kp_peers *peers, void *d_ws,
                             size_t ws_bytes, void *stream);

/* ------------------------------------------------------------ Seer plan (one CUDA graph) */
/* The whole pipeline -- kp_seer_select, then the chosen kernel's kp_prepare and
 * `iterations` kp_spmv -- as one CUDA graph.  Creation evaluates the selector on the
 * device for the plan's static (rows, cols, nnz, iterations): on the KNOWN path the known
 * tree's kernel is fixed there too ("known at no additional runtime cost", PAPER.md:138,
 * 141) and the graph is that kernel's body alone; on the GATHERED path every launch runs
 * the feature pass + gathered tree, whose kernel index steers a conditional SWITCH node on
 * the device (no host round trip).  d_out holds the outcome either way.  The matrix, x, y, trees,
 * outcome and reduction workspace are bound at creation; d_buf (kp_seer_plan_bytes) holds
 * every kernel's prepared format and the SpMV workspace.  `stream` must be a created
 * (non-legacy) stream; creation captures through it. */
typedef struct kp_seer_plan kp_seer_plan;
KP_API int kp_seer_plan_bytes(const kp_csr *A, int64_t ell_cap, size_t *bytes);
KP_API int kp_seer_plan_create(const kp_csr *A, int64_t iterations, int64_t ell_cap,
                               const void *d_selector, const void *d_known, const void *d_gathered,
                               const void *d_x, void *d_y, void *d_buf, size_t bytes, void *d_red_ws,
                               kp_outcome *d_out, kp_seer_plan **plan, void *stream);
KP_API int kp_seer_plan_launch(kp_seer_plan *plan, void *stream);
KP_API int kp_seer_plan_destroy(kp_seer_plan *plan);
/* How a plan selects on each launch: KP_SELECT_STATIC (known path, resolved at creation:
 * the graph is the chosen body alone), KP_SELECT_EMITTED (the bundle compiled in from
 * include/kp_seer_trees.h, used when the plan's trees equal it byte for byte),
 * KP_SELECT_PARAM (packed trees by value in the selection kernel's parameters) or
 * KP_SELECT_TABLE (trees deeper than 127 nodes, walked in device memory). */
#define KP_SELECT_STATIC 0
#define KP_SELECT_EMITTED 1
#define KP_SELECT_PARAM 2
#define KP_SELECT_TABLE 3
KP_API int kp_seer_plan_select_kind(const kp_seer_plan *plan);

/* -------------------------------------------------------- emitted trees
 * The frozen bundle's three trees compiled into the library as nested conditionals
 * (include/kp_seer_trees.h, generated by tools/emit_trees.py from models/seer_b200.json).
 * d_out[i] = tree(d_x[i*nf:]) for tree 0 = selector (nf 4), 1 = known (nf 4),
 * 2 = gathered (nf 8); the same answers as kp_tree_predict on the packed bundle. */
KP_API int kp_seer_emitted_predict(int32_t tree, const double *d_x, int64_t n, int32_t *d_out,
                                   void *stream);
/* KP_SEER_TREES_SHA256 of the compiled-in bundle (sha256 of the three packed trees). */
KP_API const char *kp_seer_emitted_sha256(void);

/* ------------------------------------------------------------ canonicalisation (COO -> CSR) */
/* Scratch bytes kp_csr_from_coo needs for n triples (n < 2^31). */
KP_API int kp_coo_workspace_bytes(int64_t n, int64_t n_rows, int64_t n_cols, size_t *bytes);
/* sparse.csr_from_coo (sparse.py:87-103) on the device: stable sort of the triples by
 * (row, col) (np.lexsort), duplicates summed exactly as np.add.reduceat does (first value +
 * numpy pairwise sum of the rest, input order), offsets from the per-row counts.
 * d_rows / d_cols int64[n], d_vals f64[n]; outputs d_off int64[n_rows+1], d_col int32[<= n],
 * d_val f64[<= n] and d_out2 (device int64[2]) = {nnz, number of out-of-range triples}
 * (the caller rejects the result when the second is non-zero). */
KP_API int kp_csr_from_coo(int64_t n_rows, int64_t n_cols, const int64_t *d_rows,
                           const int64_t *d_cols, const double *d_vals, int64_t n, int64_t *d_off,
                           int32_t *d_col, double *d_val, int64_t *d_out2, void *d_ws,
                           size_t ws_bytes, void *stream);

/* ------------------------------------------------------------ Matrix Market ingest (host) */
/* sparse.parse_matrix_market (sparse.py:106-196): header / size line / entry grammar,
 * checks and 1-based error lines as the reference (Python splitlines / strip / int / float
 * semantics for ASCII text); symmetric and skew-symmetric storage mirrored right after each
 * entry; pattern values 1.0.  Parallel native parse (OpenMP, n_threads <= 0: all). */
typedef struct kp_mm_info {
    int64_t n_rows, n_cols, n_entries;  /* size line                                  */
    int64_t n_triples;                  /* triples after symmetric expansion          */
    int32_t field;                      /* 0 real, 1 integer, 2 pattern               */
    int32_t symmetry;                   /* 0 general, 1 symmetric, 2 skew-symmetric   */
    int64_t err_line;                   /* KP_EPARSE: 1-based line of the first error */
    char err[192];                      /* KP_EPARSE: the reference's message         */
} kp_mm_info;
/* Header + size line only (capacity planning: n_entries x (symmetry ? 2 : 1)). */
KP_API int kp_mm_header(const char *buf, size_t len, kp_mm_info *info);
/* Full parse into caller arrays (0-based int64 rows / cols, f64 values, input order);
 * KP_ENOMEM with info->n_triples set when capacity is too small. */
KP_API int kp_mm_parse(const char *buf, size_t len, int64_t *rows, int64_t *cols, double *vals,
                       int64_t capacity, int32_t n_threads, kp_mm_info *info);

/* -------------------------------------------- compact host->device column transfer
 * A host-resident matrix moved every step is PCIe-bound; its column indices need only
 * b = kp_pack_bits(n_cols) = ceil(log2(n_cols)) bits.  kp_pack_cols (HOST, OpenMP) writes
 * them as one little-endian bitstream of 32-bit words (column i at bits [i*b, (i+1)*b)),
 * kp_pack_cols_bytes bytes; kp_unpack_cols (DEVICE, async) restores the int32 array the
 * SpMV entry points read.  KP_ERANGE from kp_pack_cols: a column outside [0, n_cols). */
KP_API int32_t kp_pack_bits(int64_t n_cols);
KP_API size_t kp_pack_cols_bytes(int64_t n, int64_t n_cols);
KP_API int kp_pack_cols(const int32_t *h_cols, int64_t n, int64_t n_cols, uint32_t *h_out,
                        int32_t n_threads);
KP_API int kp_unpack_cols(const uint32_t *d_packed, int64_t n, int64_t n_cols, int32_t *d_cols,
                          void *stream);

/* ------------------------------------------------------------ multi-GPU (K14) */
/* nnz-balanced row cut: d_cuts[p] = lower_bound(row_offsets, p*nnz/parts), p = 0..parts
 * (d_cuts[parts] = n_rows). */
KP_API int kp_shard_partition(const void *d_off, int32_t off_type, int64_t n_rows, int32_t parts,
                       int64_t *d_cuts, void *stream);

/* ------------------------------------------------------------ failure detection (multi-GPU) */
/* Watchdog over an NCCL communicator (no reference counterpart): a native thread
 * polls ncclCommGetAsyncError every poll_ms and the host heartbeat; on an NCCL error, or no
 * heartbeat for timeout_ms (a hung collective or peer; 0 = no timeout), it calls
 * ncclCommAbort so blocked collectives return.  `nccl_comm` is an ncclComm_t (e.g. torch's
 * ProcessGroupNCCL._comm_ptr()); NCCL symbols come from the process's libnccl.so.2
 * (KP_EUNSUPPORTED when absent).  heartbeat / status / stop return the state below. */
#define KP_WD_OK 0
#define KP_WD_NCCL_ERROR 1
#define KP_WD_TIMEOUT 2
typedef struct kp_watchdog kp_watchdog;
KP_API int kp_watchdog_start(void *nccl_comm, int64_t timeout_ms, int64_t poll_ms, kp_watchdog **out);
KP_API int kp_watchdog_heartbeat(kp_watchdog *w);
KP_API int kp_watchdog_status(kp_watchdog *w, int32_t *nccl_result, char *msg, size_t msg_len);
KP_API int kp_watchdog_stop(kp_watchdog *w);

/* Library identification: "kpb200 <version> sm_100a". */
KP_API const char *kp_version(void);
/* Number of kernel launches issued by this library since load (instrumentation). */
KP_API uint64_t kp_launch_count(void);
/* Test hook: number of resident warps the persistent work distribution (CSR,MP / CSR,WO /
 * COO,WM) targets; 0 = one full wave from the occupancy API (default).  Small values force
 * many units per warp on small matrices.  Affects kp_prepare and kp_spmv alike; returns
 * the previous value. */
KP_API int64_t kp_debug_set_wave_warps(int64_t warps);

#ifdef __cplusplus
}
#endif
#endif /* KERNELPICK_B200_H */
