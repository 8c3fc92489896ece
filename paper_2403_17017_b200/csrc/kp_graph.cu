// kp_graph.cu -- the whole Seer pipeline as ONE CUDA graph with device-side dispatch.
//
// Known-path plans (selector -> USE_KNOWN on the plan's static shape, resolved on the device
// at creation) are the chosen kernel's body alone.  Gathered-path plans:
//   [k_seer_plan_select: selector -> feature pass -> tree, cudaGraphSetConditional(h, kernel)]
//        -> SWITCH(h) { body i = kp_prepare(i) + iterations x kp_spmv(i), i = 0..7 }
//
// The three trees are copied to the host once at creation and passed BY VALUE to the
// selection kernel (parameter space), which also sets the switch value: one launch before
// the body.  Trees deeper than the parameter table fall back to kp_seer_select (trees in
// device memory) + a separate set-switch kernel.
//
// SPEC.md:376-384 infer followed by the chosen kernel's preprocessing and k iterations
// (SURVEY 8d T_seer) with no host round trip: the kernel index written by the selection
// kernel steers the conditional node on the device.  Each body is captured
// through the same C-ABI calls a host-driven run makes (cudaStreamBeginCaptureToGraph),
// so graph and eager runs execute identical kernels.  Buffers are carved from one
// caller allocation (kp_seer_plan_bytes); x / y / the matrix are bound at creation.
#include <cuda.h>
#include <stdlib.h>

#include "kp_internal.cuh"

struct kp_seer_plan {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphConditionalHandle handle = 0;
    int32_t static_kernel = -1;  // >= 0: known-path plan (body only, no SWITCH)
    int32_t select_kind = KP_SELECT_STATIC;
    kp_prepared prep[KP_NUM_KERNELS] = {};
};

namespace kp {
int ensure_kernel_attrs();
namespace {

constexpr size_t kAl = 256;
size_t al(size_t v) { return (v + kAl - 1) / kAl * kAl; }

__global__ void k_set_switch(cudaGraphConditionalHandle h, const kp_outcome *o) {
    const int k = o->kernel;
    cudaGraphSetConditional(h, (k >= 0 && k < KP_NUM_KERNELS) ? (unsigned)k : (unsigned)KP_NUM_KERNELS);
}

struct PlanLayout {
    size_t prep[KP_NUM_KERNELS] = {};
    size_t prep_off[KP_NUM_KERNELS] = {};
    size_t ws = 0, ws_off = 0, total = 0;
};

int plan_layout(const kp_csr *A, int64_t ell_cap, PlanLayout *L) {
    size_t o = 0;
    for (int k = 0; k < KP_NUM_KERNELS; ++k) {
        size_t b = 0;
        int rc = kp_prepare_bytes(k, A, k == KP_ELL_TM ? ell_cap : 0, &b);
        if (rc) return rc;
        L->prep[k] = b;
        L->prep_off[k] = o;
        o += al(b);
        size_t w = 0;
        rc = kp_spmv_workspace_bytes(k, A, &w);
        if (rc) return rc;
        if (w > L->ws) L->ws = w;
    }
    L->ws_off = o;
    o += al(L->ws);
    L->total = o;
    return KP_OK;
}

}  // namespace
}  // namespace kp

using namespace kp;

extern "C" {

int kp_seer_plan_bytes(const kp_csr *A, int64_t ell_cap, size_t *bytes) {
    if (!bytes || ell_cap < 1) return KP_EINVAL;
    PlanLayout L;
    const int rc = plan_layout(A, ell_cap, &L);
    if (rc) return rc;
    *bytes = L.total;
    return KP_OK;
}

int kp_seer_plan_create(const kp_csr *A, int64_t iterations, int64_t ell_cap, const void *d_selector,
                        const void *d_known, const void *d_gathered, const void *d_x, void *d_y, void *d_buf,
                        size_t bytes, void *d_red_ws, kp_outcome *d_out, kp_seer_plan **plan_out, void *stream) {
    KP_NVTX("kp_seer_plan_create");
    if (!plan_out || !d_buf || !d_out || !d_red_ws || iterations < 1 || ell_cap < 1 || !d_y) return KP_EINVAL;
    if (((uintptr_t)d_buf & (kAl - 1)) != 0) return KP_EINVAL;
    PlanLayout L;
    int rc = plan_layout(A, ell_cap, &L);
    if (rc) return rc;
    if (bytes < L.total) return KP_ENOMEM;
    cudaStream_t s = (cudaStream_t)stream;
    if (!s) return KP_EINVAL;  // capture needs a real (non-legacy) stream
    rc = ensure_kernel_attrs();  // no attribute calls inside the capture
    if (rc) return rc;
    unsigned char *base = reinterpret_cast<unsigned char *>(d_buf);
    // trees small enough to travel by value (depth <= 6) -> single-kernel selection
    ParamTrees *trees = new ParamTrees();
    const bool use_param_trees = plan_trees_load(d_selector, d_known, d_gathered, trees) == KP_OK;
    cudaGetLastError();
    // the bundle compiled in from include/kp_seer_trees.h, when these are its trees
    // (KP_NO_EMITTED_TREES=1 forces the interpreter, for A/B timing)
    const char *no_emit = getenv("KP_NO_EMITTED_TREES");
    const bool use_emitted = use_param_trees && !(no_emit && no_emit[0] == '1') && emitted_trees_match(*trees);
    struct TreesGuard {
        ParamTrees *t;
        ~TreesGuard() { delete t; }
    } guard{trees};
    kp_seer_plan *P = new kp_seer_plan();
    auto fail = [&](int code) {
        if (P->exec) cudaGraphExecDestroy(P->exec);
        if (P->graph) cudaGraphDestroy(P->graph);
        delete P;
        cudaGetLastError();
        return code;
    };
    if (cudaGraphCreate(&P->graph, 0) != cudaSuccess) return fail(KP_ECUDA);
    void *ws = base + L.ws_off;
    // the SpMV workspace starts zeroed (the row-mapped schedules' long-row list counter;
    // kernels leave it zeroed again) -- once, here, outside any capture
    if (L.ws && cudaMemsetAsync(ws, 0, L.ws, s) != cudaSuccess) return fail(KP_ECUDA);
    // 0) Known-feature decisions depend only on the plan's static shape (rows, cols, nnz,
    //    iterations): "known at no additional runtime cost".  Evaluate
    //    the selector (and, on the known path, the known tree) on the device once, now.
    //    KNOWN -> the graph is the chosen kernel's body alone; GATHERED -> the feature pass
    //    runs every launch and steers a SWITCH node on the device.
    rc = kp_seer_select(A->row_offsets, A->off_type, A->n_rows, A->n_cols, A->nnz, iterations, d_selector, d_known,
                        d_gathered, d_out, d_red_ws, s);
    if (rc) return fail(rc);
    kp_outcome o0;
    if (cudaMemcpyAsync(&o0, d_out, sizeof(o0), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(KP_ECUDA);
    if (o0.path == KP_USE_KNOWN && o0.kernel >= 0 && o0.kernel < KP_NUM_KERNELS) {
        const int k = o0.kernel;
        if (cudaStreamBeginCaptureToGraph(s, P->graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
            cudaSuccess)
            return fail(KP_ECUDA);
        rc = kp_prepare(k, A, k == KP_ELL_TM ? ell_cap : 0, base + L.prep_off[k], L.prep[k], &P->prep[k], s);
        for (int64_t it = 0; rc == KP_OK && it < iterations; ++it)
            rc = kp_spmv(k, A, &P->prep[k], d_x, d_y, ws, L.ws, s);
        cudaGraph_t got = nullptr;
        if (cudaStreamEndCapture(s, &got) != cudaSuccess || rc != KP_OK) return fail(rc ? rc : KP_ECUDA);
        P->static_kernel = k;
        if (cudaGraphInstantiate(&P->exec, P->graph, 0) != cudaSuccess) return fail(KP_ECUDA);
        *plan_out = P;
        return KP_OK;
    }
    if (cudaGraphConditionalHandleCreate(&P->handle, P->graph, KP_NUM_KERNELS, cudaGraphCondAssignDefault) !=
        cudaSuccess)
        return fail(KP_ECUDA);
    // 1) selection + switch value
    if (cudaStreamBeginCaptureToGraph(s, P->graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
        cudaSuccess)
        return fail(KP_ECUDA);
    if (use_param_trees) {
        // one kernel: selection with the trees in its parameter space, sets the SWITCH value
        rc = launch_plan_select(A->row_offsets, A->off_type, A->n_rows, A->n_cols, A->nnz, iterations, *trees,
                                use_emitted, d_out, d_red_ws, P->handle, s);
        P->select_kind = use_emitted ? KP_SELECT_EMITTED : KP_SELECT_PARAM;
    } else {
        rc = kp_seer_select(A->row_offsets, A->off_type, A->n_rows, A->n_cols, A->nnz, iterations, d_selector,
                            d_known, d_gathered, d_out, d_red_ws, s);
        P->select_kind = KP_SELECT_TABLE;
        if (rc == KP_OK) {
            k_set_switch<<<1, 1, 0, s>>>(P->handle, d_out);
            ++g_launches;
        }
    }
    cudaGraph_t captured = nullptr;
    if (cudaStreamEndCapture(s, &captured) != cudaSuccess || rc != KP_OK) return fail(rc ? rc : KP_ECUDA);
    // the leaf of the captured chain is the set-switch kernel
    size_t n = 0;
    cudaGraphGetNodes(P->graph, nullptr, &n);
    cudaGraphNode_t *nodes = (cudaGraphNode_t *)malloc(n * sizeof(cudaGraphNode_t));
    cudaGraphGetNodes(P->graph, nodes, &n);
    cudaGraphNode_t leaf = nullptr;
    for (size_t i = 0; i < n; ++i) {
        size_t nd = 0;
        cudaGraphNodeGetDependentNodes(nodes[i], nullptr, &nd);
        if (nd == 0) leaf = nodes[i];
    }
    free(nodes);
    if (!leaf) return fail(KP_ECUDA);
    // 2) SWITCH node: body k = prepare(k) + iterations x spmv(k)
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = P->handle;
    cp.conditional.type = cudaGraphCondTypeSwitch;
    cp.conditional.size = KP_NUM_KERNELS;
    cudaGraphNode_t cnode;
    if (cudaGraphAddNode(&cnode, P->graph, &leaf, 1, &cp) != cudaSuccess) return fail(KP_ECUDA);
    for (int k = 0; k < KP_NUM_KERNELS; ++k) {
        cudaGraph_t body = cp.conditional.phGraph_out[k];
        if (cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
            cudaSuccess)
            return fail(KP_ECUDA);
        rc = kp_prepare(k, A, k == KP_ELL_TM ? ell_cap : 0, base + L.prep_off[k], L.prep[k], &P->prep[k], s);
        for (int64_t it = 0; rc == KP_OK && it < iterations; ++it)
            rc = kp_spmv(k, A, &P->prep[k], d_x, d_y, ws, L.ws, s);
        cudaGraph_t got = nullptr;
        if (cudaStreamEndCapture(s, &got) != cudaSuccess || rc != KP_OK) return fail(rc ? rc : KP_ECUDA);
    }
    if (cudaGraphInstantiate(&P->exec, P->graph, 0) != cudaSuccess) return fail(KP_ECUDA);
    *plan_out = P;
    return KP_OK;
}

int kp_seer_plan_launch(kp_seer_plan *plan, void *stream) {
    KP_NVTX("kp_seer_plan_launch");
    if (!plan || !plan->exec) return KP_EINVAL;
    if (cudaGraphLaunch(plan->exec, (cudaStream_t)stream) != cudaSuccess) {
        cudaGetLastError();
        return KP_ECUDA;
    }
    return KP_OK;
}

int kp_seer_plan_select_kind(const kp_seer_plan *plan) { return plan ? plan->select_kind : KP_EINVAL; }

int kp_seer_plan_destroy(kp_seer_plan *plan) {
    if (!plan) return KP_EINVAL;
    if (plan->exec) cudaGraphExecDestroy(plan->exec);
    if (plan->graph) cudaGraphDestroy(plan->graph);
    delete plan;
    return KP_OK;
}

}  // extern "C"
