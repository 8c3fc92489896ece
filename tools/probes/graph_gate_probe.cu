// Gated parallel bodies vs a SWITCH node for a realistic body length: a selection kernel
// followed by L kernels (one body of a plan: prepare + iterations x spmv).
//   (a) plain chain 1 + L        (b) set kernel + SWITCH(8), body = L kernels
//   (c) set kernel + 8 parallel branches of L gated kernels (grid G, all but one exit)
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 graph_gate_probe.cu -o graph_gate_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_work(int *p) { if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p, 1); }
__global__ void k_set(cudaGraphConditionalHandle h, unsigned v, int *gates) {
    if (gates) { for (int i = 0; i < 8; ++i) gates[i] = i != (int)v; }
    else cudaGraphSetConditional(h, v);
}
__global__ void k_gated(const int *gate, int *p) {
    if (*gate) return;
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p, 1);
}

static float time_graph(cudaGraph_t g, cudaStream_t s, int reps) {
    cudaGraphExec_t e;
    if (cudaGraphInstantiate(&e, g, 0) != cudaSuccess) return -1.f;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 20; ++i) cudaGraphLaunch(e, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    for (int i = 0; i < reps; ++i) cudaGraphLaunch(e, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaGraphExecDestroy(e);
    return 1000.f * ms / reps;
}

int main() {
    int *d, *gates;
    cudaMalloc(&d, 4); cudaMalloc(&gates, 64);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaStream_t br[8]; cudaEvent_t fork, join[8];
    cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    for (int i = 0; i < 8; ++i) { cudaStreamCreate(&br[i]); cudaEventCreateWithFlags(&join[i], cudaEventDisableTiming); }
    const int reps = 2000;
    const int Ls[] = {2, 4, 11, 21};
    const int Gs[] = {1, 148, 1184, 8192};
    for (int L : Ls) {
        cudaGraph_t g;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i <= L; ++i) k_work<<<148, 256, 0, s>>>(d);
        cudaStreamEndCapture(s, &g);
        printf("L=%2d chain 1+L            : %6.2f us\n", L, time_graph(g, s, reps));
        cudaGraphDestroy(g);
        cudaGraphConditionalHandle h;
        cudaGraphCreate(&g, 0);
        cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault);
        cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
        k_set<<<1, 1, 0, s>>>(h, 3, nullptr);
        cudaStreamEndCapture(s, &g);
        size_t n = 0; cudaGraphGetNodes(g, nullptr, &n);
        cudaGraphNode_t nodes[4]; cudaGraphGetNodes(g, nodes, &n);
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeSwitch; cp.conditional.size = 8;
        cudaGraphNode_t cn; cudaGraphAddNode(&cn, g, &nodes[n - 1], 1, &cp);
        for (int b = 0; b < 8; ++b) {
            cudaStreamBeginCaptureToGraph(s, cp.conditional.phGraph_out[b], nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
            for (int i = 0; i < L; ++i) k_work<<<148, 256, 0, s>>>(d);
            cudaGraph_t tmp; cudaStreamEndCapture(s, &tmp);
        }
        printf("L=%2d set + SWITCH(8)      : %6.2f us\n", L, time_graph(g, s, reps));
        cudaGraphDestroy(g);
        for (int G : Gs) {
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            k_set<<<1, 1, 0, s>>>(0, 3, gates);
            cudaEventRecord(fork, s);
            for (int b = 0; b < 8; ++b) {
                cudaStreamWaitEvent(br[b], fork, 0);
                for (int i = 0; i < L; ++i) k_gated<<<G, 256, 0, br[b]>>>(gates + b, d);
                cudaEventRecord(join[b], br[b]);
                cudaStreamWaitEvent(s, join[b], 0);
            }
            cudaStreamEndCapture(s, &g);
            printf("L=%2d set + 8 gated G=%5d : %6.2f us\n", L, G, time_graph(g, s, reps));
            cudaGraphDestroy(g);
        }
    }
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
