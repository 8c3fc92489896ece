// Cost of device-side dispatch structures inside a CUDA graph (B200): a chain of two tiny
// kernels vs a SWITCH conditional node (8 bodies) vs an IF node vs 8 parallel gated branches.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 graph_cond_probe.cu -o graph_cond_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tiny(int *p) { if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p, 1); }
__global__ void k_set_switch(cudaGraphConditionalHandle h, unsigned v) { cudaGraphSetConditional(h, v); }
__global__ void k_gate(const int *sel, int me, int *p) {
    if (*sel != me) return;
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p, 1);
}

static float time_graph(cudaGraphExec_t e, cudaStream_t s, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) cudaGraphLaunch(e, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    for (int i = 0; i < reps; ++i) cudaGraphLaunch(e, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return 1000.f * ms / reps;
}

int main() {
    int *d, *sel;
    cudaMalloc(&d, 4); cudaMalloc(&sel, 4);
    cudaMemset(sel, 0, 4);
    cudaStream_t s; cudaStreamCreate(&s);
    const int reps = 2000;
    // (a) chain of 2 tiny kernels
    {
        cudaGraph_t g; cudaGraphExec_t e;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        k_tiny<<<1, 32, 0, s>>>(d); k_tiny<<<1, 32, 0, s>>>(d);
        cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&e, g, 0);
        printf("chain of 2 tiny kernels      : %.2f us/launch\n", time_graph(e, s, reps));
    }
    // (b) set-switch kernel -> SWITCH(8) with a tiny kernel per body
    {
        cudaGraph_t g; cudaGraphExec_t e; cudaGraphConditionalHandle h;
        cudaGraphCreate(&g, 0);
        cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault);
        cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
        k_set_switch<<<1, 1, 0, s>>>(h, 3);
        cudaStreamEndCapture(s, &g);
        size_t n = 0; cudaGraphGetNodes(g, nullptr, &n);
        cudaGraphNode_t nodes[8]; cudaGraphGetNodes(g, nodes, &n);
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeSwitch; cp.conditional.size = 8;
        cudaGraphNode_t cn; cudaGraphAddNode(&cn, g, &nodes[n - 1], 1, &cp);
        for (int i = 0; i < 8; ++i) {
            cudaStreamBeginCaptureToGraph(s, cp.conditional.phGraph_out[i], nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
            k_tiny<<<1, 32, 0, s>>>(d);
            cudaGraph_t tmp; cudaStreamEndCapture(s, &tmp);
        }
        cudaGraphInstantiate(&e, g, 0);
        printf("set kernel + SWITCH(8)       : %.2f us/launch\n", time_graph(e, s, reps));
    }
    // (c) set kernel -> IF
    {
        cudaGraph_t g; cudaGraphExec_t e; cudaGraphConditionalHandle h;
        cudaGraphCreate(&g, 0);
        cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault);
        cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
        k_set_switch<<<1, 1, 0, s>>>(h, 1);
        cudaStreamEndCapture(s, &g);
        size_t n = 0; cudaGraphGetNodes(g, nullptr, &n);
        cudaGraphNode_t nodes[8]; cudaGraphGetNodes(g, nodes, &n);
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf; cp.conditional.size = 1;
        cudaGraphNode_t cn; cudaGraphAddNode(&cn, g, &nodes[n - 1], 1, &cp);
        cudaStreamBeginCaptureToGraph(s, cp.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
        k_tiny<<<1, 32, 0, s>>>(d);
        cudaGraph_t tmp; cudaStreamEndCapture(s, &tmp);
        cudaGraphInstantiate(&e, g, 0);
        printf("set kernel + IF              : %.2f us/launch\n", time_graph(e, s, reps));
    }
    // (d) kernel -> 8 parallel gated branches (fork/join via events)
    {
        cudaGraph_t g; cudaGraphExec_t e;
        cudaStream_t br[8]; cudaEvent_t fork, join[8];
        cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
        for (int i = 0; i < 8; ++i) { cudaStreamCreate(&br[i]); cudaEventCreateWithFlags(&join[i], cudaEventDisableTiming); }
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        k_tiny<<<1, 32, 0, s>>>(d);
        cudaEventRecord(fork, s);
        for (int i = 0; i < 8; ++i) {
            cudaStreamWaitEvent(br[i], fork, 0);
            k_gate<<<148, 256, 0, br[i]>>>(sel, i, d);
            cudaEventRecord(join[i], br[i]);
            cudaStreamWaitEvent(s, join[i], 0);
        }
        cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&e, g, 0);
        printf("kernel + 8 gated branches    : %.2f us/launch\n", time_graph(e, s, reps));
    }
    cudaError_t err = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(err));
    return 0;
}
