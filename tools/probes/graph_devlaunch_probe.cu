// Device graph launch (tail launch from a kernel) as an alternative to a SWITCH node.
// nvcc -gencode arch=compute_100a,code=sm_100a -rdc=true -O2 graph_devlaunch_probe.cu -lcudadevrt -o graph_devlaunch_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tiny(int *p) { if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p, 1); }
__global__ void k_pick(cudaGraphExec_t *execs, int which) {
    if (threadIdx.x == 0 && blockIdx.x == 0) cudaGraphLaunch(execs[which], cudaStreamGraphTailLaunch);
}

int main() {
    int *d; cudaMalloc(&d, 4); cudaMemset(d, 0, 4);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaGraphExec_t hexec[8];
    for (int i = 0; i < 8; ++i) {
        cudaGraph_t g;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        k_tiny<<<1, 32, 0, s>>>(d);
        cudaStreamEndCapture(s, &g);
        cudaError_t e1 = cudaGraphInstantiate(&hexec[i], g, cudaGraphInstantiateFlagDeviceLaunch);
        cudaError_t e2 = cudaGraphUpload(hexec[i], s);
        if (e1 || e2) { printf("instantiate/upload: %s %s\n", cudaGetErrorString(e1), cudaGetErrorString(e2)); return 1; }
    }
    cudaGraphExec_t *dexec; cudaMalloc(&dexec, sizeof(hexec));
    cudaMemcpy(dexec, hexec, sizeof(hexec), cudaMemcpyHostToDevice);
    for (int variant = 0; variant < 2; ++variant) {
        cudaGraph_t pg; cudaGraphExec_t pe;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        k_tiny<<<1, 32, 0, s>>>(d);
        k_pick<<<1, 32, 0, s>>>(dexec, 3);
        cudaStreamEndCapture(s, &pg);
        cudaError_t e = cudaGraphInstantiate(&pe, pg, variant ? cudaGraphInstantiateFlagDeviceLaunch : 0);
        if (e) { printf("parent instantiate (flag %d): %s\n", variant, cudaGetErrorString(e)); continue; }
        if (variant) cudaGraphUpload(pe, s);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int i = 0; i < 10; ++i) cudaGraphLaunch(pe, s);
        cudaError_t se = cudaStreamSynchronize(s);
        if (se) { printf("run (flag %d): %s\n", variant, cudaGetErrorString(se)); return 1; }
        int before; cudaMemcpy(&before, d, 4, cudaMemcpyDeviceToHost);
        const int reps = 2000;
        cudaEventRecord(a, s);
        for (int i = 0; i < reps; ++i) cudaGraphLaunch(pe, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        int after; cudaMemcpy(&after, d, 4, cudaMemcpyDeviceToHost);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("parent flag=%d: kernel + tail-launched body: %.2f us/launch (body ran %d times / %d)\n", variant,
               1000.f * ms / reps, (after - before) - reps, reps);
    }
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
