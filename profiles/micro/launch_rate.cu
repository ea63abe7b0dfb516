// Back-to-back launch cost on one stream: N empty kernels between two events, plain launches vs
// one CUDA graph holding the same N kernels.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty(int* p) { if (threadIdx.x == 0 && p[blockIdx.x] == 12345) p[0] = 1; }
int main() {
    int* p; cudaMalloc(&p, 1 << 20); cudaMemset(p, 0, 1 << 20);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int grid : {1, 148, 592}) {
        const int N = 100;
        for (int w = 0; w < 3; ++w) empty<<<grid, 128, 0, s>>>(p);
        cudaEventRecord(e0, s);
        for (int i = 0; i < N; ++i) empty<<<grid, 128, 0, s>>>(p);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < N; ++i) empty<<<grid, 128, 0, s>>>(p);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float mg; cudaEventElapsedTime(&mg, e0, e1);
        printf("grid %4d: plain %.2f us/launch, graph %.2f us/kernel\n", grid, 1e3 * ms / N, 1e3 * mg / N);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
