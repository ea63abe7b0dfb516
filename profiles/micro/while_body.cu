// Micro-benchmark: per-iteration cost of a CUDA-graph WHILE conditional node, vs the same kernels
// in a plain unrolled graph and as stream launches.  Body = K dependent tiny kernels; the last one
// counts iterations and clears the condition after N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o while_body while_body.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void work(double* v, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = v[i] * 0.999 + 1.0;
}
__global__ void ctl(int* it, int n, cudaGraphConditionalHandle h) {
    if (++*it >= n) cudaGraphSetConditional(h, 0);
}
__global__ void ctl_plain(int* it) { ++*it; }

int main(int argc, char** argv) {
    const int N = 1000, n = argc > 1 ? atoi(argv[1]) : 262144;  // elements per work kernel
    double* v;
    int* it;
    CK(cudaMalloc(&v, n * 8));
    CK(cudaMalloc(&it, 4));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int K : {1, 4, 8}) {
        // WHILE graph
        cudaGraph_t g;
        CK(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        for (int k = 0; k < K; ++k) work<<<(n + 255) / 256, 256, 0, s>>>(v, n);
        ctl<<<1, 1, 0, s>>>(it, N, h);
        CK(cudaStreamEndCapture(s, &body));
        cudaGraphExec_t ex;
        CK(cudaGraphInstantiate(&ex, g, 0));
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaMemsetAsync(it, 0, 4, s));
            CK(cudaEventRecord(a, s));
            CK(cudaGraphLaunch(ex, s));
            CK(cudaEventRecord(b, s));
            CK(cudaStreamSynchronize(s));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            best = ms < best ? ms : best;
        }
        // unrolled plain graph of N iterations
        cudaGraph_t g2;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        for (int i = 0; i < N; ++i) {
            for (int k = 0; k < K; ++k) work<<<(n + 255) / 256, 256, 0, s>>>(v, n);
            ctl_plain<<<1, 1, 0, s>>>(it);
        }
        CK(cudaStreamEndCapture(s, &g2));
        cudaGraphExec_t ex2;
        CK(cudaGraphInstantiate(&ex2, g2, 0));
        float best2 = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(a, s));
            CK(cudaGraphLaunch(ex2, s));
            CK(cudaEventRecord(b, s));
            CK(cudaStreamSynchronize(s));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            best2 = ms < best2 ? ms : best2;
        }
        // stream launches
        float best3 = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(a, s));
            for (int i = 0; i < N; ++i) {
                for (int k = 0; k < K; ++k) work<<<(n + 255) / 256, 256, 0, s>>>(v, n);
                ctl_plain<<<1, 1, 0, s>>>(it);
            }
            CK(cudaEventRecord(b, s));
            CK(cudaStreamSynchronize(s));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            best3 = ms < best3 ? ms : best3;
        }
        std::printf("n=%d K=%d kernels + ctl per iteration: WHILE %.2f us/iter, unrolled graph %.2f us/iter, stream %.2f us/iter\n",
                    n, K, best * 1e3f / N, best2 * 1e3f / N, best3 * 1e3f / N);
        cudaGraphExecDestroy(ex);
        cudaGraphExecDestroy(ex2);
        cudaGraphDestroy(g);
        cudaGraphDestroy(g2);
    }
    return 0;
}
