// Launch-latency floor on B200: event-to-event time of an (almost) empty kernel with the fused
// operator's launch shape (201 x 512 threads, ~100 KB dynamic smem), normal vs cooperative, with
// and without a 256 MB L2-flush kernel in front.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void body(int* p) { if (threadIdx.x == 0 && p[blockIdx.x] == 12345) p[0] = 1; }
__global__ void flushk(int* f, size_t n) { for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) f[i] += 1; }
int main() {
    int* p; cudaMalloc(&p, 1 << 20); cudaMemset(p, 0, 1 << 20);
    int* f; size_t nf = 64u << 20; cudaMalloc(&f, nf * 4);
    cudaFuncSetAttribute(body, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int shapes[][2] = {{1, 32}, {148, 128}, {148, 256}, {148, 512}, {201, 512}, {296, 256}, {148, 1024}};
    for (auto& sh : shapes)
    for (int smem : {0, 100 * 1024})
    for (int coop = 0; coop < 2; ++coop)
    for (int fl = 0; fl < 2; ++fl) {
        if (coop && fl == 0) continue;
        float tot = 0; int n = 0;
        for (int it = 0; it < 60; ++it) {
            if (fl) flushk<<<1184, 256>>>(f, nf);
            cudaEventRecord(e0);
            if (coop) { void* args[] = {&p}; cudaLaunchCooperativeKernel((void*)body, dim3(sh[0]), dim3(sh[1]), args, smem, 0); }
            else body<<<sh[0], sh[1], smem>>>(p);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 10) { tot += ms; ++n; }
        }
        printf("grid %3d x %4d smem %6d coop %d flush %d: %.2f us\n", sh[0], sh[1], smem, coop, fl, 1e3 * tot / n);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
