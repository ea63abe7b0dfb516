// DMMA throughput of the MTTKRP consumer pattern: per k-step a warp loads 4 A and 4 B fragments
// from shared memory (conflict-free pitches) and issues the 4 x 4 = 16 DMMAs; 8 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(int iters, double* sink) {
    __shared__ double sa[32][132];
    __shared__ double sb[32][36];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, kq = lane & 3, g = lane >> 2;
    for (int e = threadIdx.x; e < 32 * 132; e += blockDim.x) (&sa[0][0])[e] = 1e-3 * e;
    for (int e = threadIdx.x; e < 32 * 36; e += blockDim.x) (&sb[0][0])[e] = 1e-3 * e;
    __syncthreads();
    double acc[4][4][2];
    for (int x = 0; x < 4; ++x) for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0;
    const int rg = warp & 3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) {
            const int kr = ((it & 1) * 16 + (warp >> 2) * 8 + k2 * 2) % 32 + (kq & 1);
            double af[4], bf[4];
#pragma unroll
            for (int mf = 0; mf < 4; ++mf) af[mf] = MODE == 0 ? sa[kr][rg * 32 + mf * 8 + g] : 1.0 + mf;
#pragma unroll
            for (int nf = 0; nf < 4; ++nf) bf[nf] = MODE == 0 ? sb[nf * 8 + g][kr] : 2.0 + nf;
#pragma unroll
            for (int mf = 0; mf < 4; ++mf)
#pragma unroll
                for (int nf = 0; nf < 4; ++nf) dmma(acc[mf][nf], af[mf], bf[nf]);
        }
    }
    double t = 0;
    for (int x = 0; x < 4; ++x) for (int y = 0; y < 4; ++y) t += acc[x][y][0] + acc[x][y][1];
    if (t == 1.2345) *sink = t;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink; cudaMalloc(&sink, 8);
    for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8, 16}) {
        const int iters = 2048;
        auto kern = mode == 0 ? k<0> : k<1>;
        kern<<<sms, 32 * warps>>>(iters, sink);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kern<<<sms, 32 * warps>>>(iters, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 2.0 * 256 * 16 * 4 * (double)iters * sms * warps;
        printf("mode %s warps/SM %2d: %.2f TF\n", mode == 0 ? "lds" : "reg", warps, fl / ms / 1e9);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
