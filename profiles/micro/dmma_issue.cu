// DMMA m8n8k4 issue model on sm_100a: TFLOP/s vs warps per SM and independent chains per warp,
// with and without shared-memory operand loads between the MMAs.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int CH, bool LDS>
__global__ void k(int iters, double seed, double* sink) {
    __shared__ double sa[64][33];
    const int lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < 64 * 33; e += blockDim.x) (&sa[0][0])[e] = seed + e * 1e-9;
    __syncthreads();
    double acc[CH][2];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
    double a = seed + lane, b = seed - lane;
    for (int it = 0; it < iters; ++it) {
        if (LDS) {
            a = sa[(it & 31) + (lane & 3)][lane >> 2];
            b = sa[32 + (lane & 3)][(it & 31)];
        }
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(acc[c], a, b);
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) t += acc[c][0] + acc[c][1];
    if (t == 12345.678) *sink = t;
}
template <int CH, bool LDS>
void run(int warps_per_block, int blocks_per_sm, int sms) {
    double* sink; cudaMalloc(&sink, 8);
    int iters = 4096 * 8 / CH;
    dim3 g(sms * blocks_per_sm), b(32 * warps_per_block);
    k<CH, LDS><<<g, b>>>(iters, 1.0, sink);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<CH, LDS><<<g, b>>>(iters, 1.0, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * CH * (double)iters * g.x * warps_per_block;
    printf("chains %2d lds %d warps/SM %3d : %6.2f TF\n", CH, (int)LDS, warps_per_block * blocks_per_sm, fl / ms / 1e9);
    cudaFree(sink);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 16, 32}) {
        run<4, false>(w, 1, sms); run<8, false>(w, 1, sms); run<16, false>(w, 1, sms); run<32, false>(w, 1, sms);
        run<16, true>(w, 1, sms);
    }
    run<8, false>(8, 8, sms);
    return 0;
}
