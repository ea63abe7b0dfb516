// lanegroup.cuh — reductions over lane groups of G consecutive lanes (full-warp participation).
#pragma once

namespace cphifi {

// Sum each of d[0..B) over the G lanes of the caller's lane group; every lane ends with all B
// totals.  Reduce-scatter over offsets G/2 .. G/B (each step halves the values a lane carries),
// butterfly over the remaining offsets, then all-gather in reverse: for G = 8, B = 4 that is 7
// double shuffles and 4 adds instead of 12 and 12.  Every lane of the warp must call it (full
// mask).  Fixed order: deterministic.
template <int B, int G>
__device__ __forceinline__ void group_reduce(double (&d)[B], int lane) {
    if constexpr (G == 1) {
        return;
    } else if constexpr (B == 1 || B > G) {
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1) d[i] += __shfl_xor_sync(0xffffffffu, d[i], off, G);
    } else {
        double v[B];
#pragma unroll
        for (int i = 0; i < B; ++i) v[i] = d[i];
        int w = B;
        int off = G / 2;
#pragma unroll
        for (int st = 0; (1 << st) < B; ++st) {
            const bool hi = (lane & off) != 0;
            const int h = w / 2;
#pragma unroll
            for (int i = 0; i < h; ++i) {
                const double keep = hi ? v[i + h] : v[i];
                const double send = hi ? v[i] : v[i + h];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off, G);
            }
            w = h;
            off >>= 1;
        }
#pragma unroll
        for (; off > 0; off >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], off, G);
        int wg = 1;
        int og = G / B;
#pragma unroll
        for (int st = 0; (1 << st) < B; ++st) {
            const bool hi = (lane & og) != 0;
#pragma unroll
            for (int i = 0; i < wg; ++i) {
                const double other = __shfl_xor_sync(0xffffffffu, v[i], og, G);
                const double mine = v[i];
                v[i] = hi ? other : mine;
                v[i + wg] = hi ? mine : other;
            }
            wg *= 2;
            og *= 2;
        }
#pragma unroll
        for (int i = 0; i < B; ++i) d[i] = v[i];
    }
}

}  // namespace cphifi
