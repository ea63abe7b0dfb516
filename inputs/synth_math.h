/*
 * synth_math.h — the counter-based observation generator of BASELINE configs 3 and 4, written
 * once for the host (inputs/synth_host.cpp, g++ -ffp-contract=off) and the device
 * (paper_2603_25691_b200/csrc/k_synth.cu) so both produce the SAME bits.
 *
 * Draw l of stream s:   u64(l, s) = splitmix64(seed ^ splitmix64(l * 0x9E3779B97F4A7C15 + s))
 *   uniform index in [0, n):  (u64 >> 32) * n >> 32
 *   Zipf mode:                smallest i with cdf[i] > (u64 >> 11) * 2^-53, cdf built on the host
 *   value:                    sum_j prod_m A_m(i_m, j) + noise_std * N(0,1)
 * N(0,1) is Box-Muller, sqrt(-2 log f1) cos(2 pi f2), with log and cos evaluated by the
 * polynomials below: only +, *, / and sqrt, every operation explicitly rounded (no FMA
 * contraction on either side), so the host and the device agree bit for bit (tested:
 * tests/test_inputs.py on the host, tests/test_gpu_synth.py against the device).
 *
 * Test / benchmark input generation only: not part of the solver path.
 */
#ifndef CPHIFI_SYNTH_MATH_H
#define CPHIFI_SYNTH_MATH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define SYN_HD __host__ __device__ __forceinline__
#else
#define SYN_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define SYN_MUL(a, b) __dmul_rn((a), (b))
#define SYN_ADD(a, b) __dadd_rn((a), (b))
#define SYN_DIV(a, b) __ddiv_rn((a), (b))
#define SYN_SQRT(a) __dsqrt_rn(a)
#else
#include <math.h>
#define SYN_MUL(a, b) ((a) * (b))
#define SYN_ADD(a, b) ((a) + (b))
#define SYN_DIV(a, b) ((a) / (b))
#define SYN_SQRT(a) sqrt(a)
#endif

SYN_HD uint64_t syn_splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

SYN_HD uint64_t syn_draw(uint64_t seed, uint64_t l, uint64_t s) {
    return syn_splitmix64(seed ^ syn_splitmix64(l * 0x9E3779B97F4A7C15ull + s));
}

SYN_HD int64_t syn_uniform_index(uint64_t u, int64_t n) { return (int64_t)(((u >> 32) * (uint64_t)n) >> 32); }

SYN_HD double syn_unit(uint64_t u) { return (double)(u >> 11) * 0x1.0p-53; }  /* [0, 1) */

SYN_HD int64_t syn_zipf_index(uint64_t u, const double* cdf, int64_t n) {
    const double v = syn_unit(u);
    int64_t lo = 0, hi = n - 1;  /* smallest i with cdf[i] > v */
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cdf[mid] > v) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

/* x = m 2^e with m in [1, 2) from the bits (x normal and positive; exact) */
SYN_HD double syn_log(double x) {
    union {
        double d;
        uint64_t u;
    } b;
    b.d = x;
    int e = (int)((b.u >> 52) & 0x7ff) - 1023;
    b.u = (b.u & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
    double m = b.d;
    if (m > 1.4142135623730951) {  /* m in [sqrt2/2, sqrt2): |t| <= 0.1716 */
        m = SYN_MUL(m, 0.5);
        e += 1;
    }
    const double t = SYN_DIV(SYN_ADD(m, -1.0), SYN_ADD(m, 1.0));
    const double t2 = SYN_MUL(t, t);
    /* log m = 2 atanh t = 2 (t + t^3/3 + ... + t^23/23), truncation < 1e-19 */
    double s = 1.0 / 23.0;
    s = SYN_ADD(SYN_MUL(s, t2), 1.0 / 21.0);
    s = SYN_ADD(SYN_MUL(s, t2), 1.0 / 19.0);
    s = SYN_ADD(SYN_MUL(s, t2), 1.0 / 17.0);
    s = SYN_ADD(SYN_MUL(s, t2), 1.0 / 15.0);
    s = SYN_ADD(SYN_MUL(s, t2), 1.0 / 13.0);
    s = SYN_ADD(SYN_MUL(s, t2), 1.0 / 11.0);
    s = SYN_ADD(SYN_MUL(s, t2), 1.0 / 9.0);
    s = SYN_ADD(SYN_MUL(s, t2), 1.0 / 7.0);
    s = SYN_ADD(SYN_MUL(s, t2), 1.0 / 5.0);
    s = SYN_ADD(SYN_MUL(s, t2), 1.0 / 3.0);
    s = SYN_ADD(SYN_MUL(s, t2), 1.0);
    const double lm = SYN_MUL(SYN_MUL(2.0, t), s);
    const double de = (double)e;
    return SYN_ADD(SYN_MUL(de, 0.6931471803691238), SYN_ADD(SYN_MUL(de, 1.9082149292705877e-10), lm));
}

/* sin / cos of a in [0, pi/4] by their Taylor series (truncation < 1e-20) */
SYN_HD double syn_sin_small(double a) {
    /* a (1 - a^2/3! + a^4/5! - ...), Horner in -a^2 */
    const double a2 = SYN_MUL(a, a);
    double s = 1.0 / 121645100408832000.0;           /* 1/19! */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 355687428096000.0);  /* 1/17! */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 1307674368000.0);    /* 1/15! */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 6227020800.0);       /* 1/13! */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 39916800.0);         /* 1/11! */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 362880.0);           /* 1/9!  */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 5040.0);             /* 1/7!  */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 120.0);              /* 1/5!  */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 6.0);                /* 1/3!  */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0);
    return SYN_MUL(a, s);
}
SYN_HD double syn_cos_small(double a) {
    const double a2 = SYN_MUL(a, a);
    double s = 1.0 / 20922789888000.0;                      /* 1/16! */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 87178291200.0);      /* 1/14! */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 479001600.0);        /* 1/12! */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 3628800.0);          /* 1/10! */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 40320.0);            /* 1/8!  */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 720.0);              /* 1/6!  */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 24.0);               /* 1/4!  */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0 / 2.0);                /* 1/2!  */
    s = SYN_ADD(SYN_MUL(s, -a2), 1.0);
    return s;
}

/* cos(2 pi f), f in [0, 1): quadrant k = floor(4 f) and g = 4 f - k are exact */
SYN_HD double syn_cos2pi(double f) {
    const double f4 = SYN_MUL(f, 4.0);
    const int k = (int)f4;
    const double g = SYN_ADD(f4, -(double)k);  /* [0, 1): angle (pi/2) g in the quadrant */
    const double hp = 1.5707963267948966;      /* pi/2 */
    double c, s;                                /* cos / sin of (pi/2) g */
    if (g <= 0.5) {
        const double a = SYN_MUL(hp, g);
        c = syn_cos_small(a);
        s = syn_sin_small(a);
    } else {
        const double a = SYN_MUL(hp, SYN_ADD(1.0, -g));  /* 1 - g exact */
        c = syn_sin_small(a);
        s = syn_cos_small(a);
    }
    switch (k & 3) {
        case 0: return c;
        case 1: return -s;
        case 2: return -c;
        default: return s;
    }
}

/* Box-Muller from draws 64 and 65 of observation l */
SYN_HD double syn_normal(uint64_t seed, uint64_t l) {
    const uint64_t u1 = syn_draw(seed, l, 64), u2 = syn_draw(seed, l, 65);
    const double f1 = SYN_MUL(SYN_ADD((double)(u1 >> 11), 1.0), 0x1.0p-53);  /* (0, 1] */
    const double f2 = syn_unit(u2);
    return SYN_MUL(SYN_SQRT(SYN_MUL(-2.0, syn_log(f1))), syn_cos2pi(f2));
}

#endif /* CPHIFI_SYNTH_MATH_H */
