// rsim_log.h -- glibc 2.39's double log, restated operation by operation (C and CUDA).
//
// The reference's synthetic generator takes its arrival gaps from random.expovariate, i.e.
// -log(1.0 - random()) / rate (trace.py:231,236; CPython Lib/random.py:599-613), and
// CPython's math.log is the C library's. That log (glibc sysdeps/ieee754/dbl-64/e_log.c, the
// Arm optimized-routines table log; x86-64 libm runs its FMA build on FMA+AVX2 CPUs) is not
// correctly rounded, so the device generator evaluates the same formula: the same table
// (rsim_glibc_log.h, extracted from the system libm), the same operation order and the same
// fused multiply-adds as the FMA build's machine code. Inputs here are 1 - k * 2^-53 in
// (0, 1], all normal, so the subnormal / negative / inf / nan branches are not restated;
// glibc_log() returns NaN for them and the generator reports an error.
//
// Host builds must not contract a*b+c themselves (gcc -ffp-contract=off); device builds use
// the _rn intrinsics, which nvcc never contracts.
#pragma once
#include <stdint.h>
#include <string.h>
#include "rsim_glibc_log.h"

#ifdef __CUDACC__
#define RSIM_LOG_HD __host__ __device__ __forceinline__
#else
#define RSIM_LOG_HD static inline
#include <math.h>
#endif

#if defined(__CUDA_ARCH__)
#define RL_FMA(a, b, c) __fma_rn(a, b, c)
#define RL_ADD(a, b) __dadd_rn(a, b)
#define RL_SUB(a, b) __dsub_rn(a, b)
#define RL_MUL(a, b) __dmul_rn(a, b)
#define RL_BITS(x) ((uint64_t)__double_as_longlong(x))
#define RL_DBL(u) __longlong_as_double((long long)(u))
#else
#define RL_FMA(a, b, c) fma(a, b, c)
#define RL_ADD(a, b) ((a) + (b))
#define RL_SUB(a, b) ((a) - (b))
#define RL_MUL(a, b) ((a) * (b))
RSIM_LOG_HD uint64_t rl_bits_(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
RSIM_LOG_HD double rl_dbl_(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
#define RL_BITS(x) rl_bits_(x)
#define RL_DBL(u) rl_dbl_(u)
#endif

// tab: the 256 doubles of RSIM_LOG_TAB_INIT ({invc, logc} x 128).
RSIM_LOG_HD double glibc_log(double x, const double *tab) {
    const uint64_t ix = RL_BITS(x);
    if (ix - 0x3fee000000000000ull <= 0x308ffffffffffull) {   // |x - 1| < ~0x1p-4
        if (ix == 0x3ff0000000000000ull) return 0.0;
        const double r = RL_SUB(x, 1.0);
        const double r2 = RL_MUL(r, r), r3 = RL_MUL(r, r2);
        double p2 = RL_FMA(r, RSIM_LOG_B2, RSIM_LOG_B1);
        double p5 = RL_FMA(r, RSIM_LOG_B5, RSIM_LOG_B4);
        double p8 = RL_FMA(r, RSIM_LOG_B8, RSIM_LOG_B7);
        p2 = RL_FMA(r2, RSIM_LOG_B3, p2);
        p5 = RL_FMA(r2, RSIM_LOG_B6, p5);
        double p = RL_FMA(r2, RSIM_LOG_B9, p8);
        p = RL_FMA(r3, RSIM_LOG_B10, p);
        p = RL_FMA(p, r3, p5);
        p = RL_FMA(p, r3, p2);
        const double t = RL_FMA(r, 0x1p27, r);                // w = r * 2^27; rhi = r + w - w
        const double rhi = RL_FMA(-0x1p27, r, t);
        const double rlo = RL_SUB(r, rhi);
        const double rr = RL_MUL(rhi, rhi);
        const double hi = RL_FMA(rr, RSIM_LOG_B0, r);         // hi = r + rhi^2 * B0
        double lo = RL_FMA(rr, RSIM_LOG_B0, RL_SUB(r, hi));
        lo = RL_FMA(RL_MUL(RSIM_LOG_B0, rlo), RL_ADD(r, rhi), lo);
        return RL_ADD(hi, RL_FMA(p, r3, lo));
    }
    if (((ix >> 48) - 0x0010u) >= 0x7fe0u) return RL_DBL(0x7ff8000000000000ull);  // not restated
    const uint64_t tmp = ix - 0x3fe6000000000000ull;
    const int i = (int)((tmp >> 45) & 127);
    const double kd = (double)(int)((int64_t)tmp >> 52);
    const double z = RL_DBL(ix - (tmp & 0xfff0000000000000ull));
    const double invc = tab[2 * i], logc = tab[2 * i + 1];
    const double w = RL_FMA(kd, RSIM_LOG_LN2HI, logc);
    const double r = RL_FMA(z, invc, -1.0);
    const double q = RL_FMA(r, RSIM_LOG_A2, RSIM_LOG_A1);
    const double hi = RL_ADD(r, w);
    const double r2 = RL_MUL(r, r);
    double lo = RL_ADD(RL_SUB(w, hi), r);
    lo = RL_FMA(kd, RSIM_LOG_LN2LO, lo);
    const double r3 = RL_MUL(r, r2);
    double p = RL_FMA(r, RSIM_LOG_A4, RSIM_LOG_A3);
    lo = RL_FMA(r2, RSIM_LOG_A0, lo);
    p = RL_FMA(p, r2, q);
    return RL_ADD(RL_FMA(r3, p, lo), hi);
}
