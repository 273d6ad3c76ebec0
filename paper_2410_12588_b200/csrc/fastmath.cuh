// fastmath.cuh — branch-free table-driven fp64 log and exp for the BOCD cell loop.
//
// libdevice's log / exp spend 30 / 18 FP64-pipe instructions plus ~40 integer,
// uniform-move and branch instructions per call and split every call into its
// own control-flow region (special-case branches), which stops ptxas from
// interleaving the 8 independent cells of a thread.  The cell loop only ever
// needs
//   fast_log(b) for b = beta' > 0 finite normal (the NIG scale), and
//   fast_exp(d) for d = lp - M <= ~0 (the log-sum-exp terms; d may be -inf),
// so both are written without special-case branches:
//
// log:  b = 2^k z, z in [0.70703125, 1.4140625) (integer split of the bit
//       pattern), z falls in one of 128 sub-intervals i with precomputed
//       invc_i ~ 1/c_i and logc_i = -log(invc_i) (long double on the host);
//       r = fma(z, invc_i, -1) is exact up to one rounding, |r| < 0.0040, and
//       log b = k ln2 + logc_i + log1p(r) with log1p(r) = r + r^2 P(r), P the
//       degree-4 Taylor tail (truncation < 2e-18).  12 FP64 + ~7 integer ops.
//       Valid for 2^-1000 < b < 2^1000 (the 2^-k scaling is folded into invc_i).
// exp:  d clamped to >= -708 on the integer pipe (exp < 4e-308 is irrelevant
//       next to the max term 1), d = (64 k + j) ln2/64 + r, |r| <= ln2/128,
//       exp d = 2^k T_j (1 + q(r)), T_j = 2^(j/64) from a 64-entry table,
//       q the degree-5 Taylor polynomial (truncation < 4e-17).  10 FP64 ops.
// Both tables live in shared memory (loaded once per CTA).  Accuracy is
// tested against mpmath in tests/test_gpu_fastmath.py (<= 2 ulp).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fbocd {

constexpr int kLogTab = 128;
constexpr int kExpTab = 64;

struct FastMathTables {
    double2 logtab[kLogTab];  // {invc_i, logc_i}
    double exptab[kExpTab];   // 2^(j/64)
};

// z-interval of index i (see fast_log): i < 75 -> [c0 + i/256, +1/256), else [1 + (i-75)/128, +1/128)
inline void fill_fastmath_tables(FastMathTables* t) {
    const long double c0 = 0.70703125L;
    for (int i = 0; i < kLogTab; ++i) {
        long double lo, w;
        if (i < 75) {
            lo = c0 + (long double)i / 256.0L;
            w = 1.0L / 256.0L;
        } else {
            lo = 1.0L + (long double)(i - 75) / 128.0L;
            w = 1.0L / 128.0L;
        }
        const long double c = lo + 0.5L * w;
        const double invc = (double)(1.0L / c);
        t->logtab[i].x = invc;
        t->logtab[i].y = (double)(-logl((long double)invc));
    }
    for (int j = 0; j < kExpTab; ++j) t->exptab[j] = (double)exp2l((long double)j / 64.0L);
}

// ln2 split: LN2_HI has 32 significant bits, so k * LN2_HI is exact for |k| < 2^21.
constexpr double LN2_HI = 6.93147180369123816490e-01;  // 0x3fe62e42fee00000
constexpr double LN2_LO = 1.90821492927058770002e-10;  // 0x3dea39ef35793c76

__device__ __forceinline__ double fast_log(double x, const double2* __restrict__ logtab) {
    const int hi = __double2hiint(x);
    const int tb = hi + 0x00196000;          // (hi - 0x3FE6A000) + (1024 << 20): biased k in bits 20..31
    const double2 t = logtab[(tb >> 13) & (kLogTab - 1)];  // top 7 mantissa bits of (ix - OFF)
    // r = z * invc - 1 with z = x / 2^k: the exact power-of-two scaling is folded into invc
    const double invs =
        __hiloint2double(__double2hiint(t.x) + 0x40000000 - (tb & 0xFFF00000), __double2loint(t.x));
    const double r = fma(x, invs, -1.0);
    const double kd = __hiloint2double(0x43300000, int(unsigned(tb) >> 20)) - 4503599627371520.0;  // 2^52+1024
    const double r2 = r * r;
    double p = fma(r, -1.0 / 6.0, 0.2);
    p = fma(p, r, -0.25);
    p = fma(p, r, 1.0 / 3.0);
    p = fma(p, r, -0.5);
    const double w = fma(kd, LN2_HI, t.y);  // exact product, one rounding
    const double q = fma(r2, p, kd * LN2_LO);
    return (w + r) + q;
}

// 1/x to ~1 ulp for positive normal x: MUFU seed + one Newton step (no IEEE division path).
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ double fast_exp(double x, const double* __restrict__ exptab) {
    // clamp x >= -708 (also maps -inf / NaN patterns) on the integer pipe
    int xh = __double2hiint(x);
    int xl = __double2loint(x);
    const bool clamp = static_cast<unsigned>(xh) > 0xC0862000u;  // |x| > 708 with x < 0
    xh = clamp ? 0xC0862000 : xh;
    xl = clamp ? 0 : xl;
    const double xc = __hiloint2double(xh, xl);
    constexpr double SHIFT = 6755399441055744.0;  // 1.5 * 2^52
    constexpr double INV_L = 92.33248261689365;   // 64 / ln2
    constexpr double L1 = LN2_HI / 64.0, L2 = LN2_LO / 64.0;
    const double zf = fma(xc, INV_L, SHIFT);
    const int ki = __double2loint(zf);
    const double kd = zf - SHIFT;
    double r = fma(kd, -L1, xc);
    r = fma(kd, -L2, r);
    double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    const double q = p * r;
    const double T = exptab[ki & (kExpTab - 1)];
    const int e = ki >> 6;
    const double Ts = __hiloint2double(__double2hiint(T) + e * 1048576, __double2loint(T));
    return fma(Ts, q, Ts);
}

}  // namespace fbocd
