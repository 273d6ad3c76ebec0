// fastmath.cuh — branch-free table-driven fp64 log2 / exp2 for the BOCD cell loop.
//
// The recursion runs in base-2 log units (bocd_kernel.cuh), so the only
// transcendentals on the hot path are
//   fast_log2(b) for b = beta' > 0 (the NIG scale), and
//   fast_exp2(d) for d = lp - M <= ~0 (the log-sum-exp terms; d may be -inf).
// libdevice's log / exp spend 30 / 18 FP64-pipe instructions plus ~40 integer,
// uniform-move and branch instructions per call and split every call into its
// own control-flow region; these spend 9 FP64 instructions each, no branches.
//
// log2: b = 2^k z, z in [0.70703125, 1.4140625) (integer split of the bit
//       pattern); z lies in one of 256 sub-intervals i (width 1/512 below 1, 1/256
//       above) with precomputed invc_i ~ 1/c_i and l_i = -log2(invc_i) (long double
//       on the host); r = z invc_i - 1 is one FMA (exact product, one rounding),
//       |r| < 0.00196, log2 b = k + l_i + log2(1 + r),  log2(1 + r) = r P(r), P the
//       degree-4 Chebyshev interpolant of log1p(r)/(r ln 2) on |r| <= 0.001954
//       (max |error| of r P(r) 8.4e-19, 50-digit mpmath).
//       8 FP64 + ~7 integer ops.  Valid for 2^-1000 < b < 2^1000 (the 2^-k
//       scaling is folded into invc_i).
// exp2: d clamped to >= -1021 on the integer pipe (2^-1021 is irrelevant next to
//       the max term 1), d = (64 k + j)/64 + r exactly, |r| <= 1/128,
//       2^d = 2^k T_j (1 + q(r)), T_j = 2^(j/64) from a 64-entry table, q the
//       degree-5 Taylor polynomial of 2^r - 1 (truncation < 4e-17).  9 FP64 ops.
//       The table stores T'_j = T_j with (j << 14) subtracted from its high word, so
//       the high word of 2^k T_j is ONE integer multiply-add of the rounded argument
//       n = 64 k + j: n * 2^14 + hi(T'_j) = (k << 20) + hi(T_j)  (mod 2^32).
// Both tables live in shared memory.  Accuracy is tested against numpy/mpmath
// through the falcon_bocd_debug_fastmath hook (tests/test_gpu_fastmath.py).
#pragma once

#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

namespace fbocd {

constexpr int kLogTab = 256;
constexpr int kExpTab = 64;
constexpr double LN2 = 0.6931471805599453;
constexpr double INV_LN2 = 1.4426950408889634;

struct FastMathTables {
    double2 logtab[kLogTab];  // {invc_i, -log2(invc_i)}
    double exptab[kExpTab];   // 2^(j/64), high word minus (j << 14) (see exp2 above)
};

// z-interval of index i: i < 150 -> [c0 + i/512, +1/512), else [1 + (i-150)/256, +1/256)
inline void fill_fastmath_tables(FastMathTables* t) {
    const long double c0 = 0.70703125L;
    for (int i = 0; i < kLogTab; ++i) {
        long double lo, w;
        if (i < 150) {
            lo = c0 + (long double)i / 512.0L;
            w = 1.0L / 512.0L;
        } else {
            lo = 1.0L + (long double)(i - 150) / 256.0L;
            w = 1.0L / 256.0L;
        }
        const long double c = lo + 0.5L * w;
        const double invc = (double)(1.0L / c);
        t->logtab[i].x = invc;
        t->logtab[i].y = (double)(-log2l((long double)invc));
    }
    for (int j = 0; j < kExpTab; ++j) {
        const double v = (double)exp2l((long double)j / 64.0L);
        uint64_t b;
        static_assert(sizeof(b) == sizeof(v), "double is 64-bit");
        std::memcpy(&b, &v, sizeof(b));
        b -= uint64_t(uint32_t(j) << 14) << 32;  // pre-compensate the index bits (hi word)
        std::memcpy(&t->exptab[j], &b, sizeof(b));
    }
}

// The tables live in DYNAMIC shared memory at a 2048-B aligned address fmb (logtab at
// fmb, exptab at fmb + 4096); a lookup address is (index bits) + base (the BOCD kernel
// uses the compile-time base as an LDS immediate).  A kernel reserves kFmSmemBytes at the
// start of its dynamic shared memory (alignment slack included) and calls fm_setup once
// (then a CTA barrier).
constexpr unsigned kFmSmemBytes = 2048u + unsigned(sizeof(FastMathTables));

// Polynomial / conversion constants in constant memory, uploaded at handle creation
// (falcon_bocd_create -> upload_fastmath_constants): not known to the compiler, so DFMA /
// DADD read them as constant-bank operands instead of re-materialising 64-bit immediates
// in registers every step.
static __constant__ double c_fm[16];
// Leading (highest-degree) coefficients rounded to 20 mantissa bits, so that DFMA takes
// them as 32-bit immediates (no register or uniform-register operand): the rounding
// (relative 7e-8) is weighted by r^6 < 5e-15 (log2) and r^5 < 3e-11 (exp2), i.e. below
// 1e-20 absolute.
constexpr double kLog2C0 = 0.2885398864746094;    // 0x3fd2777000000000 ~ c_fm[0]
constexpr double kExp2C0 = 0.0013333559036254883;  // 0x3f55d88000000000 ~ c_fm[8]
static const double kFastMathConstants[16] = {
    0.2885399918194671,    -0.36067490780407263, 0.48089834696204886,  -0.7213475204433863,  // log2 P (r^4 .. r^1)
    1.4426950408889634,    0.0,                  4503599627371520.0,   6755399441055744.0,   // r^0, -, 2^52+1024, 1.5*2^52
    0.0013333558146428443, 0.009618129107628477, 0.05550410866482158,  0.24022650695910072,  // exp2 poly
    0.6931471805599453,    64.0,                 -0.015625,            0.0};

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// Copies the tables to the first 2048-B aligned address of dyn (a dynamic shared-memory
// region of kFmSmemBytes) and returns that address.
__device__ __forceinline__ unsigned fm_setup(unsigned char* dyn, const FastMathTables* __restrict__ src) {
    const unsigned b = smem_addr(dyn);
    const unsigned fmb = (b + 2047u) & ~2047u;
    const double* s = reinterpret_cast<const double*>(src);
    double* d = reinterpret_cast<double*>(dyn + (fmb - b));
    for (int k = threadIdx.x; k < int(sizeof(FastMathTables) / 8); k += blockDim.x) d[k] = s[k];
    return fmb;
}

__device__ __forceinline__ double2 lds_v2f64(unsigned a) {
    double2 v;
    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ double fast_log2(double x, unsigned fmb) {
    const unsigned tb = unsigned(__double2hiint(x)) + 0x00196000u;  // (hi - 0x3FE6A000) + (1024 << 20)
    // entry (tb >> 12) & 255 (top 8 mantissa bits of ix - OFF), as a byte offset
    const double2 t = lds_v2f64(((tb >> 8) & 0xFF0u) + fmb);
    // r = z * invc - 1 with z = x / 2^k: the exact power-of-two scaling is folded into invc
    const double invs =
        __hiloint2double(__double2hiint(t.x) + 0x40000000 - int(tb & 0xFFF00000u), __double2loint(t.x));
    const double r = fma(x, invs, -1.0);
    // k + l_i first (off the polynomial's dependency chain; the BOCD cell loop evaluates
    // the same expression stage by stage and must agree bit for bit)
    const double kt = (__hiloint2double(0x43300000, int(tb >> 20)) - c_fm[6]) + t.y;  // k (2^52 + 1024 bias)
    double p = fma(r, kLog2C0, c_fm[1]);
    p = fma(p, r, c_fm[2]);
    p = fma(p, r, c_fm[3]);
    p = fma(p, r, c_fm[4]);
    return fma(r, p, kt);
}

__device__ __forceinline__ double fast_exp2(double x, unsigned fmb) {
    // clamp x >= -1021 on the integer pipe: only the high word is clamped (a clamped
    // argument keeps stray low mantissa bits: -1021 - 2^-33 at most, irrelevant)
    const int xh = int(min(unsigned(__double2hiint(x)), 0xC08FE800u));  // -inf / NaN patterns too
    const double xc = __hiloint2double(xh, __double2loint(x));
    const double zf = fma(xc, c_fm[13], c_fm[7]);  // round(64 x) in the low word (1.5 * 2^52 shift)
    const unsigned ki = unsigned(__double2loint(zf));
    const double kd = zf - c_fm[7];
    const double r = fma(kd, c_fm[14], xc);  // exact: |r| <= 1/128
    double p = fma(r, kExp2C0, c_fm[9]);
    p = fma(p, r, c_fm[10]);
    p = fma(p, r, c_fm[11]);
    p = fma(p, r, c_fm[12]);
    const double q = p * r;
    const double T = lds_f64(((ki << 3) & 0x1F8u) + (fmb + 4096u));
    int th;  // high word of T_j * 2^(ki >> 6) = ki * 2^14 + hi(T'_j): one IMAD
    asm("mad.lo.s32 %0, %1, 16384, %2;" : "=r"(th) : "r"(ki), "r"(__double2hiint(T)));
    const double Ts = __hiloint2double(th, __double2loint(T));
    return fma(Ts, q, Ts);
}

// 1/x to ~1 ulp for positive normal x: MUFU seed + one Newton step (no IEEE division path).
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

}  // namespace fbocd
