// cellmath.cuh — the BOCD cell loop's log2 / exp2.
//
// The cell loop needs, per run-length cell and step, lg beta' and 2^(l - Dc)
// (bocd_kernel.cuh).  In the log-joint form an error in either enters only the
// current step's q' (it is not carried forward by a multiplicative recursion), so
// polynomial degree is traded for table size against the 1e-9 parity budget
// (BASELINE.json north_star; the measured errors stay orders of magnitude below it):
//   cell_log2<LB>: b = 2^k z, z in [1, 2) split into 2^LB intervals of width 2^-LB by the
//              top LB mantissa bits; {invc_i, l_i = -log2(invc_i)} from the table;
//              r = z invc_i - 1 (one FMA, |r| <= 2^-(LB+1)); log2 b = k + l_i + r P(r),
//              P the degree-3 Chebyshev interpolant of log2(1+r)/r: max |error| of r P(r)
//              1.0e-15 (LB = 8), 9.9e-19 (LB = 10).  7 FP64 ops.
//   cell_exp2: d = (256 k + j)/256 + r exactly (|r| <= 2^-9), 2^d = 2^k T_j (1 + r Q(r)),
//              T_j = 2^(j/256) from a 256-entry table, Q the degree-3 Chebyshev interpolant
//              of (2^r - 1)/r (max |error| of r Q(r) 4.8e-18).  8 FP64 ops.  A degree-2 Q
//              (minimax of the relative error, 2.4e-14; c_cell[21..22] + kCellExpQ2c) serves
//              the FULL kernels' slots >= 1, whose masses are never carried forward
//              (bocd_kernel.cuh, EXP3).
// The coefficients were fitted with 60-digit mpmath (Chebyshev nodes on the reduced
// interval) and rounded to double; the leading ones are DFMA immediates.  Tables are
// computed on the host in long double.  Accuracy: tests/test_gpu_fastmath.py.
//
// Shared-memory layout inside the BOCD kernel's dynamic window (absolute shared addresses,
// LDS immediates): the exp2 table replicated EC times (entry j of copy c at kCellExpBase +
// 8 (EC j + c); lane L reads copy L mod EC, so EC = 16 makes a warp-wide lookup
// conflict-free), then the log2 table (2^LB entries of 16 B).
#pragma once

#include <cstdint>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>

namespace fbocd {

// log2 table bits: 8 for the R <= 1024 FULL kernels (speed), 10 for the others: there alpha
// reaches 1024-2048 and the log's error, carried along the MERGE bucket's chain of merged
// masses, would approach the parity budget (measured 6.2e-10 at R = 2048 with LB = 8).
__host__ __device__ constexpr int cell_logbits(bool full, int r_full) { return (full && r_full <= 1024) ? 8 : 10; }
constexpr int kCellEB = 8;  // exp2 table bits (degree-4 / degree-3 fits; 9 bits measured slower)
constexpr int kCellExpTab = 1 << kCellEB;
constexpr double kCellExpScale = double(kCellExpTab);          // the rounding grid 2^-EB
constexpr unsigned kCellExpLo = 0x80000000u - 1021u * kCellExpTab;  // 2^-1021: floor / dead

struct CellTables {
    double exptab[kCellExpTab];  // 2^(j/2^EB), high word minus (j << (20 - EB))
    double2 log8[256];           // {invc_i, -log2(invc_i)}, z in [1 + i/2^LB, 1 + (i+1)/2^LB)
    double2 log10[1024];
    double2 log8h[256];          // {invc_i, -log2(invc_i) / 2}: the FULL kernels' half-log (below)
    double2 log10h[1024];
};

inline void fill_cell_tables(CellTables* t) {
    for (int j = 0; j < kCellExpTab; ++j) {
        const double v = (double)exp2l((long double)j / (long double)kCellExpTab);
        uint64_t b;
        std::memcpy(&b, &v, sizeof(b));
        b -= uint64_t(uint32_t(j) << (20 - kCellEB)) << 32;  // n 2^(20-EB) + hi(T'_j) = (k << 20) + hi(T_j)
        std::memcpy(&t->exptab[j], &b, sizeof(b));
    }
    auto fill_log = [](double2* tab, int n, long double scale) {
        for (int i = 0; i < n; ++i) {
            const long double c = 1.0L + ((long double)i + 0.5L) / (long double)n;
            const double invc = (double)(1.0L / c);
            tab[i].x = invc;
            tab[i].y = (double)(-log2l((long double)invc) * scale);  // scale 1/2: exactly half
        }
    };
    fill_log(t->log8, 256, 1.0L);
    fill_log(t->log10, 1024, 1.0L);
    fill_log(t->log8h, 256, 0.5L);
    fill_log(t->log10h, 1024, 0.5L);
}

// Polynomial coefficients (constant bank; uploaded with the fast-math constants): P0..P2 of
// the log for LB = 8, 9, 10 at 3 (LB - 8), Q0..Q2 of the exp at 9.
// 12..20: the log coefficients halved (exact), for the half-log lg(b)/2 of the FULL kernels.
static __constant__ double c_cell[23];
static const double kCellConstants[23] = {
    1.4426950408884385, -0.7213475204440444, 0.4808994476545776,   // LB = 8
    1.4426950408889305, -0.7213475204444544, 0.4808986221353932,   // LB = 9
    1.4426950408889614, -0.72134752044448, 0.4808984157560584,     // LB = 10
    // exp: Q0, Q1, Q2 (+ Q3 immediate; max error of r Q(r) 4.8e-18)
    0.6931471805599428, 0.24022650695910044, 0.05550411375117056,
    0.5 * 1.4426950408884385, 0.5 * -0.7213475204440444, 0.5 * 0.4808994476545776,
    0.5 * 1.4426950408889305, 0.5 * -0.7213475204444544, 0.5 * 0.4808986221353932,
    0.5 * 1.4426950408889614, 0.5 * -0.72134752044448, 0.5 * 0.4808984157560584,
    // 21, 22: exp Q0, Q1 of the degree-3 fit (+ kCellExpQ2c immediate; max error of
    // 1 + r Q(r) vs 2^r 2.4e-14 relative, |r| <= 2^-9), for the cells that feed no chain
    0.6931471805600506, 0.24022653734438304};
// leading coefficients rounded to 20 mantissa bits (DFMA immediates; the rounding is weighted
// by r^4 <= 2^-36, i.e. below 1e-18)
template <int LB>
constexpr double kCellLogP3 = LB == 8 ? -0.3606746196746826 : -0.3606739044189453;
template <int LB>
constexpr double kCellLogP3h = 0.5 * kCellLogP3<LB>;
constexpr double kCellExpQ3 = 0.009618133306503296;  // 0.009618129695226546 rounded
constexpr double kCellExpQ2c = 0.05550408363342285;  // 0.055504081729180456 rounded (degree 3)

constexpr unsigned kCellExpBase = 0x1A00u;
template <int EC>
__host__ __device__ constexpr unsigned cell_log_base() { return kCellExpBase + kCellExpTab * EC * 8u; }
template <int EC, int LB>
__host__ __device__ constexpr unsigned cell_tables_end() { return cell_log_base<EC>() + (16u << LB); }

// log2 table entry of b, tb = hi(b)
template <int EC, int LB>
__device__ __forceinline__ double2 cell_log_entry(unsigned tb) {
    double2 v;
    asm("ld.shared.v2.f64 {%0, %1}, [%2+%3];"
        : "=d"(v.x), "=d"(v.y)
        : "r"((tb >> (16 - LB)) & (((1u << LB) - 1u) << 4)), "n"(cell_log_base<EC>()));
    return v;
}

template <int EC, int LB>
__device__ __forceinline__ double cell_log2(double b) {
    const unsigned tb = unsigned(__double2hiint(b));
    const double2 t = cell_log_entry<EC, LB>(tb);
    const double invs = __hiloint2double(__double2hiint(t.x) + 0x3FF00000 - int(tb & 0x7FF00000u), __double2loint(t.x));
    const double r = fma(b, invs, -1.0);
    const double kt = __int2double_rn(int(tb >> 20) - 1023) + t.y;  // k + l_i (k exact)
    constexpr int o = 3 * (LB - 8);
    double p = fma(r, kCellLogP3<LB>, c_cell[o + 2]);
    p = fma(p, r, c_cell[o + 1]);
    p = fma(p, r, c_cell[o]);
    return fma(r, p, kt);
}

// Half-log lg(b)/2, bit-for-bit half of cell_log2 (every coefficient and table value is
// scaled by the exact factor 1/2, so each rounding is the scaled rounding).  The FULL kernels
// form alpha_r lg beta' as (2 alpha_r)(lg beta'/2) with 2 alpha_r an exactly converted integer
// (no alpha column in the per-r table); the product, and so every result, is unchanged.
// The shared-memory log table must hold the halved entries (log8h / log10h).
template <int EC, int LB>
__device__ __forceinline__ double cell_log2h(double b) {
    const unsigned tb = unsigned(__double2hiint(b));
    const double2 t = cell_log_entry<EC, LB>(tb);
    const double invs = __hiloint2double(__double2hiint(t.x) + 0x3FF00000 - int(tb & 0x7FF00000u), __double2loint(t.x));
    const double r = fma(b, invs, -1.0);
    const double kt = fma(__int2double_rn(int(tb >> 20) - 1023), 0.5, t.y);  // k/2 + l_i/2 (k exact)
    constexpr int o = 12 + 3 * (LB - 8);
    double p = fma(r, kCellLogP3h<LB>, c_cell[o + 2]);
    p = fma(p, r, c_cell[o + 1]);
    p = fma(p, r, c_cell[o]);
    return fma(r, p, kt);
}

// exp2 table entry for the rounded argument ki (low word of the 1.5 2^52 + 2^31 rounding);
// lbe = 8 (lane mod EC), EC = 4, 8 or 16
template <int EC>
__device__ __forceinline__ double cell_exp_entry(unsigned ki, unsigned lbe) {
    double v;
    constexpr int sh = EC == 16 ? 7 : EC == 8 ? 6 : EC == 4 ? 5 : 4;  // 3 + log2(EC)
    asm("ld.shared.f64 %0, [%1+%2];"
        : "=d"(v)
        : "r"(((ki << sh) & ((unsigned(kCellExpTab) - 1u) << sh)) | lbe), "n"(kCellExpBase));
    return v;
}

}  // namespace fbocd
