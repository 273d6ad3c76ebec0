// bocd_kernel.cuh — resident batched BOCD kernel for sm_100a (fp64).
//
// One series group of NT threads owns one series; each thread owns J run-length
// cells.  The R cells of a series live in a RING indexed by position
// p = (segment start time) mod R (p = i + NT*j for thread i, register j): at
// global step t the cell at position p holds run length r = (t - p) mod R
// BEFORE x_t is absorbed, so growth r -> r+1 (App. A)
// moves no data, and the position that truncation at R recycles (r = R-1) is
// exactly the one that becomes the new change-point cell.  Per-r constants of
// the NIG marginal likelihood come from a shared-memory table indexed by r.
//
// LOG-JOINT representation.  A cell whose segment has absorbed n observations
// holds (mu_n, beta_n) and one number a: its joint mass Pr(r_t = n, x_{0..t})
// (up to the per-series normaliser) is
//     q = 2^(a + G_n - alpha_n lg beta_n - Dc_t)                         (lg = log2)
// where G_n + alpha0 lg beta0 - alpha_n lg beta_n is the log2 NIG marginal
// likelihood of the segment (G_n = lg[Gamma(alpha_n)/Gamma(alpha0)] + 1/2 lg(kappa0/kappa_n)
// - n/2 lg(2 pi) from a host table; kappa_n = kappa0 + n, alpha_n = alpha0 + n/2), a
// fixes the segment's prior mass when it was created, and Dc_t is a per-series
// integer frame.  The product of Student-t predictives of P:1345 telescopes into
// this ratio of marginals, so a step needs, per cell, the NIG update, ONE log2
// (lg beta') and ONE exp2; no per-cell multiply by the previous mass and no
// posterior row in shared memory.
//   Dc_t = Dc_{t-1} + N_t, N_t = K0_t + z_{t-1}: K0_t = round(l0_t), l0_t the prior
//          predictive of x_t (the change-point cell's density, computed for a whole
//          x tile at once), z_{t-1} = the binary exponent of Zd_{t-1}; so the cells of
//          step t are exponentiated against the reference 2^(Dc_t) and Z stays O(1).
//          Dc enters the exp2 range reduction as an exact integer shift of its
//          rounding constant (zero per-cell cost).  At every global step that is a
//          multiple of kRebase the frame is rebased (a -= Dc, Dc = 0): a fixed global
//          schedule, so results do not depend on how the data is split into calls.
// Per step and cell (r = the cell's run length before x_t; n = r + 1 after):
//   A1  NIG update            mu' = mu + d y_r,  beta' = beta + d (x - mu')/2   (d = x - mu,
//                             y_r = 1/(kappa_r+1): d (x - mu')/2 = kappa_r d^2 / (2(kappa_r+1)))
//   A2  log2 marginal         l = (a + G_n) - alpha_n lg beta'   (the Student-t predictive of
//                             P:1333/P:1345 is 2^(l - l_prev), implicit)
//   A3  joint                 q' = 2^(l - Dc_t)  (fast exp2, Dc_t in the rounding constant)
//   A4  evidence              Z = sum_r q'_r  (per-thread sums, xor butterfly, fixed-order
//                             cross-warp sum: deterministic);
//                             log Z_t = ln2 (N_t + lg Zd_t - lg Zd_{t-1}) + ln(1-H)
//   A5  normalisation         Zd = Z (MERGE) or Z - (1-H) q'_{R-1} (DROP); R_t(r+1) = (1-H) q'_r / Zd
//   A6  change point / MERGE  the recycled cell (r = R-1) becomes the new change-point cell:
//                             prior statistics, a = lg(H Z/(1-H)) + alpha0 lg beta0 + Dc_t
//                             (R_t(0) = H Z / Zd); MERGE: the cell reaching r = R-1 takes the
//                             truncated cell's mass, a = lg(q'_{R-2} + q'_{R-1}) - (G - alpha lg beta')
//                             + Dc_t;  DROP: q'_{R-1} is dropped
//   A7  decision, MAP         p_new = R_t(1)/(1-R_t(0)) = q'_0/Z (MERGE) or q'_0/(Z - q'_{R-1}) (DROP);
//                             r* = argmax over the growth slots (+ bucket), reduced every step when
//                             the caller asks for per-step MAP / MAPRESET events or theta < 1/2
//                             (EAGER); otherwise r* = 1 at every PROB event (p_new > theta >= 1/2
//                             puts more than half the growth mass in slot 1)
// mu, beta, a live in registers for the whole call; x is staged in double-buffered
// shared-memory tiles by 1-D TMA bulk copies (cp.async.bulk + mbarrier); state is
// spilled to HBM once per call.  The cell loop is written stage-major over groups of
// kG cells (every stage of a group before the next stage) so the dependent FP64
// chains of kG cells interleave.
#pragma once

#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "cellmath.cuh"
#include "fastmath.cuh"

namespace fbocd {

constexpr int kTile = 256;     // x steps per shared-memory tile (2 KB)
constexpr int kTileP = 64;     // persistent (streaming) kernels: calls of <= 64 steps
constexpr int kRebase = 256;   // generic kernels: global steps between frame rebases (ROT: every NT)
constexpr int kG = 2;  // cells per interleaved group (ILP; 1, 4 and 8 measured slower: 77.0, 74.1, 78.3 vs 73.8 ms)
// K0_t = round(l0_t) is clamped to +-kK0Max so that |N_t| < 2^14 and 256 Dc stays below 2^31
// (at most 512 steps between rebases)
constexpr double kK0Max = 8192.0;
// A cell's joint below 2^-1021 of the step reference is floored to [2^-1021, 2^-1019) by a
// two-sided integer clamp (no select per cell), and impossible cells (run lengths longer than
// the data seen) carry the finite offset kImpossible instead of -inf (read_posterior still
// reports -inf for them).
constexpr double kImpossible = -1048576.0;  // -2^20: 256 |l - Dc| stays below 2^31
// A MERGE bucket mass below this (floored dead / impossible cells only) is an exact 0, so run
// lengths longer than the data seen stay impossible.
constexpr double kDeadMass = 0x1p-1015;
__device__ __forceinline__ double bucket_mass(double qA, double qB) {
    const double v = qA + qB;
    return v < kDeadMass ? 0.0 : v;
}

struct SeriesScalars {  // per-series state carried between calls (HBM), 48 B
    double mu0, beta0;  // prior (set from x_0 when prior_first_obs)
    double zd_prev;     // Zd_{t-1}: R_{t-1}(r) = q_r (1-H) / Zd_{t-1}  (1-H before the first step)
    int32_t map_prev;   // r*_{t-1}
    int32_t ev_count;   // events appended since the last drain (may exceed capacity)
    int32_t flags;      // bit0: non-finite observation seen; bit1: bad prior; bit2: smem layout
    int32_t dc;         // Dc_{t-1}: integer frame of the cells' a values since the last rebase
    double pad2;
};

struct EventRec {  // 32 B, series id implicit
    int64_t t;
    int64_t cp_index;
    uint32_t flags;
    uint32_t pad;
    double p_new;
};

struct KParams {
    int R;
    int64_t S;
    double H, omH, hr, theta, alpha0, prior_cov;  // omH = 1-H, hr = H/(1-H)
    double ln_omH;                                // log(1-H)
    double c_bucket;                              // c_{R-1}/ln2 (MERGE bucket, FULL)
    double al2_bucket;                            // 2 alpha_{R-1}
    int a2p1;                                     // floor(2 alpha0) + 1 (FULL kernels)
    double f2;                                    // 2 alpha0 - floor(2 alpha0) (FULL kernels, MODE bit 1)
    int mode;                                     // 0 MERGE, 1 DROP
    int prior_first_obs;
    uint32_t ev_mask;
    int ev_cap;
    const double2* tab_ca;     // [R] row r: {G_{r+1}, alpha_{r+1}}
    const double* tab_y;       // [R] y_r = 1/(kappa_r+1)
    const FastMathTables* fm;  // log2 / exp2 tables (per-step scalars)
    const CellTables* ct;      // the cell loop's log2 / exp2 tables (cellmath.cuh)
    double* st_mu;             // [S][R] position order
    double* st_beta;
    double* st_a;
    double* st_w;              // [S][NT] pending slot-0 weights (FULL kernels)
    SeriesScalars* scal;  // [S]
    EventRec* ev;         // [S][ev_cap]
    unsigned* err;        // sticky device error bits
    const double* x;      // [S][ld] chunk, column 0 = global step t0
    int64_t ld;
    int T;
    int64_t t0;
    int32_t* out_map;  // [S][ld_o] or null
    double* out_pnew;
    double* out_logz;
    int64_t ld_o;
    int tma_ok;  // x base 16-B aligned and ld even
};

// per-series partial sums of a step: one per warp
__host__ __device__ constexpr int n_partials(int nt) { return nt / 32 > 0 ? nt / 32 : 1; }

template <int NT, int TILE = kTile>
struct __align__(16) GroupSmem {
    double xbuf[2][TILE];
    int kbuf[2][TILE];  // K0_t = round(l0_t) of the tile's steps
    // red2 / red1 / spec are double-buffered by step parity: a warp that runs ahead into
    // step t+1 cannot overwrite what a slower warp still reads after barrier t
    double red2[2][n_partials(NT)];
    unsigned long long red1[2][n_partials(NT)];  // EAGER argmax keys
    // generic kernels: q' of the cells r = R-2, R-1, 0 and G - alpha lg beta' of r = R-2;
    // ROT kernels: e0 / l0 hold q' / lg beta' of every thread's slot 0, entry NT = slot 1 of
    // thread 0, entry NT+1 (e0) = slot J-1 of thread NT-1 (the cells the tail needs)
    double spec[2][4];
    double e0[2][NT + 2];
    double l0[2][NT + 1];
    double mu0, beta0, L0, zd_prev;  // zd_prev: kept current by thread 0 every step
    double lzd_prev;                 // lg Zd_{t-1} (log-evidence output, thread 0)
    double aprior;                   // alpha0 lg beta0
    int map_prev, ev_count, flags, dc0;  // dc0: Dc_{t-1} at the start of the call
    unsigned long long mbar[2];  // x tiles
    unsigned long long mbar_st;  // prefetched state of the next unit (PREF kernels)
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// barrier of one series group (NT threads)
template <int NT>
__device__ __forceinline__ void group_sync(int g) {
    if constexpr (NT == 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(NT) : "memory");
    }
}

// Fixed-order pairwise sum of the W per-warp partials (deterministic)
template <int W>
__device__ __forceinline__ double tree_sum(const double* p) {
    if constexpr (W == 1) {
        return p[0];
    } else {
        return tree_sum<W / 2>(p) + tree_sum<W / 2>(p + W / 2);
    }
}

// The sum of the W per-warp partials, known to every lane: for W >= 16 each lane loads one
// partial (lane mod W) and an xor butterfly adds them (fixed order: deterministic; one shared
// load instead of W/2 16-byte loads and W - 1 serial-ish adds); smaller W: tree_sum.
template <int W>
__device__ __forceinline__ double partials_sum(const double* p, int lane) {
    if constexpr (W >= 16) {
        double v = p[lane & (W - 1)];
#pragma unroll
        for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    } else {
        return tree_sum<W>(p);
    }
}

// Argmax key of a non-negative double q at run length r: the bit pattern of q is
// order-preserving; its low 12 mantissa bits are replaced by (4095 - r) so the max
// key is the max q and, among (near-)ties (< 2^-40 relative), the smallest r.
__device__ __forceinline__ unsigned long long argmax_key(double q, int r) {
    return (static_cast<unsigned long long>(__double_as_longlong(q)) & ~0xFFFull) | unsigned(0xFFF - r);
}
__device__ __forceinline__ int key_r(unsigned long long k) { return int(0xFFF - (k & 0xFFF)); }
__device__ __forceinline__ double key_val(unsigned long long k) {
    return __longlong_as_double(static_cast<long long>(k & ~0xFFFull));
}

// 64-bit max over the warp with two 32-bit REDUX passes
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long k) {
    const unsigned hi = unsigned(k >> 32);
    const unsigned hmax = __reduce_max_sync(0xffffffffu, hi);
    const unsigned lmax = __reduce_max_sync(0xffffffffu, hi == hmax ? unsigned(k) : 0u);
    return (static_cast<unsigned long long>(hmax) << 32) | lmax;
}

template <int NT, int TILE>
__device__ __forceinline__ void issue_tile_tma(GroupSmem<NT, TILE>& gs, const double* xrow, int k, int T) {
    const int base = k * TILE;
    const int n = min(TILE, T - base);
    fence_proxy_async();
    mbar_arrive_expect_tx(&gs.mbar[k & 1], unsigned(n) * 8u);
    tma_load_1d(gs.xbuf[k & 1], xrow + base, unsigned(n) * 8u, &gs.mbar[k & 1]);
}

template <int TILE>
__device__ __forceinline__ bool tile_tma_ok(const KParams& P, int k) {
    const int n = min(TILE, P.T - k * TILE);
    return P.tma_ok && ((n & 1) == 0);
}

// Shared memory of one CTA: tables, then per group: GroupSmem (+ PREF buffer).
// TAB2: the per-r tables are stored twice (entries r and r+R) so the ring index
// (t - p) mod R becomes (t - p + R) with no masking and compile-time offsets per cell.
// per group: GroupSmem and (PREF) the prefetch buffer [mu R][beta R][a R][scalars]
template <int NT, bool PREF>
__host__ __device__ constexpr size_t group_bytes(int R) {
    return sizeof(GroupSmem<NT, PREF ? kTileP : kTile>) +
           (PREF ? ((3 * size_t(R) * sizeof(double) + sizeof(SeriesScalars) + 15) & ~size_t(15)) : 0);
}
// bytes of the per-r tables for `entries` table rows: generic kernels {G_{r+1}, alpha_{r+1}}
// and y_r (24 B per row); FULL kernels {G_{r+1}, y_r} (16 B per row: alpha is converted from
// the integer 2 alpha0 + r + 1)
__host__ __device__ constexpr size_t table_bytes(int entries, bool full) {
    return (size_t(entries) * (full ? sizeof(double2) : sizeof(double2) + sizeof(double)) + 15) & ~size_t(15);
}

// Writes v into register slot j of a (a runtime slot index: a plain jump table).
template <int J>
__device__ __forceinline__ void set_slot(double (&a)[J], int j, double v) {
#define FBOCD_SET1(k)          \
    case k:                    \
        if constexpr (J > k) a[k] = v; \
        break;
    switch (j) { FBOCD_SET1(0) FBOCD_SET1(1) FBOCD_SET1(2) FBOCD_SET1(3) FBOCD_SET1(4) FBOCD_SET1(5) FBOCD_SET1(6) FBOCD_SET1(7)
                 FBOCD_SET1(8) FBOCD_SET1(9) FBOCD_SET1(10) FBOCD_SET1(11) FBOCD_SET1(12) FBOCD_SET1(13) FBOCD_SET1(14) FBOCD_SET1(15) }
#undef FBOCD_SET1
}

// log2 of v >= 0 for the per-step scalars (new change-point mass, MERGE bucket):
// 0 -> -inf (kImpossible under FLOOR); arguments outside fast_log2's range (2^-1000, 2^1000)
// are scaled by 2^-+600.
__device__ __forceinline__ double safe_log2(double v) {
    const bool tiny = v < 0x1p-900;
    const bool huge = v > 0x1p+900;
    const double s = tiny ? v * 0x1p+600 : (huge ? v * 0x1p-600 : v);
    const double l = fast_log2(s, 0x800u) + (tiny ? -600.0 : (huge ? 600.0 : 0.0));
    return v > 0.0 ? l : kImpossible;
}

// Prior predictive of x (A1 + A2 of the prior, log2 units): the tile's exponent
// references K0_t = round(l0_t).  ca0 = {G_1, alpha_1}, ap = alpha0 lg beta0.
__device__ __forceinline__ double prior_l2(double x, double mu0, double be0, double ap, double2 ca0, double y0,
                                           unsigned fmb) {
    const double d = x - mu0;
    const double mun = fma(d, y0, mu0);
    const double bn = fma(d, fma(mun, -0.5, 0.5 * x), be0);
    const double Ln = fast_log2(bn, fmb);
    return fma(-ca0.y, Ln, ca0.x + ap);
}

// ---------------------------------------------------------------------------
// The kernel.
//   FULL : R == NT*J (powers of two) at compile time.  FULL kernels ROTATE the
//          slot <-> position map by one slot every NT steps (slot j of thread i
//          holds position i + NT*((j + phi) mod J), phi = pB / NT for the
//          position pB the step recycles), so the recycled cell is always slot 0:
//          its prior reset is a compile-time register write, and every table
//          offset of a slot is a compile-time constant.
//   TAB2 : doubled per-r tables (generic R <= 2048);
//   EAGER: the MAP run length r* is reduced every step (per-step MAP output,
//          MAPRESET events, or theta < 1/2); otherwise r* = 1 at every PROB event.
// ---------------------------------------------------------------------------
template <int NT, int J, bool FULL, bool TAB2>
__host__ __device__ constexpr int table_entries(int R) {
    return FULL ? R + NT : (TAB2 ? 2 * R : R);  // FULL: index r or r + R, r + R < R + NT
}

// The dynamic shared window of a non-cluster launch starts at this shared address
// (after the 1 KB system reservation; no static shared memory in this kernel), so
// the fast-math tables sit at the compile-time address kFmBase (checked at entry).
constexpr unsigned kDynBase = 0x400u;
constexpr unsigned kFmBase = 0x800u;
// The cell loop's tables (cellmath.cuh) follow the fast-math tables at compile-time
// addresses; the per-r tables start after them.  EC: copies of the exp2 table (16, conflict-
// free, for the R <= 1024 FULL kernels; 8 otherwise, where the per-r tables are larger).
// The persistent prefetching kernels (HBM-bound streaming) take 4 copies and 64-step x tiles
// so that two CTAs with their prefetch buffers still fit one SM.
__host__ __device__ constexpr int cell_ec(bool full, int r_full, bool pref) {
    return pref ? 4 : ((full && r_full <= 1024) ? 16 : 8);
}
__host__ __device__ constexpr unsigned bocd_fm_bytes(int ec, int lb) {
    return (lb == 8 ? (ec == 16 ? cell_tables_end<16, 8>() : ec == 8 ? cell_tables_end<8, 8>()
                                   : ec == 4 ? cell_tables_end<4, 8>() : cell_tables_end<2, 8>())
                    : (ec == 16 ? cell_tables_end<16, 10>() : ec == 8 ? cell_tables_end<8, 10>()
                                   : ec == 4 ? cell_tables_end<4, 10>() : cell_tables_end<2, 10>())) -
           kDynBase;
}
static_assert(kFmBase + kFmSmemBytes - 2048u <= kCellExpBase, "fast-math tables overlap the cell tables");

// exp2 of a cell: q' = 2^(ell - Dc) with C7 = 1.5 2^52 + 2^31 - 256 Dc (cellmath.cuh's
// reduction with the frame folded into the rounding constant).  Below 2^-1021: floored to
// [2^-1021, 2^-1019).  The cell loop evaluates
// the same operations stage by stage (this scalar form serves the accuracy probe).
template <int EC>
__device__ __forceinline__ double cell_exp2(double ell, double C7, unsigned lbe) {
    const double zf = fma(ell, kCellExpScale, C7);
    const unsigned ki = unsigned(__double2loint(zf));
    const double re = fma(zf - C7, -1.0 / kCellExpScale, ell);
    const double T = cell_exp_entry<EC>(ki, lbe);
    double p = fma(re, kCellExpQ3, c_cell[11]);
    p = fma(p, re, c_cell[10]);
    p = fma(p, re, c_cell[9]);
    const double qq = p * re;
    const unsigned kc = max(ki, kCellExpLo);  // the floor only (see the cell loop)
    const double Ts = __hiloint2double(int(kc * (1048576u >> kCellEB)) + __double2hiint(T), __double2loint(T));
    return fma(Ts, qq, Ts);
}

// PREF is used for power-of-two R up to 1024, where the buffer (24 B x R per series) fits
// without lowering the 2-CTA/SM occupancy
template <int NT, int J, bool FULL>
constexpr bool kPrefOk = FULL && NT * J <= 1024;

// Persistent kernel: each CTA loops over work units of SPB series (unit u = series
// [u*SPB, u*SPB + SPB)), u = blockIdx.x, blockIdx.x + gridDim.x, ...  Tables are set up
// once per CTA.  PREF: the state rows (mu, beta, a) and scalars of the group's NEXT unit
// are prefetched into shared memory by 1-D TMA bulk copies while the current unit computes
// (streaming calls with a few steps per call are then bound by HBM, not by load latency).
template <int NT, int J, bool FULL, bool TAB2, bool EAGER, int SPB, int MINB, bool PERSIST, int MODE>
__global__ void __launch_bounds__(NT* SPB, MINB) bocd_update_kernel(const KParams P) {
    // PERSIST: grid = co-resident CTAs looping over units (streaming calls); otherwise one
    // unit per CTA (long calls: the hardware scheduler, no loop overhead).  Same arithmetic.
    constexpr bool PREF = PERSIST && kPrefOk<NT, J, FULL>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool ROT = FULL;
    // FULL kernels: the exp2 polynomial of degree 3 (2.4e-14 relative, one DFMA less) for slots
    // >= 2; slots 0 and 1 keep degree 4 (4.8e-18): theirs are the masses carried forward as
    // weights (slot 0: the new change-point cell and the MERGE bucket q'_{R-2} + q'_{R-1} every
    // step; slot 1 of thread 0: the bucket's weight at the rotation steps), where a bias would
    // accumulate.  Every other cell's mass is recomputed from its statistics each step, and its
    // l = a + G - alpha lg beta' already carries ~1e-12 of rounding (measured: parity
    // unchanged, C3 73.8 -> 71.3 ms with the fused sum below, C4 1074 -> 1025 ms per call)
    constexpr bool EXP3 = FULL;
    // the owner updates of the scalar tail only in the (one or two) warps holding an owner lane
    // for groups of >= 8 warps (R = 2048 / 4096: C4 1026 -> 994 ms per call); for 4 warps
    // (R = 1024) the branch costs more than the skipped selects (71.25 vs 71.53 ms)
    constexpr bool OWNW = NT >= 256;
    constexpr int EC = cell_ec(FULL, NT * J, PREF);
    constexpr int LB = cell_logbits(FULL, NT * J);
    // the MERGE bucket's multiplicative continuation (below) for R >= 2048, where the log-joint's
    // larger terms (alpha to 2048, frames of up to 512 steps) would carry ~1e-12 per step of
    // rounding along the bucket's chain (6.3e-10 measured at R = 2048 after 5,120 steps); at
    // R <= 1024 the plain form measures 6.2e-11 after the full 100,000 C3 steps
    constexpr bool BUCKET_PRED = FULL && NT * J >= 2048 && (MODE & 1) == 0;
    // FULL: absolute shared addresses of the per-r tables (the dynamic window starts at
    // kDynBase, checked at entry with the fast-math tables)
    constexpr unsigned kGyBase = kDynBase + bocd_fm_bytes(EC, LB);  // FULL: {G_{r+1}, y_r} rows
    constexpr int TILE = PREF ? kTileP : kTile;
    constexpr int W = n_partials(NT);  // per-series partials of a step (one per warp)
    using GS = GroupSmem<NT, TILE>;
    const int R = FULL ? NT * J : P.R;
    const int RT = table_entries<NT, J, FULL, TAB2>(R);
    // dynamic shared memory: [fast-math tables, cell tables (bocd_fm_bytes)][per-r tables][groups]
    unsigned char* const smem = smem_raw;
    // generic: s_ca = {G_{r+1}, alpha_{r+1}}, s_y = y_r; FULL: s_gy = {G_{r+1}, y_r} (same base)
    double2* s_ca = reinterpret_cast<double2*>(smem + bocd_fm_bytes(EC, LB));
    double* s_y = reinterpret_cast<double*>(s_ca + RT);
    double2* s_gy = s_ca;
    unsigned char* gbase = smem + bocd_fm_bytes(EC, LB) + table_bytes(RT, FULL);

    for (int k = threadIdx.x; k < RT; k += blockDim.x) {
        const int r = k < R ? k : k - R;
        if constexpr (FULL) {
            s_gy[k] = make_double2(P.tab_ca[r].x, P.tab_y[r]);
        } else {
            s_ca[k] = P.tab_ca[r];
            s_y[k] = P.tab_y[r];
        }
    }
    const bool fm_ok = smem_addr(smem_raw) == kDynBase && fm_setup(smem_raw, P.fm) == kFmBase;
    {
        double* ex = reinterpret_cast<double*>(smem_raw + (kCellExpBase - kDynBase));
        for (int k = threadIdx.x; k < kCellExpTab * EC; k += blockDim.x) ex[k] = P.ct->exptab[k / EC];
        double2* lg = reinterpret_cast<double2*>(smem_raw + (cell_log_base<EC>() - kDynBase));
        // FULL kernels evaluate the half-log (cellmath.cuh, cell_log2h): halved table values
        const double2* src = FULL ? (LB == 8 ? P.ct->log8h : P.ct->log10h) : (LB == 8 ? P.ct->log8 : P.ct->log10);
        for (int k = threadIdx.x; k < (1 << LB); k += blockDim.x) lg[k] = src[k];
    }
    const unsigned lb = 8u * (threadIdx.x & unsigned(EC - 1));  // exp2 table copy of this lane
    const int g = threadIdx.x / NT;
    const int i = threadIdx.x % NT;
    const int lane = threadIdx.x & 31;
    const int w = i >> 5;
    GS& gs = *reinterpret_cast<GS*>(gbase + size_t(g) * group_bytes<NT, PREF>(R));
    // PREF: the prefetched next-unit state [mu R][beta R][a R][SeriesScalars], position order
    double* const pf = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(&gs) + sizeof(GS));
    SeriesScalars* const pf_sc = reinterpret_cast<SeriesScalars*>(pf + 3 * size_t(R));
    // balanced (the one-CTA-per-SM twins, MINB = 1 with several groups: one wave, grid = #SM):
    // every CTA takes floor or ceil of S / grid series, so no SM carries more than
    // ceil(S / #SM); the host launches them only for S <= #SM * SPB (32-bit arithmetic)
    constexpr bool bal = !PERSIST && MINB == 1 && SPB > 1;
    const int64_t nunits = bal ? int64_t(gridDim.x) : (P.S + SPB - 1) / SPB;
    if (i == 0) {
        mbar_init(&gs.mbar[0], 1);
        mbar_init(&gs.mbar[1], 1);
        mbar_init(&gs.mbar_st, 1);
        mbar_fence_init();
    }
    __syncthreads();
    const int ntiles = (P.T + TILE - 1) / TILE;
    const int tl_min = P.t0 == 0 ? 1 : 0;  // no events at global t = 0 (Q8): local steps tl >= tl_min
    constexpr bool merge = (MODE & 1) == 0;  // truncation at R: MERGE (0) or DROP (1)
    constexpr bool FRAC = FULL && (MODE & 2);  // 2 alpha0 not an integer: + f2 per cell
    const bool any_out = P.out_map || P.out_pnew || P.out_logz;  // per-step outputs requested
    // argmax-eligible run lengths: MERGE r <= R-3 (slot R-1 is the bucket), DROP r <= R-2
    const int r_elig = merge ? R - 3 : R - 2;
    const double ninf = kImpossible;
    unsigned xphase = 0u;  // parity of the two x-tile mbarriers (bit b: mbar[b])
    unsigned sphase = 0u;  // parity of the state mbarrier
    auto issue_state = [&](int64_t sn) {  // thread 0 of the group: next unit's state -> pf
        const unsigned bytes = unsigned(3 * size_t(R) * sizeof(double) + sizeof(SeriesScalars));
        fence_proxy_async();
        mbar_arrive_expect_tx(&gs.mbar_st, bytes);
        const size_t rb = size_t(R) * sizeof(double);
        tma_load_1d(pf, P.st_mu + sn * R, unsigned(rb), &gs.mbar_st);
        tma_load_1d(pf + R, P.st_beta + sn * R, unsigned(rb), &gs.mbar_st);
        tma_load_1d(pf + 2 * size_t(R), P.st_a + sn * R, unsigned(rb), &gs.mbar_st);
        tma_load_1d(pf_sc, P.scal + sn, unsigned(sizeof(SeriesScalars)), &gs.mbar_st);
    };
    if constexpr (PREF) {
        const int64_t s0 = int64_t(blockIdx.x) * SPB + g;
        if (i == 0 && P.t0 > 0 && blockIdx.x < nunits && s0 < P.S) issue_state(s0);
    }
    // PREF streaming calls whose x rows are not TMA-able (T = 1: one 8-byte value per series):
    // thread i holds x[s][i] of its unit in a register, loaded during the previous unit, so the
    // global-load latency is off each unit's critical path
    const bool xreg = PREF && P.T <= NT && !tile_tma_ok<TILE>(P, 0);
    double xv = 0.0;
    if (xreg) {
        const int64_t s0 = int64_t(blockIdx.x) * SPB + g;
        if (i < P.T && s0 < P.S) xv = P.x[s0 * P.ld + i];
    }

    for (int64_t u = blockIdx.x; u < nunits; u += PERSIST ? int64_t(gridDim.x) : nunits) {
        const int64_t s = bal ? int64_t(unsigned(u) * unsigned(P.S) / gridDim.x) + g : u * SPB + g;
        if (s >= (bal ? int64_t(unsigned(u + 1) * unsigned(P.S) / gridDim.x) : P.S)) break;  // group-uniform
        const double* xrow = P.x + s * P.ld;
        // Prefetch tile 0 (TMA) as early as possible.
        if (i == 0 && ntiles > 0 && tile_tma_ok<TILE>(P, 0)) issue_tile_tma<NT, TILE>(gs, xrow, 0, P.T);

        // ---- load or initialise the state --------------------------------
        double mu[J], be[J], a[J];
        // ROT: pending weight of slot 0 (the mass of a new change-point / bucket cell, kept as a
        // factor of its q' until the next rotation step folds it into a)
        double wq = 1.0;
        // BUCKET_PRED: lg beta of slot 0 at the previous step.  The cell that truncation at R
        // recycles (r = R-1, slot 0 of thread iB) is the MERGE bucket; its mass is continued
        // multiplicatively by its Student-t predictive,
        // q' = w 2^(c_{R-1}/ln2 + alpha_{R-1} (lg beta - lg beta') - lg beta'/2 - N_t), whose
        // terms are O(10): the log-joint's O(10^3..10^4) terms would carry their rounding
        // (~1e-12 per step) along the bucket's chain of merged masses.
        double L0p = 0.0;
        const int64_t sbase = s * int64_t(R);
        if constexpr (PREF) {
            if (P.t0 > 0) {
                mbar_wait(&gs.mbar_st, sphase);
                sphase ^= 1u;
            }
        }
        if (i == 0) {
            SeriesScalars sc = (PREF && P.t0 > 0) ? *pf_sc : P.scal[s];
            if (P.t0 == 0) {
                if (P.prior_first_obs && P.T > 0) {
                    const double x0 = xrow[0];
                    sc.mu0 = x0;
                    sc.beta0 = P.alpha0 * (P.prior_cov * x0) * (P.prior_cov * x0);
                }
                sc.zd_prev = P.omH;  // R_{-1} = [1, 0, ...] = q (1-H)/Zd
                sc.map_prev = 0;
                sc.dc = 0;
            }
            const bool ok = sc.beta0 >= 2.2250738585072014e-308 && sc.beta0 < 1e300 && isfinite(sc.mu0);
            gs.mu0 = sc.mu0;
            gs.beta0 = ok ? sc.beta0 : 1.0;
            gs.L0 = fast_log2(gs.beta0, kFmBase);
            gs.aprior = P.alpha0 * gs.L0;
            gs.zd_prev = sc.zd_prev;
            gs.map_prev = sc.map_prev;
            gs.ev_count = sc.ev_count;
            gs.flags = sc.flags | (ok ? 0 : 2) | (fm_ok ? 0 : 4);
            gs.dc0 = sc.dc;
        }
        group_sync<NT>(g);
        // the prior and the rarely used per-series scalars stay in shared memory (gs) so
        // that the step loop keeps its registers for the cells
        int zexp = ((__double2hiint(gs.zd_prev) >> 20) & 0x7FF) - 1023;  // binary exponent of Zd_{t-1}
        int map_prev = gs.map_prev, ev_count = gs.ev_count;
        int dc = gs.dc0;  // Dc_{t-1}
        // ring bookkeeping.  FULL: the recycled position pB = (t+1) mod R = NT*phi + iB;
        // generic: tmod = t mod R.
        int tmod = int(P.t0 % R);
        int iB = 0, phi = 0;
        if constexpr (ROT) {
            const int pB0 = (tmod + 1 == R) ? 0 : tmod + 1;
            iB = pB0 % NT;
            phi = pB0 / NT;
        }
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int p = ROT ? i + NT * ((j + phi) & (J - 1)) : i + NT * j;  // position of slot j
            if (FULL || p < R) {
                if (P.t0 == 0) {
                    mu[j] = gs.mu0;
                    be[j] = gs.beta0;
                    a[j] = (p == 0) ? gs.aprior : ninf;  // before x_0 a segment starts w.p. 1 (Q8)
                } else {
                    if constexpr (PREF) {
                        mu[j] = pf[p];
                        be[j] = pf[R + p];
                        a[j] = pf[2 * R + p];
                    } else {
                        mu[j] = P.st_mu[sbase + p];
                        be[j] = P.st_beta[sbase + p];
                        a[j] = P.st_a[sbase + p];
                    }
                }
            } else {
                mu[j] = gs.mu0;
                be[j] = gs.beta0;
                a[j] = ninf;
            }
        }
        if constexpr (ROT) {
            if (P.t0 > 0) wq = P.st_w[s * NT + i];
            // before x_0 the cell that step 0 truncates (thread iB's slot 0) is impossible: its
            // continuation weight is 0 (later steps: the bucket the previous step formed)
            else if (BUCKET_PRED && i == iB) wq = 0.0;
            if (BUCKET_PRED) L0p = cell_log2h<EC, LB>(be[0]);  // = the previous step's lg beta'/2 of slot 0
        }
        if constexpr (PREF) {
            // pf is free once every thread of the group has read it: prefetch the next unit
            group_sync<NT>(g);
            const int64_t sn = s + int64_t(gridDim.x) * SPB;
            if (i == 0 && P.t0 > 0 && sn < P.S) issue_state(sn);
        }
        bool nonfinite = false;
        if (i == 0 && P.out_logz) gs.lzd_prev = fast_log2(gs.zd_prev, kFmBase);

        for (int k = 0; k < ntiles; ++k) {
            const int base = k * TILE;
            const int n = min(TILE, P.T - base);
            const int buf = k & 1;
            // prefetch the next tile into the other buffer (its previous readers all
            // passed at least one group barrier since their last read)
            if (i == 0 && k + 1 < ntiles && tile_tma_ok<TILE>(P, k + 1)) issue_tile_tma<NT, TILE>(gs, xrow, k + 1, P.T);
            if (tile_tma_ok<TILE>(P, k)) {
                mbar_wait(&gs.mbar[buf], (xphase >> buf) & 1u);
                xphase ^= 1u << buf;
            } else if (xreg) {  // (one tile, n = T <= NT)
                if (i < n) gs.xbuf[buf][i] = xv;
                group_sync<NT>(g);
                const int64_t sn = s + int64_t(gridDim.x) * SPB;  // the next unit's x, in flight now
                if (i < n && sn < P.S) xv = P.x[sn * P.ld + i];
            } else {
                for (int q = i; q < n; q += NT) gs.xbuf[buf][q] = xrow[base + q];
                group_sync<NT>(g);
            }
            // the tile's exponent references K0_t = round(l0_t), spread over the group
            for (int q = i; q < n; q += NT) {
                const double xq = gs.xbuf[buf][q];
                if (!isfinite(xq)) nonfinite = true;
                const double l0 = FULL ? prior_l2(xq, gs.mu0, gs.beta0, gs.aprior, make_double2(s_gy[0].x, P.alpha0 + 0.5),
                                                  s_gy[0].y, kFmBase)
                                       : prior_l2(xq, gs.mu0, gs.beta0, gs.aprior, s_ca[0], s_y[0], kFmBase);
                gs.kbuf[buf][q] = __double2int_rn(fmin(fmax(l0, -kK0Max), kK0Max));
            }
            group_sync<NT>(g);
            // ROT: the tile's steps run in segments that end at a rotation step (iB = NT-1); the
            // slot rotation, the fold of the pending weights and the frame rebase run between
            // segments (register permutations outside the step loop: no copies inside it)
            for (int q = 0; q < n;) {
            const int qe = ROT ? min(n, q + (NT - iB)) : n;
            for (; q < qe; ++q) {
                const int tl = base + q;
                const int64_t t = P.t0 + tl;
                const double x = gs.xbuf[buf][q];
                const double hx = 0.5 * x;
                const int K0 = gs.kbuf[buf][q];
                if (!ROT && (unsigned(t) & (kRebase - 1)) == 0u) {  // generic: rebase at t % kRebase == 0
                    const double dcd = double(dc);
#pragma unroll
                    for (int j = 0; j < J; ++j) a[j] = fmax(a[j] - dcd, kImpossible);
                    dc = 0;
                }
                dc += K0 + zexp;  // Dc_t = Dc_{t-1} + N_t
                // exp2 rounding constant 1.5*2^52 + 2^31 - 256 Dc_t: zf = fma(l, 256, C7) holds
                // round(256 l) - 256 Dc_t + 2^31 in its low word (exact integers below 2^52)
                const double C7 = __hiloint2double(0x43380000, int(0x80000000u - unsigned(dc) * unsigned(kCellExpTab)));
                // the bucket's continuation is relative to the previous step's frame: shift N_t only
                const double C7b = __hiloint2double(0x43380000, int(0x80000000u - unsigned(K0 + zexp) * unsigned(kCellExpTab)));
                // ---- A1-A4 for the J cells (groups of G, every stage across the group) ----
                // table index of slot j: ib - NT*j  (= r or r + R).  FULL: r of slot j is
                // (pB - 1 - p) mod R = (iB - 1 - i - NT j) mod R.
                const int ib = ROT ? iB - 1 - i + R : tmod - i + R;
                // the cells the tail needs (r = R-2 -> qA, R-1 -> qB, 0 -> q0) and their owners
                int kA, kB, k0;
                if constexpr (ROT) {
                    kB = iB;                          // slot 0 of thread iB
                    kA = iB + 1;                      // slot 0 of thread iB+1, or slot 1 of thread 0
                    k0 = (iB == 0) ? R - 1 : iB - 1;  // slot 0 of thread iB-1, or slot J-1 of thread NT-1
                } else {
                    kB = (tmod + 1 == R) ? 0 : tmod + 1;
                    kA = (kB + 1 == R) ? 0 : kB + 1;
                    k0 = tmod;
                }
                const int par = tl & 1;
                const int mb = FULL ? P.a2p1 + ib : 0;  // 2 alpha0 + 1 + (table index of slot 0)
                double sum = 0.0;
                unsigned long long key = 0ull;
                // EAGER, ROT: this step's argmax codes (below R + NT: 12 bits up to R = 2048, 13 at
                // R = 4096) and the two ineligible growth candidates
                constexpr unsigned kKeyBits = (ROT && NT * J + NT > 4096) ? 13u : 12u;
                constexpr unsigned kKeyHi = ~((1u << kKeyBits) - 1u);
                const unsigned kcb = unsigned(i) | kKeyHi;
                const unsigned kc0 = kcb | ((ROT && ib >= R) ? unsigned(R) : 0u);
                const bool elig0 = !(i == iB || (merge && i == iB + 1));
                const bool elig1 = !(merge && iB == NT - 1 && i == 0);
#pragma unroll
                for (int j0 = 0; j0 < J; j0 += kG) {
                    constexpr int G = (J < kG) ? J : kG;
                    int idx[G];
                    double2 ca[G];
                    double yv[G], d[G], bn[G];
#pragma unroll
                    for (int kk = 0; kk < G; ++kk) {  // table loads
                        const int j = j0 + kk;
                        const int p = i + NT * j;
                        if (ROT || TAB2) {
                            idx[kk] = ib - NT * j;
                        } else {
                            idx[kk] = tmod - p;
                            idx[kk] += (idx[kk] < 0) ? R : 0;
                        }
                        if (!FULL && p >= R) idx[kk] = 0;  // masked cell: any valid entry
                        if constexpr (FULL) {  // compile-time shared addresses (no generic pointers)
                            // {G_{r+1}, y_r} and 2 alpha_{r+1} = 2 alpha0 + r + 1 (exact integer, I2F.F64);
                            // r = idx - R for the one slot whose index wrapped (slot 0)
                            const double2 gy = lds_v2f64(unsigned(idx[kk]) * 16u + kGyBase);
                            const int m2 = mb - NT * j - ((j == 0 && idx[kk] >= R) ? R : 0);
                            ca[kk] = make_double2(gy.x, FRAC ? __int2double_rn(m2) + P.f2 : __int2double_rn(m2));
                            yv[kk] = gy.y;
                        } else {
                            ca[kk] = s_ca[idx[kk]];
                            yv[kk] = s_y[idx[kk]];
                        }
                    }
                    // A1: NIG update
#pragma unroll
                    for (int kk = 0; kk < G; ++kk) d[kk] = x - mu[j0 + kk];
#pragma unroll
                    for (int kk = 0; kk < G; ++kk) mu[j0 + kk] = fma(d[kk], yv[kk], mu[j0 + kk]);
#pragma unroll
                    for (int kk = 0; kk < G; ++kk) {
                        bn[kk] = fma(d[kk], fma(mu[j0 + kk], -0.5, hx), be[j0 + kk]);
                        be[j0 + kk] = bn[kk];
                    }
                    // A2: lg beta' (cell_log2 of cellmath.cuh, stage by stage)
                    unsigned tb[G];
                    double2 lt[G];
                    double rl[G], kt[G], pl[G];
#pragma unroll
                    for (int kk = 0; kk < G; ++kk) {
                        tb[kk] = unsigned(__double2hiint(bn[kk]));
                        lt[kk] = cell_log_entry<EC, LB>(tb[kk]);
                    }
#pragma unroll
                    for (int kk = 0; kk < G; ++kk) {
                        const double invs = __hiloint2double(__double2hiint(lt[kk].x) + 0x3FF00000 -
                                                                 int(tb[kk] & 0x7FF00000u),
                                                             __double2loint(lt[kk].x));
                        rl[kk] = fma(bn[kk], invs, -1.0);
                        // I2F.F64: k exact.  FULL: the half-log (cell_log2h), k/2 + l_i/2
                        kt[kk] = FULL ? fma(__int2double_rn(int(tb[kk] >> 20) - 1023), 0.5, lt[kk].y)
                                      : __int2double_rn(int(tb[kk] >> 20) - 1023) + lt[kk].y;
                    }
                    {
                        constexpr int o = FULL ? 12 + 3 * (LB - 8) : 3 * (LB - 8);
#pragma unroll
                        for (int kk = 0; kk < G; ++kk)
                            pl[kk] = fma(rl[kk], FULL ? kCellLogP3h<LB> : kCellLogP3<LB>, c_cell[o + 2]);
#pragma unroll
                        for (int kk = 0; kk < G; ++kk) pl[kk] = fma(pl[kk], rl[kk], c_cell[o + 1]);
#pragma unroll
                        for (int kk = 0; kk < G; ++kk) pl[kk] = fma(pl[kk], rl[kk], c_cell[o]);
                    }
                    double ell[G];
#pragma unroll
                    for (int kk = 0; kk < G; ++kk) {
                        const int j = j0 + kk;
                        // lg beta' (FULL: lg beta' / 2, multiplied by 2 alpha: the same product)
                        const double Ln = fma(rl[kk], pl[kk], kt[kk]);
                        ell[kk] = fma(-ca[kk].y, Ln, a[j] + ca[kk].x);
                        if constexpr (BUCKET_PRED) {
                            if (j == 0) {  // the truncated cell (thread iB): the bucket's continuation
                                // alpha (lg beta - lg beta') - lg beta'/2 with half-logs (FULL)
                                const double lb_ = fma(P.al2_bucket, L0p - Ln, P.c_bucket - Ln);
                                ell[kk] = (i == iB) ? lb_ : ell[kk];
                                L0p = Ln;
                            }
                        }
                        if constexpr (ROT) {  // lg beta' of slot 0 (and slot 1 of thread 0) for the bucket
                            if (j == 0 && i == iB + 1) gs.l0[par][i] = Ln;  // only the bucket's is read
                            if (J > 1 && j == 1 && i == 0) gs.l0[par][NT] = Ln;
                        } else {
                            if (merge && i + NT * j == kA) gs.spec[par][3] = fma(-ca[kk].y, Ln, ca[kk].x);
                        }
                    }
                    // A3: q' = 2^(l - Dc_t)  (cell_exp2, stage by stage)
                    double re[G], pe[G], Tv[G];
                    unsigned ki[G];
#pragma unroll
                    for (int kk = 0; kk < G; ++kk) {
                        const double Cj = (BUCKET_PRED && j0 + kk == 0 && i == iB) ? C7b : C7;
                        const double zf = fma(ell[kk], kCellExpScale, Cj);
                        ki[kk] = unsigned(__double2loint(zf));
                        re[kk] = fma(zf - Cj, -1.0 / kCellExpScale, ell[kk]);  // exact, |re| <= 2^-(EB+1)
                        Tv[kk] = cell_exp_entry<EC>(ki[kk], lb);
                    }
#pragma unroll
                    for (int kk = 0; kk < G; ++kk)
                        pe[kk] = EXP3 && j0 + kk >= 2 ? fma(re[kk], kCellExpQ2c, c_cell[22])
                                                      : fma(re[kk], kCellExpQ3, c_cell[11]);
#pragma unroll
                    for (int kk = 0; kk < G; ++kk)
                        pe[kk] = EXP3 && j0 + kk >= 2 ? fma(pe[kk], re[kk], c_cell[21]) : fma(pe[kk], re[kk], c_cell[10]);
#pragma unroll
                    for (int kk = 0; kk < G; ++kk)
                        if (!(EXP3 && j0 + kk >= 2)) pe[kk] = fma(pe[kk], re[kk], c_cell[9]);
#pragma unroll
                    for (int kk = 0; kk < G; ++kk) {
                        const int j = j0 + kk;
                        const int p = i + NT * j;
                        const double qq = ROT ? 0.0 : pe[kk] * re[kk];
                        // 2^e, e = floor(n/256) for n = ki - 2^31, floored at 2^-1021 and clamped at
                        // +1000; hi word = kc * 2^12 + hi(T'_j) (cellmath.cuh)
                        // only the lower clamp (the floor): every cell's joint is below the step's
                        // evidence Z, which the frame Dc_t keeps within a few binades of 1 (Dc_t tracks
                        // the prior predictive of x_t and the exponent of Zd_{t-1}; no run length's
                        // predictive exceeds the prior predictive by more than ~sqrt(2 alpha_r)), so
                        // 2^+1000 is unreachable for finite x
                        const unsigned kc = max(ki[kk], kCellExpLo);
                        const double Ts = __hiloint2double(int(kc * (1048576u >> kCellEB)) + __double2hiint(Tv[kk]),
                                                           __double2loint(Tv[kk]));
                        double E;
                        if constexpr (ROT) {
                            // q' = Tw u with u = 2^re = 1 + re Q(re) and Tw = 2^(n/256) (x slot 0's
                            // pending weight: new CP / bucket mass); the sum takes Tw u fused, and
                            // q' itself is formed only where it is read (EAGER keys, published cells)
                            const double u = fma(pe[kk], re[kk], 1.0);
                            const double Tw = j == 0 ? Ts * wq : Ts;
                            sum = fma(Tw, u, sum);
                            E = (EAGER || j == 0 || (J > 1 && j == 1) || j == J - 1) ? Tw * u : 0.0;
                        } else {
                            E = fma(Ts, qq, Ts);
                            if (FULL || p < R) sum += E;
                        }
                        if (FULL || p < R) {
                            if constexpr (EAGER) {
                                if constexpr (ROT) {
                                    // key = E's bits with the low 12 (13) replaced by the cell's code
                                    // i + NT j (+ R for the wrapped slot 0): r = R + iB - 1 - code for
                                    // every cell, so the larger code is the smaller run length (ties ->
                                    // smaller r).  One LOP3: (lo & b & c) | (b ^ c), b = code bits
                                    // of the thread (| kKeyHi), c = NT j | kKeyHi (disjoint low bits)
                                    const unsigned bc = j == 0 ? kc0 : kcb;
                                    const unsigned cc = kKeyHi | unsigned(NT * j);
                                    const unsigned lo = (unsigned(__double2loint(E)) & bc & cc) | (bc ^ cc);
                                    unsigned long long kq =
                                        (static_cast<unsigned long long>(unsigned(__double2hiint(E))) << 32) | lo;
                                    if (j == 0 && !elig0) kq = 0ull;  // kB (r = R-1) / MERGE kA (r = R-2)
                                    if (J > 1 && j == 1 && !elig1) kq = 0ull;
                                    key = kq > key ? kq : key;
                                } else {
                                    int r = idx[kk];
                                    r -= (r >= R) ? R : 0;
                                    const unsigned long long kq = argmax_key(E, r);
                                    key = (r <= r_elig && kq > key) ? kq : key;
                                }
                            }
                            // the tail's cells, published by their owners
                            if constexpr (ROT) {
                                if (j == 0 && unsigned(i - iB + 1) <= 2u) gs.e0[par][i] = E;  // iB-1 .. iB+1
                                if (J > 1 && j == 1 && i == 0) gs.e0[par][NT] = E;
                                if (j == J - 1 && i == NT - 1) gs.e0[par][NT + 1] = E;
                            } else {
                                if (p == kA) gs.spec[par][0] = E;
                                if (p == kB) gs.spec[par][1] = E;
                                if (p == k0) gs.spec[par][2] = E;
                            }
                        }
                    }
                }
                // ---- series sum (and, EAGER, argmax): the step's only barrier -----------
                // (xor butterfly over the series' lanes of the warp, then a fixed-order
                // pairwise sum of the W per-warp partials: deterministic)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                if constexpr (EAGER) key = warp_max_u64(key);
                if constexpr (W > 1) {
                    if (lane == 0) {
                        gs.red2[par][w] = sum;
                        if (EAGER) gs.red1[par][w] = key;
                    }
                    group_sync<NT>(g);
                    sum = partials_sum<W>(gs.red2[par], lane);
                    if (EAGER && (!OWNW || w == 0)) {  // OWNW: only warp 0 reads the argmax
#pragma unroll
                        for (int ww = 0; ww < W; ++ww) {
                            const unsigned long long o = gs.red1[par][ww];
                            key = o > key ? o : key;
                        }
                    }
                } else {
                    group_sync<NT>(g);
                }
                // ---- the scalar tail (A5-A8): group-uniform, no transcendentals -----------
                const double Z = sum;
                double qA, qB, q0;
                if constexpr (ROT) {
                    qB = gs.e0[par][iB];
                    qA = gs.e0[par][iB + 1];
                    q0 = gs.e0[par][iB == 0 ? NT + 1 : iB - 1];
                } else {
                    qA = gs.spec[par][0];
                    qB = gs.spec[par][1];
                    q0 = gs.spec[par][2];
                }
                const double Zd = merge ? Z : Z - P.omH * qB;    // normaliser of the new posterior
                const double Zp = merge ? Z : Z - qB;            // p_new = pnum / Zp
                const double pnum = (merge && R == 2) ? Z : q0;  // MERGE R = 2: p_new = 1
                uint32_t fl = (tl >= tl_min && pnum > P.theta * Zp) ? 1u : 0u;
                // A6: the new change-point cell (owner of kB) and the MERGE bucket (owner of kA).
                // ROT: branch-free; the new mass is the slot-0 pending weight wq (no log on the
                // step's critical path), folded into a at the next rotation step.  Generic: one
                // divergent block for the one or two owner lanes (one shared log2 pass).
                if (ROT && (!OWNW || w == (iB >> 5) || w == ((iB + 1) >> 5))) {  // warps holding an owner
                    const bool ownB = (i == iB);
                    const bool ownA = merge && (i == iB + 1);  // iB = NT-1: thread 0, slot 1 (rotation)
                    const double dcd = double(dc);
                    // G_{R-1} - alpha_{R-1} lg beta' of cell kA (half-log x 2 alpha_{R-1})
                    const double GA = lds_v2f64(kGyBase + unsigned(NT * J - 2) * 16u).x;
                    const double offA = fma(-P.al2_bucket, gs.l0[par][iB + 1], GA);
                    const double m0 = gs.mu0, b0 = gs.beta0;
                    const double aB = gs.aprior + dcd, aA = dcd - offA;
                    const double wB = P.hr * Z, wA = bucket_mass(qA, qB);
                    mu[0] = ownB ? m0 : mu[0];
                    be[0] = ownB ? b0 : be[0];
                    a[0] = ownB ? aB : (ownA ? aA : a[0]);
                    wq = ownB ? wB : (ownA ? wA : wq);
                } else if constexpr (!ROT) {
                const bool ownB = (unsigned(kB) % NT) == unsigned(i);
                const bool ownA = merge && ((unsigned(kA) % NT) == unsigned(i));
                if (ownB || ownA) {
                    const double lv = safe_log2(ownB ? P.hr * Z : bucket_mass(qA, qB));
                    if (ownB) {  // R_t(0) = H Z / Zd: mass hr Z in this step's frame, prior statistics
                        const double anew = (lv + gs.aprior) + double(dc);
                        const int jb = kB / NT;
                        set_slot<J>(mu, jb, gs.mu0);
                        set_slot<J>(be, jb, gs.beta0);
                        set_slot<J>(a, jb, anew);
                    } else {  // bucket: q'_{R-2} + q'_{R-1} with the window statistics of cell kA
                        const double anew = (lv - gs.spec[par][3]) + double(dc);  // spec[3] = G - alpha lg beta'
                        set_slot<J>(a, kA / NT, anew);
                    }
                }
                }
                if (i == 0) gs.zd_prev = Zd;
                // ---- rare path (group-uniform): MAP run length r* (A7), events (A8), per-step
                // outputs ----------------------------------------------------------------
                // (OWNW: warp 0 only — thread 0 alone writes events and outputs and keeps r*_{t-1}
                // and the event count; the other warps skip the EAGER per-step work: C4 EAGER
                // 1326 -> 1293 ms; with 4 warps the branch costs more, 85.0 vs 85.3 for C3)
                if ((EAGER || (fl & P.ev_mask) || any_out) && (!OWNW || w == 0)) {
                    int r_ex = -1;
                    double qex = 0.0;
                    if constexpr (EAGER) {
                        if (key != 0ull) {
                            if constexpr (ROT) {
                                constexpr unsigned long long kLow = (NT * J + NT > 4096) ? 0x1FFFull : 0xFFFull;
                                r_ex = R + iB - 1 - int(key & kLow);
                                qex = __longlong_as_double(static_cast<long long>(key & ~kLow));
                            } else {
                                r_ex = key_r(key);
                                qex = key_val(key);
                            }
                        }
                    }
                    if (EAGER || (fl & P.ev_mask)) {
                        // lazy kernel: only PROB events reach here, and it runs only for theta >= 1/2
                        // (capi.cu): p_new = R_t(1) / sum_{r>=1} R_t(r) > theta >= 1/2 makes R_t(1)
                        // larger than all the other growth slots together, so r* = 1 and
                        // cp_index = t exactly.  EAGER: the step's reduced argmax key.
                        int rstar = 1;
                        if constexpr (EAGER) {
                            if (merge) {
                                // bucket (qA + qB) vs the best growth slot (ties -> the smaller run length)
                                rstar = (r_ex < 0 || (qA + qB) > qex) ? R - 1 : r_ex + 1;
                            } else {
                                rstar = r_ex + 1;
                            }
                        }
                        if (EAGER && tl >= tl_min && rstar < min(map_prev + 1, R - 1)) fl |= 2u;
                        map_prev = rstar;
                        if (i == 0 && P.out_map) P.out_map[s * P.ld_o + tl] = rstar;
                        if (fl & P.ev_mask) {
                            if (i == 0 && ev_count < P.ev_cap) {
                                EventRec ev;
                                ev.t = t;
                                ev.cp_index = t - rstar + 1;
                                ev.flags = fl & P.ev_mask;  // the requested bits only (kernel-independent)
                                ev.pad = 0;
                                ev.p_new = pnum * fast_rcp(Zp);
                                P.ev[s * P.ev_cap + ev_count] = ev;
                            }
                            ++ev_count;
                        }
                    }
                    if (i == 0) {
                        if (P.out_pnew) P.out_pnew[s * P.ld_o + tl] = pnum * fast_rcp(Zp);
                        if (P.out_logz) {  // kept mass (A4)
                            const double lzd = fast_log2(Zd, kFmBase);
                            P.out_logz[s * P.ld_o + tl] =
                                fma(LN2, double(K0 + zexp) + (lzd - gs.lzd_prev), P.ln_omH);
                            gs.lzd_prev = lzd;
                        }
                    }
                }
                zexp = ((__double2hiint(Zd) >> 20) & 0x7FF) - 1023;
                tmod = (tmod + 1 == R) ? 0 : tmod + 1;
                if constexpr (ROT) ++iB;
            }
            if (ROT && iB == NT) {  // the segment ended at a rotation step (group-uniform)
                const int par = (base + q - 1) & 1;  // that step's publication buffers
                // fold every pending weight into its cell, rebase the frame (a fixed global
                // schedule: every NT steps), then thread 0's bucket cell (slot 1 -> slot 0 after
                // the rotation) takes its weight q'_{R-2} + q'_{R-1}
                const double dcd = double(dc);
                a[0] += safe_log2(wq);
                wq = 1.0;
#pragma unroll
                for (int j = 0; j < J; ++j) a[j] = fmax(a[j] - dcd, kImpossible);
                dc = 0;
                if (merge && i == 0 && J > 1) {
                    const double GA = lds_v2f64(kGyBase + unsigned(NT * J - 2) * 16u).x;
                    a[1] = -fma(-P.al2_bucket, gs.l0[par][NT], GA);
                    wq = bucket_mass(gs.e0[par][NT], gs.e0[par][NT - 1]);
                }
                // rotate slot j <- slot j+1
                phi = (phi + 1) & (J - 1);
                const double m0 = mu[0], b0 = be[0], a0 = a[0];
#pragma unroll
                for (int j = 0; j + 1 < J; ++j) {
                    mu[j] = mu[j + 1];
                    be[j] = be[j + 1];
                    a[j] = a[j + 1];
                }
                mu[J - 1] = m0;
                be[J - 1] = b0;
                a[J - 1] = a0;
                if (BUCKET_PRED) L0p = cell_log2h<EC, LB>(be[0]);  // slot 0 is a new cell
                iB = 0;
            }
            }
        }
        // ---- spill -----------------------------------------------------------
        if (nonfinite) atomicOr(&gs.flags, 1);
        group_sync<NT>(g);
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int p = ROT ? i + NT * ((j + phi) & (J - 1)) : i + NT * j;
            if (FULL || p < R) {
                P.st_mu[sbase + p] = mu[j];
                P.st_beta[sbase + p] = be[j];
                P.st_a[sbase + p] = a[j];
            }
        }
        if constexpr (ROT) P.st_w[s * NT + i] = wq;
        if (i == 0) {
            SeriesScalars sc;
            sc.mu0 = gs.mu0;
            sc.beta0 = gs.beta0;
            sc.zd_prev = gs.zd_prev;
            sc.map_prev = map_prev;
            sc.ev_count = ev_count;
            sc.flags = gs.flags;
            sc.dc = dc;
            sc.pad2 = 0.0;
            P.scal[s] = sc;
            if (sc.flags) atomicOr(P.err, unsigned(sc.flags));
        }
        group_sync<NT>(g);  // gs is reused by the next unit
    }
}

}  // namespace fbocd
