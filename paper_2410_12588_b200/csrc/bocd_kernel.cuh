// bocd_kernel.cuh — resident batched BOCD kernel for sm_100a (fp64).
//
// One series group of NT threads owns one series; each thread owns J run-length
// cells.  The R cells of a series live in a RING indexed by position
// p = (segment start time) mod R (p = i + NT*j for thread i, register j): at
// global step t the cell at position p holds run length r = (t - p) mod R
// BEFORE x_t is absorbed, so growth r -> r+1 (App. A)
// moves no data, and the position that truncation at R recycles (r = R-1) is
// exactly the one that becomes the new change-point cell.  Per-r constants of
// the Student-t predictive come from a shared-memory table indexed by r.
//
// Per step (all fp64, no fast-math).  Every log-domain quantity is kept in BASE-2
// units (log2), so the transcendentals are the 9-instruction branch-free
// fast_log2 / fast_exp2 of fastmath.cuh; natural-log outputs are converted once.
//   A1  NIG update           mu' = mu + d/(kappa+1),  beta' = beta + kappa d^2 / (2(kappa+1))
//   A2  Student-t predictive l_r/ln2 = c_r/ln2 + alpha_r (lg beta - lg beta') - 1/2 lg beta'
//       (lg = log2; = [c_r - 1/2 log beta - (alpha_r + 1/2) log1p(kappa d^2 / (2 beta (kappa+1)))]/ln2)
//   A3/A4  lp_r = v_r + lg(1-H) + l_r/ln2  (lg(1-H) folded into the c_r table);
//       group max (order-preserving high word, REDUX), then sum_r 2^(lp_r - M)
//       (xor butterfly + fixed-order cross-warp sum: deterministic)
//   A5  growth:  v'_{r+1} = lp_r - M;  v'_0 = lg H - lg(1-H) + lg(sum);  the stored
//       posterior is UNNORMALISED and offset by -lg(1-H):
//       log R_t(r) = ln2 (v'_r + lg(1-H) - N_t),  N_t = lg sum_r 2^(v'_r + lg(1-H))
//   A6  MERGE: v'_{R-1} = lg(e_{R-2} + e_{R-1});  DROP: e_{R-1} is discarded
//   A7  r*, p_new = e_0 / sum (MERGE) or e_0 / (sum - e_{R-1}) (DROP), flags, events
// Every lp is also written to a per-series shared-memory row (double-buffered by
// step parity) so the O(1) special cells (R-2, R-1, 0, argmax) are read there
// by the tail lanes instead of being tracked per cell.
// State stays in registers for the whole call; x is staged per series in
// double-buffered shared-memory tiles by 1-D TMA bulk copies (cp.async.bulk +
// mbarrier); state is spilled to HBM (coalesced) once per call.
#pragma once

#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "fastmath.cuh"

namespace fbocd {

constexpr int kTile = 256;  // x steps per shared-memory tile (2 KB)
constexpr int kG = 4;       // cells per interleaved group in phase 1

struct SeriesScalars {  // per-series state carried between calls (HBM), 48 B
    double mu0, beta0;  // prior (set from x_0 when prior_first_obs)
    double n_prev;      // N_{t-1}: log2 sum_r 2^(v_r + log2(1-H)) of the stored v (log2 units)
    int32_t map_prev;   // r*_{t-1}
    int32_t ev_count;   // events appended since the last drain (may exceed capacity)
    int32_t flags;      // bit0: non-finite observation seen; bit1: bad prior
    int32_t pad;
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
    double l2H, l2mH, omH, theta, l2theta, alpha0, prior_cov;  // l2H = log2 H, l2mH = log2(1-H)
    int mode;  // 0 MERGE, 1 DROP
    int prior_first_obs;
    uint32_t ev_mask;
    int ev_cap;
    const double2* tab_ca;       // [R] {c_r / ln2 + log2(1-H), alpha_r}
    const double2* tab_gk;       // [R] {g_r, 1/(kappa_r+1)}
    const FastMathTables* fm;    // log / exp tables
    double* st_mu;               // [S][R] position order
    double* st_beta;
    double* st_v;
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
    int dbg;     // profiling experiments only (FALCON_BOCD_DEBUG): 1 no tail, 2 no barriers
};

template <int NT>
struct __align__(16) GroupSmem {
    double xbuf[2][kTile];
    unsigned long long red1[NT / 32 > 0 ? NT / 32 : 1];
    double red2[NT / 32 > 0 ? NT / 32 : 1];
    int redh[NT / 32 > 0 ? NT / 32 : 1];
    unsigned long long red3[NT / 32 > 0 ? NT / 32 : 1];  // on-demand argmax (event steps)
    double spec[4];                                       // dm of the cells r = R-2, R-1, 0
    double mu0, beta0, L0, n_prev;
    int map_prev, ev_count, flags, pad;
    unsigned long long mbar[2];
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

template <int NT>
__device__ __forceinline__ void group_sync(int g, int dbg = 0) {
    if (dbg == 2) return;
    if constexpr (NT == 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(NT) : "memory");
    }
}

// Order-preserving map of a non-NaN double to a signed 64-bit key.
__device__ __forceinline__ long long ord_key(double v) {
    long long b = __double_as_longlong(v);
    return b >= 0 ? b : (b ^ 0x7FFFFFFFFFFFFFFFLL);
}
__device__ __forceinline__ double ord_val(long long k) {
    long long b = k >= 0 ? k : (k ^ 0x7FFFFFFFFFFFFFFFLL);
    return __longlong_as_double(b);
}

// Biased (unsigned-ordered) argmax key: lp with its low 12 mantissa bits replaced by
// (4095 - r), so the max key is the max lp and, among (near-)ties, the smallest r.
__device__ __forceinline__ unsigned long long argmax_key(double lp, int r) {
    const long long k = (ord_key(lp) & ~0xFFFLL) | (0xFFF - r);
    return static_cast<unsigned long long>(k) ^ 0x8000000000000000ull;
}

template <int NT>
__device__ __forceinline__ void issue_tile_tma(GroupSmem<NT>& gs, const double* xrow, int k, int T) {
    const int base = k * kTile;
    const int n = min(kTile, T - base);
    fence_proxy_async();
    mbar_arrive_expect_tx(&gs.mbar[k & 1], unsigned(n) * 8u);
    tma_load_1d(gs.xbuf[k & 1], xrow + base, unsigned(n) * 8u, &gs.mbar[k & 1]);
}

__device__ __forceinline__ bool tile_tma_ok(const KParams& P, int k) {
    const int n = min(kTile, P.T - k * kTile);
    return P.tma_ok && ((n & 1) == 0);
}

// Shared memory of one CTA: tables, then per group: GroupSmem + the v row [R].
// TAB2: the per-r tables are stored twice (entries r and r+R) so the ring index
// (t - p) mod R becomes (t - p + R) with no masking and compile-time offsets per cell.
template <int NT>
__host__ __device__ constexpr size_t group_bytes(int R) {
    return sizeof(GroupSmem<NT>) + ((size_t(R) * sizeof(double) + 15) & ~size_t(15));  // keep 16-B alignment
}
__host__ __device__ constexpr size_t table_bytes(int R, bool tab2) {
    return size_t(R) * (tab2 ? 2 : 1) * 2 * sizeof(double2);
}

// order-preserving signed int of the high word of a double (for the shift M)
__device__ __forceinline__ int ord_hi(double v) {
    const int h = __double2hiint(v);
    return h ^ ((h >> 31) & 0x7FFFFFFF);
}
__device__ __forceinline__ double ord_hi_val(int oh) {
    return __hiloint2double(oh >= 0 ? oh : (oh ^ 0x7FFFFFFF), 0);
}

// Writes one cell of the register state under a lane predicate.  j is group-uniform,
// so the switch never diverges; the body is a handful of predicated moves.
template <int J>
__device__ __forceinline__ void set_cell_pred(double (&v)[J], double (&mu)[J], double (&be)[J], double (&L)[J],
                                              int j, bool pred, double vv, double m, double b, double l) {
#define FBOCD_SET(k)                      \
    case k:                               \
        if constexpr (J > k) {            \
            if (pred) {                   \
                v[k] = vv;                \
                mu[k] = m;                \
                be[k] = b;                \
                L[k] = l;                 \
            }                             \
        }                                 \
        break;
    switch (j) { FBOCD_SET(0) FBOCD_SET(1) FBOCD_SET(2) FBOCD_SET(3) FBOCD_SET(4) FBOCD_SET(5) FBOCD_SET(6) FBOCD_SET(7)
                 FBOCD_SET(8) FBOCD_SET(9) FBOCD_SET(10) FBOCD_SET(11) FBOCD_SET(12) FBOCD_SET(13) FBOCD_SET(14) FBOCD_SET(15) }
#undef FBOCD_SET
}
template <int J>
__device__ __forceinline__ void set_stats_pred(double (&mu)[J], double (&be)[J], double (&L)[J], int j, bool pred,
                                               double m, double b, double l) {
#define FBOCD_SETS(k)                     \
    case k:                               \
        if constexpr (J > k) {            \
            if (pred) {                   \
                mu[k] = m;                \
                be[k] = b;                \
                L[k] = l;                 \
            }                             \
        }                                 \
        break;
    switch (j) { FBOCD_SETS(0) FBOCD_SETS(1) FBOCD_SETS(2) FBOCD_SETS(3) FBOCD_SETS(4) FBOCD_SETS(5) FBOCD_SETS(6) FBOCD_SETS(7)
                 FBOCD_SETS(8) FBOCD_SETS(9) FBOCD_SETS(10) FBOCD_SETS(11) FBOCD_SETS(12) FBOCD_SETS(13) FBOCD_SETS(14) FBOCD_SETS(15) }
#undef FBOCD_SETS
}
template <int J>
__device__ __forceinline__ void set_v_pred(double (&v)[J], int j, bool pred, double vv) {
#define FBOCD_SETV(k)            \
    case k:                      \
        if constexpr (J > k) {   \
            if (pred) v[k] = vv; \
        }                        \
        break;
    switch (j) { FBOCD_SETV(0) FBOCD_SETV(1) FBOCD_SETV(2) FBOCD_SETV(3) FBOCD_SETV(4) FBOCD_SETV(5) FBOCD_SETV(6) FBOCD_SETV(7)
                 FBOCD_SETV(8) FBOCD_SETV(9) FBOCD_SETV(10) FBOCD_SETV(11) FBOCD_SETV(12) FBOCD_SETV(13) FBOCD_SETV(14) FBOCD_SETV(15) }
#undef FBOCD_SETV
}

// ---------------------------------------------------------------------------
// The kernel.
//   FULL : R == NT*J (power of two) at compile time;
//   TAB2 : doubled per-r tables (R <= 2048);
//   EAGER: the MAP run length r* is reduced every step (per-step MAP output or
//          MAPRESET events requested); otherwise it is computed on demand, from the
//          step's lp row in shared memory, only at steps that report an event.
// ---------------------------------------------------------------------------
template <int NT, int J, bool FULL, bool TAB2, bool EAGER, int SPB, int MINB>
__global__ void __launch_bounds__(NT* SPB, MINB) bocd_update_kernel(const KParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int R = FULL ? NT * J : P.R;
    const int RT = TAB2 ? 2 * R : R;
    double2* s_ca = reinterpret_cast<double2*>(smem_raw);
    double2* s_gk = s_ca + RT;
    unsigned char* gbase = reinterpret_cast<unsigned char*>(s_gk + RT);

    for (int k = threadIdx.x; k < RT; k += blockDim.x) {
        const int r = k < R ? k : k - R;
        s_ca[k] = P.tab_ca[r];
        s_gk[k] = P.tab_gk[r];
    }
    load_fastmath(P.fm);
    const int g = threadIdx.x / NT;
    const int i = threadIdx.x % NT;
    const int lane = threadIdx.x & 31;
    const int w = i >> 5;
    GroupSmem<NT>& gs = *reinterpret_cast<GroupSmem<NT>*>(gbase + size_t(g) * group_bytes<NT>(R));
    // the series' unnormalised log posterior v, in ring-position order (shared memory)
    double* vrow = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(&gs) + sizeof(GroupSmem<NT>));
    const int64_t s = int64_t(blockIdx.x) * SPB + g;
    const bool active = s < P.S;
    const double* xrow = P.x + (active ? s : 0) * P.ld;
    const int ntiles = (P.T + kTile - 1) / kTile;
    if (i == 0) {
        mbar_init(&gs.mbar[0], 1);
        mbar_init(&gs.mbar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (!active) return;

    // Prefetch tile 0 (TMA) as early as possible.
    if (i == 0 && ntiles > 0 && tile_tma_ok(P, 0)) issue_tile_tma<NT>(gs, xrow, 0, P.T);

    const double l2H = P.l2H, l2mH = P.l2mH;
    // ---- load or initialise the state ------------------------------------
    double mu[J], be[J], L[J];
    const int64_t sbase = s * int64_t(R);
    if (i == 0) {
        SeriesScalars sc = P.scal[s];
        if (P.t0 == 0) {
            if (P.prior_first_obs && P.T > 0) {
                const double x0 = xrow[0];
                sc.mu0 = x0;
                sc.beta0 = P.alpha0 * (P.prior_cov * x0) * (P.prior_cov * x0);
            }
            sc.n_prev = 0.0;
            sc.map_prev = 0;
        }
        const bool ok = sc.beta0 >= 2.2250738585072014e-308 && sc.beta0 < 1e300 && isfinite(sc.mu0);
        gs.mu0 = sc.mu0;
        gs.beta0 = ok ? sc.beta0 : 1.0;
        gs.L0 = fast_log2(gs.beta0);
        gs.n_prev = sc.n_prev;
        gs.map_prev = sc.map_prev;
        gs.ev_count = sc.ev_count;
        gs.flags = sc.flags | (ok ? 0 : 2);
    }
    group_sync<NT>(g);
    const double mu0 = gs.mu0, beta0 = gs.beta0, L0 = gs.L0;
    double n_prev = gs.n_prev;  // per-series scalars are group-uniform registers
    int map_prev = gs.map_prev, ev_count = gs.ev_count;
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int p = i + NT * j;
        if (FULL || p < R) {
            if (P.t0 == 0) {
                mu[j] = mu0;
                be[j] = beta0;
                L[j] = L0;
                vrow[p] = (p == 0) ? -l2mH : -INFINITY;
            } else {
                mu[j] = P.st_mu[sbase + p];
                be[j] = P.st_beta[sbase + p];
                vrow[p] = P.st_v[sbase + p];
                L[j] = fast_log2(be[j]);
            }
        } else {
            mu[j] = mu0;
            be[j] = beta0;
            L[j] = L0;
        }
    }

    const bool merge = (P.mode == 0);
    // argmax-eligible run lengths: MERGE r <= R-3 (slot R-1 is the bucket), DROP r <= R-2
    const int r_elig = merge ? R - 3 : R - 2;
    int tmod = int(P.t0 % R);  // ring bookkeeping: t mod R
    bool nonfinite = false;

    for (int k = 0; k < ntiles; ++k) {
        const int base = k * kTile;
        const int n = min(kTile, P.T - base);
        const int buf = k & 1;
        // prefetch the next tile into the other buffer (its previous readers all
        // passed at least one group barrier since their last read)
        if (i == 0 && k + 1 < ntiles && tile_tma_ok(P, k + 1)) issue_tile_tma<NT>(gs, xrow, k + 1, P.T);
        if (tile_tma_ok(P, k)) {
            mbar_wait(&gs.mbar[buf], unsigned(k >> 1) & 1u);
        } else {
            for (int q = i; q < n; q += NT) gs.xbuf[buf][q] = xrow[base + q];
            group_sync<NT>(g);
        }
        for (int q = 0; q < n; ++q) {
            const int tl = base + q;
            const int64_t t = P.t0 + tl;
            const double x = gs.xbuf[buf][q];
            // ---- phase 1: A1 + A2 + A3 ------------------------------------------
            const int ib = tmod - i + R;  // TAB2 index of cell j: ib - NT*j  (= (t - p) mod R, + R)
            double lp[J];
            // The cells are processed in groups of G with every stage written across the
            // group, so G independent log2 chains are in flight per thread (ILP).
#pragma unroll
            for (int j0 = 0; j0 < J; j0 += kG) {
                constexpr int G = (J < kG) ? J : kG;
                int idx[G];
                double bn[G], r[G], kd[G], pp[G];
                double2 tl2[G];
#pragma unroll
                for (int kk = 0; kk < G; ++kk) {  // A1: NIG update
                    const int j = j0 + kk;
                    const int p = i + NT * j;
                    if (TAB2) {
                        idx[kk] = ib - NT * j;
                    } else if (FULL) {
                        idx[kk] = (tmod - p) & (R - 1);
                    } else {
                        idx[kk] = tmod - p;
                        idx[kk] += (idx[kk] < 0) ? R : 0;
                    }
                    if (!FULL && p >= R) idx[kk] = 0;  // masked cell: any valid entry
                    const double2 gk = s_gk[idx[kk]];
                    const double d = x - mu[j];
                    bn[kk] = fma(gk.x * d, d, be[j]);
                    mu[j] = fma(d, gk.y, mu[j]);
                }
#pragma unroll
                for (int kk = 0; kk < G; ++kk) {  // fast_log2, staged: table entry
                    const int tb = __double2hiint(bn[kk]) + 0x00196000;
                    tl2[kk] = *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(g_fm.logtab) +
                                                                ((tb >> 9) & ((kLogTab - 1) << 4)));
                    const double invs = __hiloint2double(__double2hiint(tl2[kk].x) + 0x40000000 - (tb & 0xFFF00000),
                                                         __double2loint(tl2[kk].x));
                    r[kk] = fma(bn[kk], invs, -1.0);
                    kd[kk] = __hiloint2double(0x43300000, int(unsigned(tb) >> 20)) - c_fm[6];
                }
#pragma unroll
                for (int kk = 0; kk < G; ++kk) pp[kk] = fma(r[kk], c_fm[0], c_fm[1]);
#pragma unroll
                for (int kk = 0; kk < G; ++kk) pp[kk] = fma(pp[kk], r[kk], c_fm[2]);
#pragma unroll
                for (int kk = 0; kk < G; ++kk) pp[kk] = fma(pp[kk], r[kk], c_fm[3]);
#pragma unroll
                for (int kk = 0; kk < G; ++kk) pp[kk] = fma(pp[kk], r[kk], c_fm[4]);
#pragma unroll
                for (int kk = 0; kk < G; ++kk) pp[kk] = fma(pp[kk], r[kk], c_fm[5]);
#pragma unroll
                for (int kk = 0; kk < G; ++kk) {  // A2 + A3: predictive, joint with v
                    const int j = j0 + kk;
                    const int p = i + NT * j;
                    const double Ln = kd[kk] + fma(r[kk], pp[kk], tl2[kk].y);
                    const double2 ca = s_ca[idx[kk]];
                    const double ell = fma(-0.5, Ln, fma(ca.y, L[j] - Ln, ca.x));
                    be[j] = bn[kk];
                    L[j] = Ln;
                    lp[j] = ((FULL || p < R) ? vrow[p] : -INFINITY) + ell;
                }
            }
            // shift M (max over all cells, high word is enough) and, if EAGER, the argmax key
            int mh = INT_MIN;
            unsigned long long key = 0ull;  // below every real key (biased order)
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int p = i + NT * j;
                if (FULL || p < R) {
                    mh = max(mh, ord_hi(lp[j]));
                    if constexpr (EAGER) {
                        int r = tmod - p;
                        r += (r < 0) ? R : 0;
                        const unsigned long long kk = argmax_key(lp[j], r);
                        key = (r <= r_elig && kk > key) ? kk : key;
                    }
                }
            }
            // ---- group max (and argmax) ------------------------------------
            mh = __reduce_max_sync(0xffffffffu, mh);
            if constexpr (EAGER) {
                const unsigned hi = unsigned(key >> 32);
                const unsigned hmax = __reduce_max_sync(0xffffffffu, hi);
                const unsigned lmax = __reduce_max_sync(0xffffffffu, hi == hmax ? unsigned(key) : 0u);
                key = (static_cast<unsigned long long>(hmax) << 32) | lmax;
            }
            if constexpr (NT > 32) {
                if (lane == 0) {
                    gs.red1[w] = EAGER ? key : 0ull;
                    gs.redh[w] = mh;
                }
                group_sync<NT>(g, P.dbg);
#pragma unroll
                for (int ww = 0; ww < NT / 32; ++ww) {
                    mh = max(mh, gs.redh[ww]);
                    if constexpr (EAGER) {
                        const unsigned long long o = gs.red1[ww];
                        key = o > key ? o : key;
                    }
                }
            } else {
                group_sync<NT>(g);
            }
            const double M = ord_hi_val(mh);
            // ---- phase 2: exp + sum, growth (A4, A5): v'_{r+1} = lp_r - M ------------
            // (fast_exp2 staged across groups of G cells; summation order fixed: cell 0..J-1)
            double sum = 0.0;
#pragma unroll
            for (int j0 = 0; j0 < J; j0 += kG) {
                constexpr int G = (J < kG) ? J : kG;
                double xc[G], kd[G], rr[G], pp[G];
                int ki[G];
#pragma unroll
                for (int kk = 0; kk < G; ++kk) {
                    const int j = j0 + kk;
                    const int p = i + NT * j;
                    const double dm = lp[j] - M;
                    if (FULL || p < R) vrow[p] = dm;
                    // clamp >= -1021 on the high word only (fast_exp2)
                    const int xh = int(min(unsigned(__double2hiint(dm)), 0xC08FE800u));
                    xc[kk] = __hiloint2double(xh, __double2loint(dm));
                    const double zf = fma(xc[kk], c_fm[13], c_fm[7]);
                    ki[kk] = __double2loint(zf);
                    kd[kk] = zf - c_fm[7];
                }
#pragma unroll
                for (int kk = 0; kk < G; ++kk) rr[kk] = fma(kd[kk], c_fm[14], xc[kk]);
#pragma unroll
                for (int kk = 0; kk < G; ++kk) pp[kk] = fma(rr[kk], c_fm[8], c_fm[9]);
#pragma unroll
                for (int kk = 0; kk < G; ++kk) pp[kk] = fma(pp[kk], rr[kk], c_fm[10]);
#pragma unroll
                for (int kk = 0; kk < G; ++kk) pp[kk] = fma(pp[kk], rr[kk], c_fm[11]);
#pragma unroll
                for (int kk = 0; kk < G; ++kk) pp[kk] = fma(pp[kk], rr[kk], c_fm[12]);
#pragma unroll
                for (int kk = 0; kk < G; ++kk) {
                    const int j = j0 + kk;
                    const double qq = pp[kk] * rr[kk];
                    const double T = *reinterpret_cast<const double*>(reinterpret_cast<const char*>(g_fm.exptab) +
                                                                      ((ki[kk] << 3) & 0x1F8));
                    int th;
                    asm("mad.lo.s32 %0, %1, 1048576, %2;" : "=r"(th) : "r"(ki[kk] >> 6), "r"(__double2hiint(T)));
                    const double Ts = __hiloint2double(th, __double2loint(T));
                    const double e = fma(Ts, qq, Ts);
                    if (FULL || i + NT * j < R) sum += e;
                }
            }
            // the three cells the tail needs are published by their owners (the row entries of
            // pA / pB are overwritten by the fix-ups right after the barrier)
            const int pB = (tmod + 1 == R) ? 0 : tmod + 1;  // r = R-1 (recycled)
            const int pA = (pB + 1 == R) ? 0 : pB + 1;      // r = R-2
            if ((pA % NT) == i) gs.spec[0] = vrow[pA];
            if ((pB % NT) == i) gs.spec[1] = vrow[pB];
            if ((tmod % NT) == i) gs.spec[2] = vrow[tmod];
            if (P.dbg != 4) {  // dbg 4 (profiling experiment): no warp butterfly
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            }
            if constexpr (NT > 32) {
                if (lane == 0) gs.red2[w] = sum;
                group_sync<NT>(g, P.dbg);
                sum = gs.red2[0];
#pragma unroll
                for (int ww = 1; ww < NT / 32; ++ww) sum += gs.red2[ww];
            } else {
                group_sync<NT>(g);
            }
            if (P.dbg == 1) {  // profiling experiment: no tail
                tmod = (tmod + 1 == R) ? 0 : tmod + 1;
                continue;
            }
            // ---- the scalar tail (A5-A8), computed UNIFORMLY by every thread -------
            //   recycled cell pB (r = R-1) -> new CP cell: v = lg H - lg(1-H) + lg(sum), prior stats
            //   MERGE: cell pA (r = R-2) -> bucket: v = lg(2^dA + 2^dB) = mx + lg(1 + 2^(mn - mx))
            // (the owners write the new v of the two cells into the row and reset the CP cell's
            //  statistics; everyone else reads the pre-fix values from gs.spec)
            const double dA = gs.spec[0], dB = gs.spec[1], d0 = gs.spec[2];
            const double mx = fmax(dA, dB), mn = fmin(dA, dB);
            // one log stream for two values: lanes 0-15 lg(sum), lanes 16-31 lg(1 + u)
            const double u = fast_exp2(mx == -INFINITY ? -INFINITY : mn - mx);
            const double lgx = fast_log2(lane >= 16 ? 1.0 + u : sum);
            const double lg_sum = __shfl_sync(0xffffffffu, lgx, 0);
            const double lb = __shfl_sync(0xffffffffu, lgx, 16);
            const double vb = (mx == -INFINITY) ? -INFINITY : mx + lb;
            double Nt, eB = 0.0;
            bool prob;
            if (merge) {
                Nt = lg_sum;
                // p_new = R(1) / (1 - R(0)) = 2^(d0 - lg sum)  (R(0) = H exactly; R = 2: p_new = 1)
                prob = (R == 2) ? (1.0 > P.theta) : (d0 - lg_sum > P.l2theta);
            } else {
                eB = fast_exp2(dB);
                Nt = fast_log2(sum - P.omH * eB);
                prob = fast_exp2(d0) > P.theta * (sum - eB);  // p_new = e_0 / (sum - e_{R-1})
            }
            uint32_t fl = (t > 0 && prob) ? 1u : 0u;
            {
                const bool ownB = (pB % NT) == i;
                if (ownB) vrow[pB] = l2H - l2mH + lg_sum;
                if (merge && (pA % NT) == i) vrow[pA] = vb;
                set_stats_pred<J>(mu, be, L, pB / NT, ownB, mu0, beta0, L0);
            }
            if (!isfinite(x)) nonfinite = true;
            // ---- MAP run length r* (A7): eager (key reduced at barrier A) or on demand ----
            int r_ex = -1;
            if constexpr (EAGER) {
                if (key != 0ull) {
                    const long long sk = static_cast<long long>(key ^ 0x8000000000000000ull);
                    r_ex = int(0xFFF - (sk & 0xFFF));
                }
            } else if (fl & P.ev_mask) {  // group-uniform: an event at this step
                unsigned long long kb = 0ull;
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    const int p = i + NT * j;
                    if (FULL || p < R) {
                        int r = tmod - p;
                        r += (r < 0) ? R : 0;
                        const unsigned long long kk = argmax_key(vrow[p], r);  // dm: same order as lp
                        kb = (r <= r_elig && kk > kb) ? kk : kb;
                    }
                }
                const unsigned hi = unsigned(kb >> 32);
                const unsigned hmax = __reduce_max_sync(0xffffffffu, hi);
                const unsigned lmax = __reduce_max_sync(0xffffffffu, hi == hmax ? unsigned(kb) : 0u);
                kb = (static_cast<unsigned long long>(hmax) << 32) | lmax;
                if constexpr (NT > 32) {
                    if (lane == 0) gs.red3[w] = kb;
                    group_sync<NT>(g);
#pragma unroll
                    for (int ww = 0; ww < NT / 32; ++ww) {
                        const unsigned long long o = gs.red3[ww];
                        kb = o > kb ? o : kb;
                    }
                }
                if (kb != 0ull) {
                    const long long sk = static_cast<long long>(kb ^ 0x8000000000000000ull);
                    r_ex = int(0xFFF - (sk & 0xFFF));
                }
            }
            if (EAGER || (fl & P.ev_mask)) {
                int rstar;
                if (merge) {
                    // bucket vb vs the best growth slot d_ex (ties -> the smaller run length)
                    int pex = tmod - r_ex;
                    pex += (pex < 0) ? R : 0;
                    const double dex = r_ex >= 0 ? vrow[pex] : -INFINITY;
                    rstar = (r_ex < 0 || vb > dex) ? R - 1 : r_ex + 1;
                } else {
                    rstar = r_ex + 1;
                }
                if (EAGER && t > 0 && rstar < min(map_prev + 1, R - 1)) fl |= 2u;
                map_prev = rstar;
                if (i == 0 && P.out_map) P.out_map[s * P.ld_o + tl] = rstar;
                if (fl & P.ev_mask) {
                    const double pnew = merge ? (R == 2 ? 1.0 : fast_exp2(d0 - lg_sum))
                                              : fast_exp2(d0) * fast_rcp(sum - eB);
                    if (i == 0 && ev_count < P.ev_cap) {
                        EventRec ev;
                        ev.t = t;
                        ev.cp_index = t - rstar + 1;
                        ev.flags = fl;
                        ev.pad = 0;
                        ev.p_new = pnew;
                        P.ev[s * P.ev_cap + ev_count] = ev;
                    }
                    ++ev_count;
                }
            }
            if (i == 0) {
                if (P.out_pnew)
                    P.out_pnew[s * P.ld_o + tl] = merge ? (R == 2 ? 1.0 : fast_exp2(d0 - lg_sum))
                                                        : fast_exp2(d0) * fast_rcp(sum - eB);
                if (P.out_logz) P.out_logz[s * P.ld_o + tl] = LN2 * ((M - n_prev) + Nt);
            }
            n_prev = Nt;
            tmod = (tmod + 1 == R) ? 0 : tmod + 1;
        }
    }
    // ---- spill (with the pending fix-ups applied) ----------------------------
    group_sync<NT>(g);
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int p = i + NT * j;
        if (FULL || p < R) {
            P.st_mu[sbase + p] = mu[j];
            P.st_beta[sbase + p] = be[j];
            P.st_v[sbase + p] = vrow[p];
        }
    }
    if (i == 0) {
        SeriesScalars sc;
        sc.mu0 = gs.mu0;
        sc.beta0 = gs.beta0;
        sc.n_prev = n_prev;
        sc.map_prev = map_prev;
        sc.ev_count = ev_count;
        sc.flags = gs.flags | (nonfinite ? 1 : 0);
        sc.pad = 0;
        sc.pad2 = 0.0;
        P.scal[s] = sc;
        if (sc.flags) atomicOr(P.err, unsigned(sc.flags));
    }
}

}  // namespace fbocd
