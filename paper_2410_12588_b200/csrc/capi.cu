// capi.cu — host runtime and C ABI of libfalcon_bocd.so (include/falcon_bocd.h).
//
// Owns: the per-R marginal-likelihood constant table (long double on the host,
// rounded once), the per-series state (mu, beta and the log-joint offset a of
// every cell in ring position order, plus SeriesScalars; bocd_kernel.cuh), the per-series event buffers, the
// host-staging buffers of update_chunk_host, and the drain / posterior-gather
// kernels.  Every computing entry point launches CUDA kernels; there is no CPU
// fallback.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/falcon_bocd.h"
#include "bocd_kernel.cuh"
#include "bocd_variants.h"

using fbocd::EventRec;
using fbocd::KParams;
using fbocd::SeriesScalars;

struct falcon_bocd_s {
    falcon_bocd_config cfg{};
    fbocd::Variant var{};
    size_t smem = 0;    // dynamic shared memory of the one-unit-per-CTA kernels
    size_t smem_p = 0;  // of the persistent kernels (+ the state prefetch buffers)
    int64_t grid_cap = 0;  // co-resident CTAs (persistent grid)
    size_t smem_w = 0;     // of the one-CTA-per-SM twins (var.fn_w), if any
    int n_sm = 0;          // multiprocessors of the device
    int per_sm = 0;        // co-resident one-unit CTAs per SM (regular kernels)
    int64_t t = 0;  // observations absorbed
    double c_bucket = 0.0;  // c_{R-1} / ln2 (the MERGE bucket's predictive constant)
    double2* d_ca = nullptr;
    double* d_y = nullptr;
    fbocd::FastMathTables* d_fm = nullptr;
    fbocd::CellTables* d_ct = nullptr;
    double* d_mu = nullptr;
    double* d_beta = nullptr;
    double* d_a = nullptr;  // log-joint offsets a [S][R] (bocd_kernel.cuh)
    double* d_w = nullptr;  // pending slot-0 weights [S][NT] (FULL kernels; 1 = none)
    SeriesScalars* d_scal = nullptr;
    EventRec* d_ev = nullptr;
    unsigned* d_err = nullptr;
    // drain scratch
    int32_t* d_off = nullptr;    // [S] offset of each series within its drain block
    int64_t* d_blk = nullptr;    // [nblk] drain block totals
    int32_t* d_blkovf = nullptr; // [nblk] drain block overflow bits
    int64_t* h_meta = nullptr;   // pinned, device-mapped [4]: total, overflow, error bits, drained
    falcon_bocd_event* d_evout = nullptr;
    int64_t evout_cap = 0;
    // host staging (update_chunk_host)
    double* d_stage[2] = {nullptr, nullptr};
    size_t stage_cap = 0;  // doubles per buffer
    int stage_idx = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_copied[2] = {nullptr, nullptr};
    cudaEvent_t ev_free[2] = {nullptr, nullptr};
    int32_t* d_omap = nullptr;
    double* d_opnew = nullptr;
    double* d_ologz = nullptr;
    size_t out_cap = 0;
    bool poisoned = false;
    int schedule = 0;  // falcon_bocd_set_schedule: 0 auto, 1 persistent, 2 one unit per CTA, 3 = 2 unbalanced
    std::string err;
};

namespace {

thread_local std::string g_create_err;

int fail(falcon_bocd_t h, int code, const std::string& msg) {
    if (h)
        h->err = msg;
    else
        g_create_err = msg;
    return code;
}

int cuda_fail(falcon_bocd_t h, cudaError_t e, const char* what) {
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    if (h) h->poisoned = true;
    return fail(h, e == cudaErrorMemoryAllocation ? FALCON_ENOMEM : FALCON_ECUDA, m);
}

#define CUDA_TRY(h, expr)                                   \
    do {                                                    \
        cudaError_t e_ = (expr);                            \
        if (e_ != cudaSuccess) return cuda_fail(h, e_, #expr); \
    } while (0)

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ---------------------------------------------------------------------------
// helper kernels
// ---------------------------------------------------------------------------
__global__ void init_scalars_kernel(SeriesScalars* scal, const double* mu0, const double* beta0, int64_t S,
                                    double omH) {
    for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < S; s += int64_t(gridDim.x) * blockDim.x) {
        SeriesScalars sc;
        sc.mu0 = mu0[s];
        sc.beta0 = beta0[s];
        sc.zd_prev = omH;
        sc.map_prev = 0;
        sc.ev_count = 0;
        sc.flags = 0;
        sc.dc = 0;
        sc.pad2 = 0.0;
        scal[s] = sc;
    }
}

// Before x_0 a segment starts with probability one (Q8): the cell at position 0 has
// q = 2^(a - alpha0 lg beta0) = 1, every other cell is impossible (a = -inf).
__global__ void init_state_kernel(double* mu, double* beta, double* a, const SeriesScalars* scal, int64_t S,
                                  int R, double alpha0) {
    const int64_t n = S * int64_t(R);
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t s = k / R;
        const int p = int(k - s * R);
        mu[k] = scal[s].mu0;
        beta[k] = scal[s].beta0;
        a[k] = (p == 0) ? alpha0 * log2(scal[s].beta0) : fbocd::kImpossible;
    }
}

__global__ void fill_kernel(double* v, int64_t n, double value) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
        v[k] = value;
}

// Event drain (falcon_bocd_changepoints[_async]): two launches, no host round trip between
// them.  drain_count_kernel: block b owns series [b*kDrainSpan, (b+1)*kDrainSpan); it writes
// each series' exclusive offset WITHIN the block (kept = min(count, cap)) and the block's
// total and overflow bit.  drain_gather_kernel: one warp per series adds the totals of the
// blocks before its own (a warp-parallel sum over at most ~100 block totals), copies the
// kept events in time order and resets the count; block 0 / warp 0 writes the meta record
// {total, overflow, sticky error bits, drained}.  When the total exceeds `capacity`, or a
// sticky error is set, nothing is copied or reset (meta.drained = 0).  out == nullptr:
// count only.
constexpr int kDrainThreads = 256;
constexpr int kDrainPer = 4;  // series per thread
constexpr int kDrainSpan = kDrainThreads * kDrainPer;

__global__ void __launch_bounds__(kDrainThreads) drain_count_kernel(const SeriesScalars* scal, int64_t S, int cap,
                                                                    int32_t* off_local, int64_t* blk_total,
                                                                    int32_t* blk_ovf) {
    __shared__ int32_t wsum[kDrainThreads / 32];
    const int64_t s0 = int64_t(blockIdx.x) * kDrainSpan + threadIdx.x * kDrainPer;
    int32_t kept[kDrainPer];
    int32_t loc = 0, ovf = 0;
#pragma unroll
    for (int k = 0; k < kDrainPer; ++k) {
        const int64_t s = s0 + k;
        const int c = s < S ? scal[s].ev_count : 0;
        kept[k] = c < cap ? c : cap;
        ovf |= c > cap;
        loc += kept[k];
    }
    // block-wide exclusive scan of loc: warp inclusive scan, then warp totals
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[w] = inc;
    const int any_ovf = __syncthreads_or(ovf);
    int32_t base = 0;
    for (int k = 0; k < w; ++k) base += wsum[k];
    int32_t run = base + inc - loc;
#pragma unroll
    for (int k = 0; k < kDrainPer; ++k) {
        if (s0 + k < S) off_local[s0 + k] = run;
        run += kept[k];
    }
    if (threadIdx.x == kDrainThreads - 1) {
        blk_total[blockIdx.x] = base + inc;
        blk_ovf[blockIdx.x] = any_ovf;
    }
}

__global__ void drain_gather_kernel(SeriesScalars* scal, const EventRec* ev, int64_t S, int cap,
                                    const int32_t* off_local, const int64_t* blk_total, const int32_t* blk_ovf,
                                    int nblk, const unsigned* err, int64_t capacity, falcon_bocd_event* out,
                                    int64_t* meta, int64_t series_base) {
    const int64_t s = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int my_blk = s < S ? int(s / kDrainSpan) : nblk;
    int64_t before = 0, total = 0;
    int ovf = 0;
    for (int b = lane; b < nblk; b += 32) {
        const int64_t v = blk_total[b];
        total += v;
        before += b < my_blk ? v : 0;
        ovf |= blk_ovf[b];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        total += __shfl_xor_sync(0xffffffffu, total, o);
        before += __shfl_xor_sync(0xffffffffu, before, o);
        ovf |= __shfl_xor_sync(0xffffffffu, ovf, o);
    }
    const unsigned e = *err;
    const bool drain = out != nullptr && total <= capacity && (e & 7u) == 0u;
    if (s == 0 && lane == 0) {
        meta[0] = total;
        meta[1] = ovf;
        meta[2] = e;
        meta[3] = drain ? 1 : 0;
    }
    if (!drain || s >= S) return;
    const int c = scal[s].ev_count;
    const int n = c < cap ? c : cap;
    const int64_t o = before + off_local[s];
    for (int k = lane; k < n; k += 32) {
        const EventRec r = ev[s * int64_t(cap) + k];
        falcon_bocd_event q;
        q.series = series_base + s;
        q.t = r.t;
        q.cp_index = r.cp_index;
        q.flags = r.flags;
        q.reserved = 0;
        q.p_new = r.p_new;
        out[o + k] = q;
    }
    __syncwarp();
    if (lane == 0) scal[s].ev_count = 0;
}

// Ring position order -> run-length order; R_t(r) = q_r (1-H) / Zd_t with the cell's
// q_r = w 2^(a + G_r - alpha_r lg beta - Dc) (bocd_kernel.cuh), G_r / alpha_r from the
// kernel table (row r-1 = {G_r, alpha_r}; G_0 = 0, alpha_0 = alpha0).  FULL kernels (w != null):
// the pending weight w of thread i applies to its slot 0, position i + NT phi.
__global__ void posterior_kernel(const double* mu, const double* beta, const double* a, const double* w, int nt,
                                 const double2* ca, double alpha0, const SeriesScalars* scal, int64_t s0,
                                 int64_t count, int R, int64_t t, double omH, double* logR_out, double* mu_out,
                                 double* beta_out) {
    const int64_t n = count * int64_t(R);
    const int tm = int(t % R);
    const int phi = w ? ((tm + 1 == R) ? 0 : tm + 1) / nt : 0;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = k / R;
        const int r = int(k - i * R);
        int p = tm - r;
        if (p < 0) p += R;
        const int64_t src = (s0 + i) * int64_t(R) + p;
        if (logR_out) {
            const SeriesScalars& sc = scal[s0 + i];
            const double G = r ? ca[r - 1].x : 0.0;
            const double al = r ? ca[r - 1].y : alpha0;
            double lq = (a[src] + G) - al * log2(beta[src]) - double(sc.dc);
            if (w && p / nt == phi) lq += log2(w[(s0 + i) * nt + p % nt]);
            // impossible cells carry a = kImpossible (or -inf): log R = -inf
            logR_out[k] = lq < -262144.0 ? -INFINITY : 0.6931471805599453 * lq + log(omH / sc.zd_prev);
        }
        if (mu_out) mu_out[k] = mu[src];
        if (beta_out) beta_out[k] = beta[src];
    }
}

int grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    if (g > 148 * 32) g = 148 * 32;
    if (g < 1) g = 1;
    return int(g);
}

int check_sticky(falcon_bocd_t h, cudaStream_t st) {
    unsigned e = 0;
    CUDA_TRY(h, cudaMemcpyAsync(&e, h->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    if (e & 1u) {
        h->poisoned = true;
        return fail(h, FALCON_ENONFINITE, "non-finite observation seen (NaN/Inf in x)");
    }
    if (e & 2u) {
        h->poisoned = true;
        return fail(h, FALCON_ENONFINITE, "non-finite or non-positive prior (beta0 <= 0, or first observation 0)");
    }
    if (e & 4u) {  // the kernel's entry check of its shared-memory layout (bocd_kernel.cuh, kFmBase)
        h->poisoned = true;
        return fail(h, FALCON_ECUDA, "internal: dynamic shared memory not at the expected address");
    }
    return FALCON_OK;
}

// Binds the handle's device for the duration of one entry point and restores the caller's
// current device on every return path.
struct DeviceGuard {
    int prev = -1;
    int set(falcon_bocd_t h) {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
        if (prev == h->cfg.device) return FALCON_OK;
        CUDA_TRY(h, cudaSetDevice(h->cfg.device));
        return FALCON_OK;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

int falcon_bocd_abi_version(void) { return FALCON_BOCD_ABI_VERSION; }

int falcon_bocd_config_init(falcon_bocd_config* cfg) {
    if (!cfg) return FALCON_EINVAL;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->n_series = 1;
    cfg->R = 1024;
    cfg->hazard = 1.0 / 250.0;
    cfg->kappa0 = 1.0;
    cfg->alpha0 = 1.0;
    cfg->mu0_scalar = 0.0;
    cfg->beta0_scalar = 1.0;
    cfg->prior_first_obs = 0;
    cfg->prior_cov = 0.05;
    cfg->threshold = 0.9;
    cfg->trunc_mode = FALCON_TRUNC_MERGE;
    cfg->event_mask = FALCON_EV_PROB;
    cfg->event_capacity = 64;
    cfg->device = 0;
    cfg->series_base = 0;
    return FALCON_OK;
}

int falcon_bocd_predictive_constants(int32_t R, double kappa0, double alpha0, double* c, double* a, double* g,
                                     double* k1) {
    if (R < 1 || !(kappa0 > 0.0) || !(alpha0 > 0.0) || !std::isfinite(kappa0) || !std::isfinite(alpha0))
        return FALCON_EINVAL;
    // D_r = lgamma(alpha_r + 1/2) - lgamma(alpha_r) by the half-step recurrence
    // D(alpha + 1/2) = log(alpha) - D(alpha) (from Gamma(alpha + 1) = alpha Gamma(alpha)),
    // started from lgammal at alpha0: no cancellation between large lgamma values.
    long double D = lgammal((long double)alpha0 + 0.5L) - lgammal((long double)alpha0);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (int r = 0; r < R; ++r) {
        const long double kap = (long double)kappa0 + r;
        const long double alp = (long double)alpha0 + 0.5L * r;
        const long double kp1 = kap + 1.0L;
        if (c) c[r] = (double)(D - 0.5L * logl(two_pi * kp1 / kap));
        if (a) a[r] = (double)alp;
        if (g) g[r] = (double)(kap / (2.0L * kp1));
        if (k1) k1[r] = (double)(1.0L / kp1);
        D = logl(alp) - D;
    }
    return FALCON_OK;
}

int falcon_bocd_create(const falcon_bocd_config* cfg, falcon_bocd_t* out) {
    g_create_err.clear();
    if (!cfg || !out) return fail(nullptr, FALCON_EINVAL, "null argument");
    *out = nullptr;
    const falcon_bocd_config& c = *cfg;
    if (c.n_series < 1) return fail(nullptr, FALCON_EINVAL, "n_series must be >= 1");
    if (c.R < 2 || c.R > 4096) return fail(nullptr, FALCON_EINVAL, "R must be in [2, 4096]");
    if (!(c.hazard > 0.0 && c.hazard < 1.0)) return fail(nullptr, FALCON_EINVAL, "hazard must be in (0, 1)");
    if (!(c.kappa0 > 0.0) || !(c.alpha0 > 0.0) || !std::isfinite(c.kappa0) || !std::isfinite(c.alpha0))
        return fail(nullptr, FALCON_EINVAL, "kappa0 and alpha0 must be finite and > 0");
    if (c.trunc_mode != FALCON_TRUNC_MERGE && c.trunc_mode != FALCON_TRUNC_DROP)
        return fail(nullptr, FALCON_EINVAL, "trunc_mode must be MERGE or DROP");
    if (c.event_capacity < 1) return fail(nullptr, FALCON_EINVAL, "event_capacity must be >= 1");
    if (c.series_base < 0) return fail(nullptr, FALCON_EINVAL, "series_base must be >= 0");
    if (!std::isfinite(c.threshold)) return fail(nullptr, FALCON_EINVAL, "threshold must be finite");
    if (c.prior_first_obs && !(c.prior_cov > 0.0 && std::isfinite(c.prior_cov)))
        return fail(nullptr, FALCON_EINVAL, "prior_cov must be finite and > 0");
    if (!c.prior_first_obs && !c.beta0 && !(c.beta0_scalar > 0.0 && std::isfinite(c.beta0_scalar)))
        return fail(nullptr, FALCON_EINVAL, "beta0 must be finite and > 0");
    if (!c.prior_first_obs && !c.mu0 && !std::isfinite(c.mu0_scalar))
        return fail(nullptr, FALCON_EINVAL, "mu0 must be finite");
    const int64_t S = c.n_series;
    std::vector<double> mu0(S), beta0(S);
    for (int64_t s = 0; s < S; ++s) {
        mu0[s] = c.mu0 ? c.mu0[s] : c.mu0_scalar;
        beta0[s] = c.beta0 ? c.beta0[s] : c.beta0_scalar;
        if (!c.prior_first_obs && (!std::isfinite(mu0[s]) || !(beta0[s] > 0.0) || !std::isfinite(beta0[s])))
            return fail(nullptr, FALCON_EINVAL, "per-series mu0 must be finite and beta0 > 0");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, FALCON_ECUDA, "no CUDA device available (this library has no CPU fallback)");
    }
    if (c.device < 0 || c.device >= ndev) return fail(nullptr, FALCON_EINVAL, "device ordinal out of range");

    falcon_bocd_t h = new falcon_bocd_s();
    h->cfg = c;
    h->cfg.mu0 = nullptr;
    h->cfg.beta0 = nullptr;
    if (fbocd::select_variant(c.R, c.trunc_mode, c.alpha0, &h->var) != 0) {
        delete h;
        return fail(nullptr, FALCON_EINVAL, "no kernel variant for this R");
    }
    h->smem = fbocd::variant_smem(h->var, c.R, false);
    h->smem_p = fbocd::variant_smem(h->var, c.R, true);
    auto bail = [&](int code) {
        g_create_err = h->err;
        falcon_bocd_destroy(h);
        return code;
    };
    int rc;
    DeviceGuard guard;
    if ((rc = guard.set(h)) != 0) return bail(rc);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, c.device) != cudaSuccess || prop.major < 10) {
        cudaGetLastError();
        h->err = "device is not sm_100 class (this library is built for sm_100a only)";
        return bail(FALCON_ECUDA);
    }
    if (h->smem_p > 227 * 1024) {
        h->err = "shared memory footprint too large";
        return bail(FALCON_EINVAL);
    }
    if (fbocd::upload_fastmath_constants() != 0) {
        h->err = "cudaMemcpyToSymbol(c_fm) failed";
        return bail(FALCON_ECUDA);
    }
    h->n_sm = prop.multiProcessorCount;
    for (const void* fn : {h->var.fn, h->var.fn_eager}) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(h->smem));
        if (e != cudaSuccess) return bail(cuda_fail(h, e, "cudaFuncSetAttribute"));
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, h->var.nt * h->var.spb, h->smem);
        if (e != cudaSuccess || per_sm < 1) return bail(cuda_fail(h, e != cudaSuccess ? e : cudaErrorInvalidConfiguration,
                                                               "occupancy query"));
        h->per_sm = h->per_sm ? std::min(h->per_sm, per_sm) : per_sm;
    }
    if (h->var.fn_w) {
        // the balanced wave assumes exactly one CTA per SM (registers: NT * spb_w threads x up
        // to 128 fill the register file); otherwise the twins are not used
        h->smem_w = fbocd::variant_smem_wide(h->var, c.R);
        for (const void* fn : {h->var.fn_w, h->var.fn_eager_w}) {
            cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(h->smem_w));
            if (e != cudaSuccess) return bail(cuda_fail(h, e, "cudaFuncSetAttribute"));
            int per_sm = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, h->var.nt * h->var.spb_w, h->smem_w);
            if (e != cudaSuccess) return bail(cuda_fail(h, e, "occupancy query"));
            if (per_sm != 1) h->var.fn_w = h->var.fn_eager_w = nullptr;
        }
    }
    for (const void* fn : {h->var.fn_p, h->var.fn_eager_p}) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(h->smem_p));
        if (e != cudaSuccess) return bail(cuda_fail(h, e, "cudaFuncSetAttribute"));
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, h->var.nt * h->var.spb, h->smem_p);
        if (e != cudaSuccess || per_sm < 1) return bail(cuda_fail(h, e != cudaSuccess ? e : cudaErrorInvalidConfiguration,
                                                               "occupancy query"));
        // persistent grid: as many CTAs as are co-resident (the kernel loops over series units)
        const int64_t cap = int64_t(per_sm) * prop.multiProcessorCount;
        h->grid_cap = h->grid_cap ? std::min(h->grid_cap, cap) : cap;
    }

    const int R = c.R;
    std::vector<double> tc(R), ta(R), tg(R), tk(R);
    falcon_bocd_predictive_constants(R, c.kappa0, c.alpha0, tc.data(), ta.data(), tg.data(), tk.data());
    std::vector<double2> ca(R);
    {
        // base-2 units: row r holds {G_{r+1}, alpha_{r+1}} with G_n the data-independent part
        // of the log2 NIG marginal likelihood of n observations (bocd_kernel.cuh, A2),
        // G_{r+1} = G_r + c_r / ln2 (c_r: the Student-t constant), G_0 = 0
        const long double inv_ln2 = 1.442695040888963407359924681001892137L;
        long double D = lgammal((long double)c.alpha0 + 0.5L) - lgammal((long double)c.alpha0);
        const long double two_pi = 6.283185307179586476925286766559005768L;
        long double G = 0.0L;
        for (int r = 0; r < R; ++r) {
            const long double kap = (long double)c.kappa0 + r;
            const long double cr = D - 0.5L * logl(two_pi * (kap + 1.0L) / kap);
            G += cr * inv_ln2;
            if (r == R - 1) h->c_bucket = (double)(cr * inv_ln2);
            ca[r] = make_double2((double)G, (double)((long double)c.alpha0 + 0.5L * (r + 1)));
            D = logl((long double)c.alpha0 + 0.5L * r) - D;
        }
    }
    fbocd::FastMathTables fmt;
    fbocd::fill_fastmath_tables(&fmt);
    std::vector<fbocd::CellTables> cellt(1);
    fbocd::fill_cell_tables(cellt.data());
    const size_t SR = size_t(S) * size_t(R);
    double *dmu0 = nullptr, *dbeta0 = nullptr;
#define ALLOC(ptr, bytes)                                                   \
    do {                                                                    \
        cudaError_t e2 = cudaMalloc((void**)&(ptr), (bytes));               \
        if (e2 != cudaSuccess) {                                            \
            cudaFree(dmu0);                                                 \
            cudaFree(dbeta0);                                               \
            return bail(cuda_fail(h, e2, "cudaMalloc " #ptr));              \
        }                                                                   \
    } while (0)
    ALLOC(h->d_ca, R * sizeof(double2));
    ALLOC(h->d_y, R * sizeof(double));
    ALLOC(h->d_fm, sizeof(fbocd::FastMathTables));
    ALLOC(h->d_ct, sizeof(fbocd::CellTables));
    ALLOC(h->d_mu, SR * sizeof(double));
    ALLOC(h->d_beta, SR * sizeof(double));
    ALLOC(h->d_a, SR * sizeof(double));
    ALLOC(h->d_w, size_t(S) * h->var.nt * sizeof(double));
    ALLOC(h->d_scal, S * sizeof(SeriesScalars));
    ALLOC(h->d_ev, size_t(S) * c.event_capacity * sizeof(EventRec));
    ALLOC(h->d_err, sizeof(unsigned));
    ALLOC(h->d_off, S * sizeof(int32_t));
    ALLOC(h->d_blk, ((S + kDrainSpan - 1) / kDrainSpan) * sizeof(int64_t));
    ALLOC(h->d_blkovf, ((S + kDrainSpan - 1) / kDrainSpan) * sizeof(int32_t));
    ALLOC(dmu0, S * sizeof(double));
    ALLOC(dbeta0, S * sizeof(double));
#undef ALLOC
    cudaError_t e3 = cudaHostAlloc((void**)&h->h_meta, 4 * sizeof(int64_t), cudaHostAllocMapped);
    if (e3 != cudaSuccess) h->h_meta = nullptr;
    if (e3 == cudaSuccess) e3 = cudaMemcpy(h->d_ca, ca.data(), R * sizeof(double2), cudaMemcpyHostToDevice);
    if (e3 == cudaSuccess) e3 = cudaMemcpy(h->d_y, tk.data(), R * sizeof(double), cudaMemcpyHostToDevice);
    if (e3 == cudaSuccess) e3 = cudaMemcpy(h->d_fm, &fmt, sizeof(fmt), cudaMemcpyHostToDevice);
    if (e3 == cudaSuccess) e3 = cudaMemcpy(h->d_ct, cellt.data(), sizeof(fbocd::CellTables), cudaMemcpyHostToDevice);
    if (e3 == cudaSuccess) e3 = cudaMemcpy(dmu0, mu0.data(), S * sizeof(double), cudaMemcpyHostToDevice);
    if (e3 == cudaSuccess) e3 = cudaMemcpy(dbeta0, beta0.data(), S * sizeof(double), cudaMemcpyHostToDevice);
    if (e3 == cudaSuccess) e3 = cudaMemset(h->d_err, 0, sizeof(unsigned));
    if (e3 == cudaSuccess) {
        init_scalars_kernel<<<grid_for(S, 256), 256>>>(h->d_scal, dmu0, dbeta0, S, 1.0 - c.hazard);
        init_state_kernel<<<grid_for(int64_t(SR), 256), 256>>>(h->d_mu, h->d_beta, h->d_a, h->d_scal, S, R,
                                                               c.alpha0);
        fill_kernel<<<grid_for(S * h->var.nt, 256), 256>>>(h->d_w, S * h->var.nt, 1.0);
        e3 = cudaGetLastError();
    }
    if (e3 == cudaSuccess) e3 = cudaDeviceSynchronize();
    cudaFree(dmu0);
    cudaFree(dbeta0);
    if (e3 != cudaSuccess) return bail(cuda_fail(h, e3, "create: init"));
    *out = h;
    return FALCON_OK;
}

// Calls of at most this many steps run the persistent kernels (bocd_kernel.cuh, PERSIST).
constexpr int64_t kPersistMaxSteps = 64;

static int launch_update(falcon_bocd_t h, const double* x_dev, int64_t ld, int64_t T,
                         int32_t* omap, double* opnew, double* ologz, int64_t ld_o, cudaStream_t st) {
    const falcon_bocd_config& c = h->cfg;
    int64_t done = 0;
    while (done < T) {
        const int64_t n = (T - done) > (1 << 30) ? (1 << 30) : (T - done);
        KParams P;
        std::memset(&P, 0, sizeof(P));
        P.R = c.R;
        P.S = c.n_series;
        P.H = c.hazard;
        P.omH = 1.0 - c.hazard;
        P.ln_omH = log1p(-c.hazard);
        P.c_bucket = h->c_bucket;
        P.al2_bucket = 2.0 * c.alpha0 + double(c.R - 1);
        P.a2p1 = int(std::floor(2.0 * c.alpha0)) + 1;  // FULL kernels: 2 alpha_{r+1} = (a2p1 + r) + f2
        P.f2 = 2.0 * c.alpha0 - std::floor(2.0 * c.alpha0);
        P.hr = (double)((long double)c.hazard / (1.0L - (long double)c.hazard));
        P.theta = c.threshold;
        P.alpha0 = c.alpha0;
        P.prior_cov = c.prior_cov;
        P.mode = c.trunc_mode;
        P.prior_first_obs = c.prior_first_obs;
        P.ev_mask = c.event_mask;
        P.ev_cap = c.event_capacity;
        P.tab_ca = h->d_ca;
        P.tab_y = h->d_y;
        P.fm = h->d_fm;
        P.ct = h->d_ct;
        P.st_mu = h->d_mu;
        P.st_beta = h->d_beta;
        P.st_a = h->d_a;
        P.st_w = h->d_w;
        P.scal = h->d_scal;
        P.ev = h->d_ev;
        P.err = h->d_err;
        P.x = x_dev + done;
        P.ld = ld;
        P.T = int(n);
        P.t0 = h->t;
        P.out_map = omap ? omap + done : nullptr;
        P.out_pnew = opnew ? opnew + done : nullptr;
        P.out_logz = ologz ? ologz + done : nullptr;
        P.ld_o = ld_o;
        P.tma_ok = ((reinterpret_cast<uintptr_t>(P.x) & 15u) == 0) && ((ld & 1) == 0);
        const int64_t units = (c.n_series + h->var.spb - 1) / h->var.spb;
        // streaming calls (few steps): persistent grid, tables set up once per CTA and the next
        // unit's state prefetched; long calls: one unit per CTA.  Identical arithmetic.
        const bool persist = h->schedule == 1 ? n <= kPersistMaxSteps
                           : h->schedule >= 2 ? false
                                              : (n <= kPersistMaxSteps && units > h->grid_cap);
        // one wave that would load SMs unevenly (at most spb * ceil(units / #SM) series per SM
        // in CTAs of spb): one balanced CTA per SM instead, ceil(S / #SM) series at most
        const int64_t S = c.n_series, nsm = h->n_sm;
        const bool wide = !persist && h->var.fn_w && h->schedule != 3 && units <= nsm * h->per_sm &&
                          S <= nsm * h->var.spb_w &&
                          (S + nsm - 1) / nsm < int64_t(h->var.spb) * ((units + nsm - 1) / nsm);
        const int64_t grid = persist ? h->grid_cap : wide ? std::min(nsm, S) : units;
        void* args[] = {&P};
        // r* every step only when it is an output (per-step MAP, MAPRESET events); otherwise
        // r* = 1 at every PROB event (theta >= 1/2).
        // theta < 1/2 also needs it at PROB events (bocd_kernel.cuh: r* = 1 only for theta >= 1/2)
        const bool eager = (c.event_mask & FALCON_EV_MAPRESET) || omap || c.threshold < 0.5;
        const void* fn = persist ? (eager ? h->var.fn_eager_p : h->var.fn_p)
                       : wide    ? (eager ? h->var.fn_eager_w : h->var.fn_w)
                                 : (eager ? h->var.fn_eager : h->var.fn);
        cudaError_t e = cudaLaunchKernel(fn, dim3(unsigned(grid)),
                                         dim3(unsigned(h->var.nt * (wide ? h->var.spb_w : h->var.spb))), args,
                                         persist ? h->smem_p : wide ? h->smem_w : h->smem, st);
        if (e != cudaSuccess) return cuda_fail(h, e, "bocd_update_kernel launch");
        h->t += n;
        done += n;
    }
    return FALCON_OK;
}

int falcon_bocd_update_chunk(falcon_bocd_t h, const double* x_dev, int64_t ld, int64_t T,
                             const falcon_bocd_step_out* outs, void* stream) {
    if (!h) return FALCON_EINVAL;
    if (h->poisoned) return fail(h, FALCON_ESTATE, "handle poisoned by an earlier error");
    if (T < 0 || ld < T || (T > 0 && !x_dev)) return fail(h, FALCON_EINVAL, "bad x / ld / T");
    if (outs && outs->ld < T && (outs->map_rl || outs->p_new || outs->log_z))
        return fail(h, FALCON_EINVAL, "outs->ld < T");
    if (T == 0) return FALCON_OK;
    int rc;
    DeviceGuard guard;
    if ((rc = guard.set(h)) != 0) return rc;
    return launch_update(h, x_dev, ld, T, outs ? outs->map_rl : nullptr, outs ? outs->p_new : nullptr,
                         outs ? outs->log_z : nullptr, outs ? outs->ld : 0, (cudaStream_t)stream);
}

int falcon_bocd_update_chunk_host(falcon_bocd_t h, const double* x_host, int64_t ld, int64_t T,
                                  const falcon_bocd_step_out* outs, void* stream) {
    if (!h) return FALCON_EINVAL;
    if (h->poisoned) return fail(h, FALCON_ESTATE, "handle poisoned by an earlier error");
    if (T < 0 || ld < T || (T > 0 && !x_host)) return fail(h, FALCON_EINVAL, "bad x / ld / T");
    const bool want_out = outs && (outs->map_rl || outs->p_new || outs->log_z);
    if (want_out && outs->ld < T) return fail(h, FALCON_EINVAL, "outs->ld < T");
    if (T == 0) return FALCON_OK;
    int rc;
    DeviceGuard guard;
    if ((rc = guard.set(h)) != 0) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t S = h->cfg.n_series;
    const size_t need = size_t(S) * size_t(T);
    if (!h->copy_stream) {
        CUDA_TRY(h, cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_copied[b], cudaEventDisableTiming));
            CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_free[b], cudaEventDisableTiming));
        }
    }
    if (need > h->stage_cap) {
        CUDA_TRY(h, cudaDeviceSynchronize());
        for (int b = 0; b < 2; ++b) {
            cudaFree(h->d_stage[b]);
            h->d_stage[b] = nullptr;
        }
        h->stage_cap = 0;
        for (int b = 0; b < 2; ++b) CUDA_TRY(h, cudaMalloc((void**)&h->d_stage[b], need * sizeof(double)));
        h->stage_cap = need;
    }
    const int b = h->stage_idx;
    h->stage_idx ^= 1;
    // copy x (pitched host rows -> dense device rows) on the copy stream once the buffer is free
    CUDA_TRY(h, cudaStreamWaitEvent(h->copy_stream, h->ev_free[b], 0));
    CUDA_TRY(h, cudaMemcpy2DAsync(h->d_stage[b], size_t(T) * sizeof(double), x_host, size_t(ld) * sizeof(double),
                                  size_t(T) * sizeof(double), size_t(S), cudaMemcpyHostToDevice, h->copy_stream));
    CUDA_TRY(h, cudaEventRecord(h->ev_copied[b], h->copy_stream));
    CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_copied[b], 0));
    int32_t* omap = nullptr;
    double *opnew = nullptr, *ologz = nullptr;
    if (want_out) {
        if (need > h->out_cap) {
            CUDA_TRY(h, cudaStreamSynchronize(st));
            cudaFree(h->d_omap);
            cudaFree(h->d_opnew);
            cudaFree(h->d_ologz);
            h->d_omap = nullptr;
            h->d_opnew = h->d_ologz = nullptr;
            h->out_cap = 0;
            CUDA_TRY(h, cudaMalloc((void**)&h->d_omap, need * sizeof(int32_t)));
            CUDA_TRY(h, cudaMalloc((void**)&h->d_opnew, need * sizeof(double)));
            CUDA_TRY(h, cudaMalloc((void**)&h->d_ologz, need * sizeof(double)));
            h->out_cap = need;
        }
        omap = outs->map_rl ? h->d_omap : nullptr;
        opnew = outs->p_new ? h->d_opnew : nullptr;
        ologz = outs->log_z ? h->d_ologz : nullptr;
    }
    if ((rc = launch_update(h, h->d_stage[b], T, T, omap, opnew, ologz, T, st)) != 0) return rc;
    CUDA_TRY(h, cudaEventRecord(h->ev_free[b], st));
    if (want_out) {
        const size_t hp = size_t(outs->ld);
        if (omap)
            CUDA_TRY(h, cudaMemcpy2DAsync(outs->map_rl, hp * 4, omap, size_t(T) * 4, size_t(T) * 4, size_t(S),
                                          cudaMemcpyDeviceToHost, st));
        if (opnew)
            CUDA_TRY(h, cudaMemcpy2DAsync(outs->p_new, hp * 8, opnew, size_t(T) * 8, size_t(T) * 8, size_t(S),
                                          cudaMemcpyDeviceToHost, st));
        if (ologz)
            CUDA_TRY(h, cudaMemcpy2DAsync(outs->log_z, hp * 8, ologz, size_t(T) * 8, size_t(T) * 8, size_t(S),
                                          cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaStreamSynchronize(st));
    }
    // the caller may reuse x_host once the copy has landed
    CUDA_TRY(h, cudaEventSynchronize(h->ev_copied[b]));
    return FALCON_OK;
}

// Copies the drained records from the device staging buffer to page-locked host memory as
// contiguous 8-byte words (coalesced writes over the host link; the gather kernel's
// per-record 40-byte scatter would be many small host transactions).
__global__ void drain_copyout_kernel(const unsigned long long* src, unsigned long long* dst, const int64_t* meta) {
    if (!meta[3]) return;
    const int64_t n = meta[0] * int64_t(sizeof(falcon_bocd_event) / 8);
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
        dst[k] = src[k];
}

// Enqueues the two drain kernels (count, then gather into `out` unless out == nullptr);
// meta (device-accessible int64 [4]) receives {total, overflow, error bits, drained}.
// host_out: `out` is page-locked host memory, reached through the device staging buffer
// and drain_copyout_kernel.
static int enqueue_drain(falcon_bocd_t h, falcon_bocd_event* out, int64_t capacity, int64_t* meta,
                         cudaStream_t st, bool host_out = false) {
    const int64_t S = h->cfg.n_series;
    const int cap = h->cfg.event_capacity;
    const int nblk = int((S + kDrainSpan - 1) / kDrainSpan);
    drain_count_kernel<<<nblk, kDrainThreads, 0, st>>>(h->d_scal, S, cap, h->d_off, h->d_blk, h->d_blkovf);
    CUDA_TRY(h, cudaGetLastError());
    const int64_t threads = S * 32;
    falcon_bocd_event* dst = out;
    if (host_out && capacity > 0) {
        const int64_t need = std::min<int64_t>(capacity, S * int64_t(cap));
        if (need > h->evout_cap) {
            CUDA_TRY(h, cudaStreamSynchronize(st));
            cudaFree(h->d_evout);
            h->d_evout = nullptr;
            h->evout_cap = 0;
            CUDA_TRY(h, cudaMalloc((void**)&h->d_evout, size_t(need) * sizeof(falcon_bocd_event)));
            h->evout_cap = need;
        }
        dst = h->d_evout;
    }
    drain_gather_kernel<<<unsigned((threads + 255) / 256), 256, 0, st>>>(
        h->d_scal, h->d_ev, S, cap, h->d_off, h->d_blk, h->d_blkovf, nblk, h->d_err, capacity, dst, meta,
        h->cfg.series_base);
    CUDA_TRY(h, cudaGetLastError());
    if (host_out && capacity > 0) {
        drain_copyout_kernel<<<148, 256, 0, st>>>(reinterpret_cast<const unsigned long long*>(dst),
                                                  reinterpret_cast<unsigned long long*>(out), meta);
        CUDA_TRY(h, cudaGetLastError());
    }
    return FALCON_OK;
}

// Memory the drain kernels may write: device / managed memory, or page-locked host memory
// (mapped into the device address space under UVA).
static bool device_writable(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged ||
           (a.type == cudaMemoryTypeHost && a.devicePointer == p);
}

static int sticky_status(falcon_bocd_t h, int64_t e) {
    if (e & 1) {
        h->poisoned = true;
        return fail(h, FALCON_ENONFINITE, "non-finite observation seen (NaN/Inf in x)");
    }
    if (e & 2) {
        h->poisoned = true;
        return fail(h, FALCON_ENONFINITE, "non-finite or non-positive prior (beta0 <= 0, or first observation 0)");
    }
    if (e & 4) {
        h->poisoned = true;
        return fail(h, FALCON_ECUDA, "internal: dynamic shared memory not at the expected address");
    }
    return FALCON_OK;
}

int falcon_bocd_pending_events(falcon_bocd_t h, int64_t* n_out, void* stream) {
    if (!h || !n_out) return FALCON_EINVAL;
    if (!h->h_meta) return fail(h, FALCON_ENOMEM, "no drain mailbox");
    DeviceGuard g;
    int rc;
    if ((rc = g.set(h)) != 0) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if ((rc = enqueue_drain(h, nullptr, 0, h->h_meta, st)) != 0) return rc;
    CUDA_TRY(h, cudaStreamSynchronize(st));
    *n_out = h->h_meta[0];
    return FALCON_OK;
}

int falcon_bocd_changepoints(falcon_bocd_t h, falcon_bocd_event* out, int64_t capacity, int64_t* n_out,
                             void* stream) {
    if (!h || !n_out || capacity < 0 || (capacity > 0 && !out)) return FALCON_EINVAL;
    if (!h->h_meta) return fail(h, FALCON_ENOMEM, "no drain mailbox");
    *n_out = 0;
    DeviceGuard g;
    int rc;
    if ((rc = g.set(h)) != 0) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    // device memory: the gather kernel writes there directly; page-locked host memory: gathered
    // on the device and copied out by a kernel (one synchronisation either way); pageable host
    // memory: staged through the device buffer and copied after the count is known
    cudaPointerAttributes pa;
    bool dev_out = false, pinned_out = false;
    if (capacity > 0) {
        if (cudaPointerGetAttributes(&pa, out) == cudaSuccess) {
            dev_out = pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged;
            pinned_out = pa.type == cudaMemoryTypeHost && pa.devicePointer == out;
        } else {
            cudaGetLastError();
        }
    }
    const bool direct = dev_out || pinned_out;
    falcon_bocd_event* dst = out;
    if (capacity > 0 && !direct) {
        const int64_t need = std::min<int64_t>(capacity, h->cfg.n_series * int64_t(h->cfg.event_capacity));
        if (need > h->evout_cap) {
            CUDA_TRY(h, cudaStreamSynchronize(st));
            cudaFree(h->d_evout);
            h->d_evout = nullptr;
            h->evout_cap = 0;
            CUDA_TRY(h, cudaMalloc((void**)&h->d_evout, size_t(need) * sizeof(falcon_bocd_event)));
            h->evout_cap = need;
        }
        dst = h->d_evout;
    }
    if ((rc = enqueue_drain(h, capacity > 0 ? dst : nullptr, capacity, h->h_meta, st, pinned_out)) != 0) return rc;
    CUDA_TRY(h, cudaStreamSynchronize(st));
    const int64_t total = h->h_meta[0], ovf = h->h_meta[1], err = h->h_meta[2];
    if ((rc = sticky_status(h, err)) != 0) return rc;
    if (total > capacity) {
        *n_out = total;
        return fail(h, FALCON_EINVAL, "output capacity smaller than the number of buffered events");
    }
    if (total > 0 && !direct) {
        CUDA_TRY(h, cudaMemcpyAsync(out, dst, size_t(total) * sizeof(falcon_bocd_event), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaStreamSynchronize(st));
    }
    *n_out = total;
    if (ovf) {
        h->err = "event buffer overflow: some events were dropped";
        return FALCON_WARN_EVENTS_DROPPED;
    }
    return FALCON_OK;
}

int falcon_bocd_changepoints_async(falcon_bocd_t h, falcon_bocd_event* out, int64_t capacity, int64_t* meta,
                                   void* stream) {
    if (!h || !meta || capacity < 0 || (capacity > 0 && !out)) return FALCON_EINVAL;
    if (h->poisoned) return fail(h, FALCON_ESTATE, "handle poisoned by an earlier error");
    DeviceGuard g;
    int rc;
    if ((rc = g.set(h)) != 0) return rc;
    if (!device_writable(meta) || (capacity > 0 && !device_writable(out)))
        return fail(h, FALCON_EINVAL, "out / meta must be device memory or page-locked host memory");
    bool host_out = false;
    if (capacity > 0) {
        cudaPointerAttributes pa;
        host_out = cudaPointerGetAttributes(&pa, out) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
    }
    return enqueue_drain(h, capacity > 0 ? out : nullptr, capacity, meta, (cudaStream_t)stream, host_out);
}

int falcon_bocd_read_posterior(falcon_bocd_t h, int64_t s0, int64_t count, double* logR_out, double* mu_out,
                               double* beta_out, void* stream) {
    if (!h || s0 < 0 || count < 0 || s0 + count > h->cfg.n_series) return FALCON_EINVAL;
    if (count == 0 || (!logR_out && !mu_out && !beta_out)) return FALCON_OK;
    int rc;
    DeviceGuard guard;
    if ((rc = guard.set(h)) != 0) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if ((rc = check_sticky(h, st)) != 0) return rc;
    const int R = h->cfg.R;
    const size_t n = size_t(count) * R;
    double* outs[3] = {logR_out, mu_out, beta_out};
    double* dst[3] = {nullptr, nullptr, nullptr};
    double* tmp = nullptr;
    bool any_host = false;
    for (int k = 0; k < 3; ++k)
        if (outs[k] && !is_device_ptr(outs[k])) any_host = true;
    if (any_host) CUDA_TRY(h, cudaMalloc((void**)&tmp, 3 * n * sizeof(double)));
    for (int k = 0; k < 3; ++k) {
        if (!outs[k]) continue;
        dst[k] = is_device_ptr(outs[k]) ? outs[k] : tmp + k * n;
    }
    posterior_kernel<<<grid_for(int64_t(n), 256), 256, 0, st>>>(h->d_mu, h->d_beta, h->d_a,
                                                                h->var.full ? h->d_w : nullptr, h->var.nt,
                                                                h->d_ca, h->cfg.alpha0,
                                                                h->d_scal, s0, count, R, h->t, 1.0 - h->cfg.hazard,
                                                                dst[0], dst[1], dst[2]);
    cudaError_t e = cudaGetLastError();
    for (int k = 0; k < 3 && e == cudaSuccess; ++k)
        if (outs[k] && dst[k] != outs[k])
            e = cudaMemcpyAsync(outs[k], dst[k], n * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (tmp) cudaFree(tmp);
    if (e != cudaSuccess) return cuda_fail(h, e, "read_posterior");
    return FALCON_OK;
}

int falcon_bocd_set_schedule(falcon_bocd_t h, int32_t schedule) {
    if (!h || schedule < 0 || schedule > 3) return FALCON_EINVAL;
    h->schedule = schedule;
    return FALCON_OK;
}

int falcon_bocd_steps(falcon_bocd_t h, int64_t* t_out) {
    if (!h || !t_out) return FALCON_EINVAL;
    *t_out = h->t;
    return FALCON_OK;
}

int falcon_bocd_kernel_shape(falcon_bocd_t h, int32_t* nt, int32_t* j, int32_t* spb) {
    if (!h) return FALCON_EINVAL;
    if (nt) *nt = h->var.nt;
    if (j) *j = h->var.j;
    if (spb) *spb = h->var.spb;
    return FALCON_OK;
}

int falcon_bocd_destroy(falcon_bocd_t h) {
    if (!h) return FALCON_OK;
    int rc = FALCON_OK;
    DeviceGuard guard;
    if (guard.set(h) == FALCON_OK) {
        if (cudaDeviceSynchronize() != cudaSuccess) rc = FALCON_ECUDA;
        if (rc == FALCON_OK && h->d_err) {
            unsigned e = 0;
            if (cudaMemcpy(&e, h->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost) == cudaSuccess && (e & 7u))
                rc = (e & 3u) ? FALCON_ENONFINITE : FALCON_ECUDA;
        }
    }
    cudaGetLastError();
    void* ptrs[] = {h->d_ca, h->d_y, h->d_fm, h->d_ct, h->d_mu, h->d_beta, h->d_a, h->d_w, h->d_scal, h->d_ev, h->d_err, h->d_off,
                    h->d_blk, h->d_blkovf, h->d_evout, h->d_stage[0], h->d_stage[1], h->d_omap, h->d_opnew, h->d_ologz};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (int b = 0; b < 2; ++b) {
        if (h->ev_copied[b]) cudaEventDestroy(h->ev_copied[b]);
        if (h->ev_free[b]) cudaEventDestroy(h->ev_free[b]);
    }
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    if (h->h_meta) cudaFreeHost(h->h_meta);
    delete h;
    return rc;
}

const char* falcon_bocd_last_error(falcon_bocd_t h) { return h ? h->err.c_str() : g_create_err.c_str(); }

int falcon_bocd_debug_fastmath(int32_t which, const double* in_dev, double* out_dev, int64_t n, void* stream) {
    if (which < 0 || which > 4 || n < 0 || (n > 0 && (!in_dev || !out_dev))) return FALCON_EINVAL;
    if (n == 0) return FALCON_OK;
    fbocd::FastMathTables fmt;
    fbocd::fill_fastmath_tables(&fmt);
    std::vector<fbocd::CellTables> cellt(1);
    fbocd::fill_cell_tables(cellt.data());
    fbocd::FastMathTables* d = nullptr;
    fbocd::CellTables* dc = nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    if (fbocd::upload_fastmath_constants() != 0) return FALCON_ECUDA;
    if (cudaMalloc((void**)&d, sizeof(fmt)) != cudaSuccess) return FALCON_ENOMEM;
    if (cudaMalloc((void**)&dc, sizeof(fbocd::CellTables)) != cudaSuccess) {
        cudaFree(d);
        return FALCON_ENOMEM;
    }
    cudaError_t e = cudaMemcpyAsync(d, &fmt, sizeof(fmt), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dc, cellt.data(), sizeof(fbocd::CellTables), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && fbocd::launch_fastmath_probe(which, in_dev, out_dev, n, d, dc, st) != 0)
        e = cudaErrorLaunchFailure;
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d);
    cudaFree(dc);
    return e == cudaSuccess ? FALCON_OK : FALCON_ECUDA;
}

}  // extern "C"
