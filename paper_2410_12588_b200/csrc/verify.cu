// verify.cu — change-point verification and fail-slow pairing.
//
// PAPER.md §4.2 "2) Change-point verification": BOCD's raw change points
// are checked by comparing the mean iteration time before and after each one; a
// difference below 10% is a jitter.  Verified degrade / recover change points are then
// paired into fail-slow events.  Readings V1-V5: include/falcon_bocd.h.
//
// Both steps are tiny next to the BOCD recursion (a few thousand events per C3 chunk):
// one thread per event for the verification (<= 2 x window fp64 loads, sums in index
// order so the means are bit-identical to the oracle's), one thread per series segment
// for the pairing state machine, then a tiled scan + gather that compacts the events in
// (series, onset) order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/falcon_bocd.h"

namespace {

__global__ void verify_kernel(const double* __restrict__ x, int64_t ld, int64_t n_series, int64_t sbase,
                              int64_t t_lo, int64_t T, const falcon_bocd_event* __restrict__ ev, int64_t n,
                              int window, double rel, falcon_verified_cp* __restrict__ out) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const falcon_bocd_event e = ev[k];
        falcon_verified_cp v;
        v.series = e.series;
        v.t = e.t;
        v.cp_index = e.cp_index;
        v.reserved = 0;
        v.mean_before = 0.0;
        v.mean_after = 0.0;
        const int64_t row = e.series - sbase;
        const int64_t b = e.cp_index;
        int64_t nb = b - t_lo < window ? b - t_lo : window;  // V1
        int64_t na = t_lo + T - b < window ? t_lo + T - b : window;
        if (row < 0 || row >= n_series) nb = na = 0;
        nb = nb < 0 ? 0 : nb;
        na = na < 0 ? 0 : na;
        v.n_before = int32_t(nb);
        v.n_after = int32_t(na);
        if (nb == 0 || na == 0) {
            v.status = FALCON_CP_INSUFFICIENT;  // V2
        } else {
            const double* xr = x + row * ld + (b - t_lo);
            double sb = 0.0, sa = 0.0;
            for (int64_t j = -nb; j < 0; ++j) sb += xr[j];  // V5: index order
            for (int64_t j = 0; j < na; ++j) sa += xr[j];
            const double mb = sb / double(nb), ma = sa / double(na);
            v.mean_before = mb;
            v.mean_after = ma;
            if (fabs(ma - mb) / mb < rel) {
                v.status = FALCON_CP_JITTER;  // V3, "less than 10%"
            } else {
                v.status = ma > mb ? FALCON_CP_DEGRADE : FALCON_CP_RECOVER;
            }
        }
        out[k] = v;
    }
}

// V4 for the series segment starting at k (first record of its series): outputs at
// tmp[k .. k + cnt[k]).  Non-start positions write cnt = 0.  Order violations set *bad.
__global__ void pair_segments_kernel(const falcon_verified_cp* __restrict__ v, int64_t n,
                                     falcon_failslow_event* __restrict__ tmp, int64_t* __restrict__ cnt,
                                     int* __restrict__ bad) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        cnt[k] = 0;
        const int64_t s = v[k].series;
        if (k > 0) {
            const int64_t sp = v[k - 1].series;
            if (sp > s || (sp == s && v[k - 1].t > v[k].t)) atomicOr(bad, 1);
            if (sp == s) continue;
        }
        int64_t m = 0, onset = 0;
        bool open = false;
        double base = 0.0, sev = 0.0;
        for (int64_t j = k; j < n && v[j].series == s; ++j) {
            const falcon_verified_cp& r = v[j];
            if (r.status == FALCON_CP_DEGRADE) {
                if (!open) {
                    open = true;
                    onset = r.cp_index;
                    base = r.mean_before;
                    sev = r.mean_after / r.mean_before;
                } else {
                    const double q = r.mean_after / base;
                    sev = q > sev ? q : sev;
                }
            } else if (r.status == FALCON_CP_RECOVER && open) {
                tmp[k + m++] = falcon_failslow_event{s, onset, r.cp_index, sev};
                open = false;
            }
        }
        if (open) tmp[k + m++] = falcon_failslow_event{s, onset, -1, sev};
        cnt[k] = m;
    }
}

// Exclusive scan of cnt[0..n) into off, total into *total: tiles of kScanTile counts (one
// per thread), per-tile sums (scan_tiles_kernel, pass 0), their exclusive scan in one CTA
// (scan_sums_kernel), then every tile rescanned with its offset (scan_tiles_kernel, pass 1).
constexpr int kScanTile = 1024;

// block-wide inclusive scan of one int64 per thread (1024 threads); returns the inclusive
// prefix, *tile_total = the tile's sum
__device__ int64_t block_scan_incl(int64_t v, int64_t* warp_sums, int64_t* tile_total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    if (lane == 31) warp_sums[w] = v;
    __syncthreads();
    if (w == 0) {
        int64_t s = warp_sums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t u = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += u;
        }
        warp_sums[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const int64_t r = v + (w > 0 ? warp_sums[w - 1] : 0);
    *tile_total = warp_sums[31];
    return r;
}

__global__ void __launch_bounds__(kScanTile) scan_tiles_kernel(const int64_t* __restrict__ cnt, int64_t n,
                                                                int64_t* __restrict__ tile_sum,
                                                                const int64_t* __restrict__ tile_off,
                                                                int64_t* __restrict__ off, int pass) {
    __shared__ int64_t ws[32];
    const int64_t k = int64_t(blockIdx.x) * kScanTile + threadIdx.x;
    const int64_t c = k < n ? cnt[k] : 0;
    int64_t tot;
    const int64_t incl = block_scan_incl(c, ws, &tot);
    if (pass == 0) {
        if (threadIdx.x == 0) tile_sum[blockIdx.x] = tot;
    } else if (k < n) {
        off[k] = tile_off[blockIdx.x] + incl - c;
    }
}

// exclusive scan of the nt tile sums in place (one CTA, kScanTile at a time), total -> *total
__global__ void __launch_bounds__(kScanTile) scan_sums_kernel(int64_t* __restrict__ s, int64_t nt,
                                                               int64_t* __restrict__ total) {
    __shared__ int64_t ws[32];
    int64_t carry = 0;
    for (int64_t base = 0; base < nt; base += kScanTile) {
        const int64_t k = base + threadIdx.x;
        const int64_t c = k < nt ? s[k] : 0;
        int64_t tot;
        const int64_t incl = block_scan_incl(c, ws, &tot);
        if (k < nt) s[k] = carry + incl - c;
        carry += tot;
        __syncthreads();  // ws is reused by the next tile
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void gather_kernel(const falcon_failslow_event* __restrict__ tmp, const int64_t* __restrict__ cnt,
                              const int64_t* __restrict__ off, int64_t n, falcon_failslow_event* __restrict__ out) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        for (int64_t m = 0; m < cnt[k]; ++m) out[off[k] + m] = tmp[k + m];
    }
}

unsigned grid_of(int64_t n) {
    int64_t g = (n + 255) / 256;
    return unsigned(std::max<int64_t>(1, std::min<int64_t>(g, 4096)));
}

}  // namespace

extern "C" int falcon_verify_changepoints(const double* x_dev, int64_t ld, int64_t n_series, int64_t series_base,
                                          int64_t t_lo, int64_t T, const falcon_bocd_event* ev_dev, int64_t n_ev,
                                          int32_t window, double rel_threshold, falcon_verified_cp* out_dev,
                                          void* stream) {
    if (n_ev < 0 || window < 1 || !(rel_threshold > 0.0) || n_series < 0 || T < 0 || ld < T) return FALCON_EINVAL;
    if (n_ev == 0) return FALCON_OK;
    if (!ev_dev || !out_dev || (!x_dev && n_series > 0 && T > 0)) return FALCON_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    verify_kernel<<<grid_of(n_ev), 256, 0, st>>>(x_dev, ld, n_series, series_base, t_lo, T, ev_dev, n_ev, window,
                                                 rel_threshold, out_dev);
    return cudaGetLastError() == cudaSuccess ? FALCON_OK : FALCON_ECUDA;
}

extern "C" int falcon_pair_failslow(const falcon_verified_cp* v_dev, int64_t n, falcon_failslow_event* out_dev,
                                    int64_t capacity, int64_t* n_out, void* stream) {
    if (n < 0 || capacity < 0 || !n_out) return FALCON_EINVAL;
    *n_out = 0;
    if (n == 0) return FALCON_OK;
    if (!v_dev) return FALCON_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // workspace: tmp [n] events, cnt [n], off [n], tile sums [nt], total, bad flag
    char* ws = nullptr;
    const int64_t nt = (n + kScanTile - 1) / kScanTile;
    const size_t b_tmp = size_t(n) * sizeof(falcon_failslow_event);
    const size_t b_i64 = size_t(n) * sizeof(int64_t);
    const size_t bytes = b_tmp + 2 * b_i64 + size_t(nt) * sizeof(int64_t) + 2 * sizeof(int64_t);
    if (cudaMallocAsync(reinterpret_cast<void**>(&ws), bytes, st) != cudaSuccess) return FALCON_ENOMEM;
    auto* tmp = reinterpret_cast<falcon_failslow_event*>(ws);
    auto* cnt = reinterpret_cast<int64_t*>(ws + b_tmp);
    auto* off = reinterpret_cast<int64_t*>(ws + b_tmp + b_i64);
    auto* tsum = reinterpret_cast<int64_t*>(ws + b_tmp + 2 * b_i64);
    auto* total = tsum + nt;
    auto* bad = reinterpret_cast<int*>(total + 1);
    int rc = FALCON_OK;
    int64_t h_total = 0;
    int h_bad = 0;
    cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), st);
    if (e == cudaSuccess) {
        pair_segments_kernel<<<grid_of(n), 256, 0, st>>>(v_dev, n, tmp, cnt, bad);
        scan_tiles_kernel<<<unsigned(nt), kScanTile, 0, st>>>(cnt, n, tsum, tsum, off, 0);
        scan_sums_kernel<<<1, kScanTile, 0, st>>>(tsum, nt, total);
        scan_tiles_kernel<<<unsigned(nt), kScanTile, 0, st>>>(cnt, n, tsum, tsum, off, 1);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_total, total, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        rc = FALCON_ECUDA;
    } else if (h_bad) {
        rc = FALCON_EINVAL;  // not in (series, t) order
    } else if (h_total > capacity || (h_total > 0 && !out_dev)) {
        *n_out = h_total;
        rc = FALCON_EINVAL;
    } else {
        if (h_total > 0) {
            gather_kernel<<<grid_of(n), 256, 0, st>>>(tmp, cnt, off, n, out_dev);
            e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        }
        if (e != cudaSuccess) rc = FALCON_ECUDA;
        *n_out = h_total;
    }
    cudaFreeAsync(ws, st);
    return rc;
}
