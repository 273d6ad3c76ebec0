// acf.cu — ACF period detection and iteration times (§4.2,
// P:716-745), batched over series (ranks): one CTA per series.
//
// The centred codes y_t = x_t - mu (fp64) are staged in shared memory, zero-padded past L so
// that every lag sum runs over the same t range without bounds checks.  The lag sums
// sum_t y_t y_{t+k} are register-blocked: a thread owns kLagBlk = 8 consecutive lags and one
// segment of t; per t it reads y_t (a warp broadcast) and one new y_{t+k+7} into a sliding
// window of 8 registers, so 2 shared loads feed 8 FMAs (8 independent accumulators: no
// dependent FMA chain).  The warp's lanes own consecutive lag blocks, whose window loads are
// 8 doubles apart; the array is stored with one double of padding every 16 (index i at
// i + i/16) so those loads hit 16 distinct 8-byte banks per half-warp.  The segments' partial
// sums are added in a fixed order (deterministic).  The period is the smallest lag whose ACF
// reaches M (block min-reduction).  sum_k (L - k) FP64 FMAs per series.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "../../include/falcon_bocd.h"

namespace {

constexpr int kMaxL = 8192;
constexpr int kLagBlk = 8;      // lags per thread
constexpr int kAcfThreads = 256;

__host__ __device__ constexpr int pad_idx(int i) { return i + (i >> 4); }

__global__ void __launch_bounds__(kAcfThreads) acf_kernel(const int32_t* __restrict__ codes, int L, int64_t ld,
                                                          int kmax, double M, double* __restrict__ acf,
                                                          int32_t* __restrict__ period) {
    extern __shared__ double smem_acf[];
    double* y = smem_acf;  // padded: y_t at pad_idx(t), zero for t >= L
    __shared__ double red[kAcfThreads];
    __shared__ int pmin;
    const int64_t s = blockIdx.x;
    const int32_t* x = codes + s * ld;
    // mu = sum / L: integer-exact sum (codes are int32, L <= 8192: |sum| < 2^44)
    long long part = 0;
    for (int t = threadIdx.x; t < L; t += blockDim.x) part += x[t];
    __shared__ long long ired[kAcfThreads];
    ired[threadIdx.x] = part;
    if (threadIdx.x == 0) pmin = INT_MAX;
    __syncthreads();
    for (int o = kAcfThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) ired[threadIdx.x] += ired[threadIdx.x + o];
        __syncthreads();
    }
    const double mu = double(ired[0]) / double(L);
    const int nblk = (kmax + kLagBlk - 1) / kLagBlk;    // lag blocks
    const int tpad = L + nblk * kLagBlk + kLagBlk;       // zero tail for the windows
    double d2 = 0.0;
    for (int t = threadIdx.x; t < tpad; t += blockDim.x) {
        const double v = t < L ? double(x[t]) - mu : 0.0;
        y[pad_idx(t)] = v;
        d2 = fma(v, v, d2);
    }
    red[threadIdx.x] = d2;
    __syncthreads();
    for (int o = kAcfThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    const double den = red[0];
    __syncthreads();  // red is reused for the segment partial sums below
    // lag blocks in passes of up to kAcfThreads blocks; the threads of a pass split t into
    // nseg segments (nseg = threads per lag block); red holds one lag's [nseg][nb] partials
    for (int b0 = 0; b0 < nblk; b0 += kAcfThreads) {
        const int nb = min(kAcfThreads, nblk - b0);
        const int nseg = max(1, kAcfThreads / nb);
        const int blk = threadIdx.x % nb;
        const int seg = threadIdx.x / nb;
        const int k0 = 1 + (b0 + blk) * kLagBlk;            // this thread's lags k0 .. k0+7
        const int seglen = (L + nseg - 1) / nseg;
        const int t0 = seg * seglen, t1 = min(L, t0 + seglen);
        double acc[kLagBlk], win[kLagBlk];
#pragma unroll
        for (int m = 0; m < kLagBlk; ++m) acc[m] = 0.0;
        if (seg < nseg && t0 < t1) {  // (the last segments may be empty for short L)
#pragma unroll
            for (int m = 0; m < kLagBlk - 1; ++m) win[m] = y[pad_idx(t0 + k0 + m)];
            for (int t = t0; t < t1; ++t) {
                win[kLagBlk - 1] = y[pad_idx(t + k0 + kLagBlk - 1)];
                const double yt = y[pad_idx(t)];
#pragma unroll
                for (int m = 0; m < kLagBlk; ++m) acc[m] = fma(yt, win[m], acc[m]);
#pragma unroll
                for (int m = 0; m < kLagBlk - 1; ++m) win[m] = win[m + 1];
            }
        }
        // segment partial sums -> fixed-order totals, one lag at a time through shared memory
#pragma unroll
        for (int m = 0; m < kLagBlk; ++m) {
            __syncthreads();
            if (seg < nseg) red[seg * nb + blk] = acc[m];
            __syncthreads();
            if (threadIdx.x < nb) {
                const int k = k0 + m;  // (threadIdx.x == blk here)
                double num = 0.0;
                for (int g = 0; g < nseg; ++g) num += red[g * nb + threadIdx.x];
                if (k <= kmax) {
                    const double a = den > 0.0 ? num / den : 0.0;  // zero variance -> 0 (reading A2)
                    if (acf) acf[s * kmax + (k - 1)] = a;
                    if (den > 0.0 && a >= M) atomicMin(&pmin, k);
                }
            }
        }
    }
    __syncthreads();
    // -1: zero-variance window, reported as a flag; 0: no lag reaches M (reading A3)
    if (threadIdx.x == 0) period[s] = den > 0.0 ? (pmin == INT_MAX ? 0 : pmin) : -1;
}

__global__ void iter_times_kernel(const double* __restrict__ ts, int64_t S, int n, int64_t ld,
                                  const int32_t* __restrict__ period, double* __restrict__ out, int64_t ld_out,
                                  int32_t* __restrict__ n_out) {
    const int64_t s = blockIdx.y;
    const int P = period[s];
    const int cnt = P > 0 ? (n - 1) / P : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) n_out[s] = cnt;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
        out[s * ld_out + i] = ts[s * ld + int64_t(i + 1) * P] - ts[s * ld + int64_t(i) * P];
}

}  // namespace

extern "C" int falcon_detect_period(const int32_t* codes_dev, int64_t n_series, int32_t L, int64_t ld, int32_t k_max,
                                    double M, double* acf_dev, int32_t* period_dev, void* stream) {
    // SPEC detect_period pre-condition |codes| >= 2 k_max: a shorter sequence is an
    // explicit insufficient-data error (the biased ACF numerator would have too few terms)
    if (n_series < 0 || L < 2 || L > kMaxL || ld < L || k_max < 1 || 2 * int64_t(k_max) > L || !(M > -1.0 && M <= 1.0))
        return FALCON_EINVAL;
    if (n_series == 0) return FALCON_OK;
    if (!codes_dev || !period_dev || n_series > 0x7FFFFFFF) return FALCON_EINVAL;
    const int nblk = (k_max + kLagBlk - 1) / kLagBlk;
    const size_t smem = size_t(pad_idx(L + nblk * kLagBlk + kLagBlk) + 1) * sizeof(double);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(acf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return FALCON_ECUDA;
    acf_kernel<<<unsigned(n_series), kAcfThreads, smem, static_cast<cudaStream_t>(stream)>>>(codes_dev, L, ld, k_max, M,
                                                                                     acf_dev, period_dev);
    return cudaGetLastError() == cudaSuccess ? FALCON_OK : FALCON_ECUDA;
}

extern "C" int falcon_iteration_times(const double* ts_dev, int64_t n_series, int32_t n, int64_t ld,
                                      const int32_t* period_dev, double* out_dev, int64_t ld_out, int32_t* n_out_dev,
                                      void* stream) {
    if (n_series < 0 || n < 1 || ld < n || ld_out < n - 1) return FALCON_EINVAL;
    if (n_series == 0) return FALCON_OK;
    if (!ts_dev || !period_dev || !out_dev || !n_out_dev || n_series > 65535) return FALCON_EINVAL;
    const dim3 grid = dim3(unsigned((n + 255) / 256), unsigned(n_series));
    iter_times_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(ts_dev, n_series, n, ld, period_dev,
                                                                           out_dev, ld_out, n_out_dev);
    return cudaGetLastError() == cudaSuccess ? FALCON_OK : FALCON_ECUDA;
}
