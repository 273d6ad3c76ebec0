// acf.cu — ACF period detection and iteration times (§4.2,
// P:716-745), batched over series (ranks): one CTA per series.
//
// The centred codes y_t = x_t - mu (fp64) are staged in shared memory; thread k computes
// the lag sums sum_t y_t y_{t+k} for its lags with a sequential FMA over t (consecutive
// threads read consecutive y_{t+k}: conflict-free; y_t is a broadcast).  The period is the
// smallest lag whose ACF reaches M (block min-reduction).  L * k_max FP64 FMAs per series.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "../../include/falcon_bocd.h"

namespace {

constexpr int kMaxL = 8192;

__global__ void __launch_bounds__(256) acf_kernel(const int32_t* __restrict__ codes, int L, int64_t ld, int kmax,
                                                  double M, double* __restrict__ acf, int32_t* __restrict__ period) {
    extern __shared__ double y[];
    __shared__ double red[256];
    __shared__ int pmin;
    const int64_t s = blockIdx.x;
    const int32_t* x = codes + s * ld;
    // mu = sum / L: integer-exact sum (codes are int32, L <= 8192: |sum| < 2^44)
    long long part = 0;
    for (int t = threadIdx.x; t < L; t += blockDim.x) part += x[t];
    __shared__ long long ired[256];
    ired[threadIdx.x] = part;
    if (threadIdx.x == 0) pmin = INT_MAX;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) ired[threadIdx.x] += ired[threadIdx.x + o];
        __syncthreads();
    }
    const double mu = double(ired[0]) / double(L);
    double d2 = 0.0;
    for (int t = threadIdx.x; t < L; t += blockDim.x) {
        const double v = double(x[t]) - mu;
        y[t] = v;
        d2 = fma(v, v, d2);
    }
    red[threadIdx.x] = d2;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    const double den = red[0];
    for (int k = threadIdx.x + 1; k <= kmax; k += blockDim.x) {
        double num = 0.0;
        for (int t = 0; t + k < L; ++t) num = fma(y[t], y[t + k], num);
        const double a = den > 0.0 ? num / den : 0.0;  // zero variance -> 0 (reading A2)
        if (acf) acf[s * kmax + (k - 1)] = a;
        if (den > 0.0 && a >= M) atomicMin(&pmin, k);
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
    const size_t smem = size_t(L) * sizeof(double);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(acf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return FALCON_ECUDA;
    acf_kernel<<<unsigned(n_series), 256, smem, static_cast<cudaStream_t>(stream)>>>(codes_dev, L, ld, k_max, M,
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
