// groups.cu — suspicious-group classification (§4.3):
// per profiling round, the groups whose data-transfer time exceeds 1.1 x the median of all
// groups are suspicious.  One CTA per round: the times are sorted in shared memory (bitonic,
// padded to a power of two with +inf), the median is read off the sorted array, and every
// group is compared with factor x median (same operations as the oracle, bit-identical).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/falcon_bocd.h"

namespace {

constexpr int kMaxGroups = 8192;

__global__ void __launch_bounds__(1024) classify_kernel(const double* __restrict__ t, int G, int64_t ld,
                                                        double factor, uint8_t* __restrict__ flags,
                                                        double* __restrict__ med) {
    extern __shared__ double sv[];
    const int64_t b = blockIdx.x;
    const double* row = t + b * ld;
    int n2 = 1;
    while (n2 < G) n2 <<= 1;
    for (int k = threadIdx.x; k < n2; k += blockDim.x) sv[k] = k < G ? row[k] : __longlong_as_double(0x7FF0000000000000ll);
    __syncthreads();
    for (int size = 2; size <= n2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int k = threadIdx.x; k < n2 / 2; k += blockDim.x) {
                const int lo = 2 * k - (k & (stride - 1));  // first index of the compared pair
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const double a = sv[lo], c = sv[hi];
                if ((a > c) == up) {
                    sv[lo] = c;
                    sv[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    const double m = (G & 1) ? sv[G / 2] : (sv[G / 2 - 1] + sv[G / 2]) / 2.0;
    const double cut = factor * m;
    for (int k = threadIdx.x; k < G; k += blockDim.x) flags[b * G + k] = row[k] > cut ? 1 : 0;
    if (threadIdx.x == 0 && med) med[b] = m;
}

// Small rounds (G <= 64): one warp per round, the (padded) times sorted in registers by the
// same bitonic network with shuffles (element k = lane + 32 h, h < H), 8 rounds per CTA.
// The sorted values, and so the median and every flag, are those of classify_kernel.
template <int H>
__global__ void __launch_bounds__(256) classify_warp_kernel(const double* __restrict__ t, int64_t B, int G,
                                                             int64_t ld, double factor, uint8_t* __restrict__ flags,
                                                             double* __restrict__ med) {
    const int64_t b = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (b >= B) return;  // warp-uniform
    const int lane = threadIdx.x & 31;
    const double* row = t + b * ld;
    constexpr int n2 = 32 * H;
    const double inf = __longlong_as_double(0x7FF0000000000000ll);
    double x[H], v[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
        const int k = lane + 32 * h;
        x[h] = k < G ? row[k] : inf;
        v[h] = x[h];
    }
#pragma unroll
    for (int size = 2; size <= n2; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {  // H = 2, stride 32: the pair (k, k + 32) sits in one lane
                const bool up = (lane & size) == 0;
                const double a = v[0], c = v[1];
                if ((a > c) == up) {
                    v[0] = c;
                    v[1] = a;
                }
            } else {
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const int k = lane + 32 * h;
                    const double o = __shfl_xor_sync(0xffffffffu, v[h], stride);
                    const bool up = (k & size) == 0;
                    const bool low = (lane & stride) == 0;  // k is the pair's first index
                    // first index keeps the smaller value when ascending, the larger otherwise
                    const double mn = o < v[h] ? o : v[h], mx = o < v[h] ? v[h] : o;
                    v[h] = (low == up) ? mn : mx;
                }
            }
        }
    }
    // median: sorted element G/2 (and G/2 - 1 for even G) = lane (idx & 31) of v[idx >> 5]
    auto elem = [&](int idx) {
        const double e0 = __shfl_sync(0xffffffffu, v[0], idx & 31);
        const double e1 = H > 1 ? __shfl_sync(0xffffffffu, v[H - 1], idx & 31) : e0;
        return (idx >> 5) ? e1 : e0;
    };
    const double hi = elem(G / 2);
    const double lo = elem(G / 2 > 0 ? G / 2 - 1 : 0);
    const double m = (G & 1) ? hi : (lo + hi) / 2.0;
    const double cut = factor * m;
#pragma unroll
    for (int h = 0; h < H; ++h) {
        const int k = lane + 32 * h;
        if (k < G) flags[b * G + k] = x[h] > cut ? 1 : 0;
    }
    if (lane == 0 && med) med[b] = m;
}

}  // namespace

extern "C" int falcon_classify_groups(const double* times_dev, int64_t n_batches, int32_t n_groups, int64_t ld,
                                      double factor, uint8_t* flags_dev, double* median_dev, void* stream) {
    if (n_batches < 0 || n_groups < 1 || n_groups > kMaxGroups || ld < n_groups || !(factor > 0.0))
        return FALCON_EINVAL;
    if (n_batches == 0) return FALCON_OK;
    if (!times_dev || !flags_dev || n_batches > 0x7FFFFFFF) return FALCON_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n_groups <= 64) {  // one warp per round, 8 rounds per CTA
        const unsigned grid = unsigned((n_batches + 7) / 8);
        if (n_groups <= 32)
            classify_warp_kernel<1><<<grid, 256, 0, st>>>(times_dev, n_batches, n_groups, ld, factor, flags_dev,
                                                          median_dev);
        else
            classify_warp_kernel<2><<<grid, 256, 0, st>>>(times_dev, n_batches, n_groups, ld, factor, flags_dev,
                                                          median_dev);
        return cudaGetLastError() == cudaSuccess ? FALCON_OK : FALCON_ECUDA;
    }
    int n2 = 1;
    while (n2 < n_groups) n2 <<= 1;
    const size_t smem = size_t(n2) * sizeof(double);
    const int threads = n2 >= 2048 ? 1024 : (n2 / 2 >= 32 ? n2 / 2 : 32);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(classify_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return FALCON_ECUDA;
    classify_kernel<<<unsigned(n_batches), threads, smem, st>>>(
        times_dev, n_groups, ld, factor, flags_dev, median_dev);
    return cudaGetLastError() == cudaSuccess ? FALCON_OK : FALCON_ECUDA;
}
