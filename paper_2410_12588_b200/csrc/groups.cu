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

}  // namespace

extern "C" int falcon_classify_groups(const double* times_dev, int64_t n_batches, int32_t n_groups, int64_t ld,
                                      double factor, uint8_t* flags_dev, double* median_dev, void* stream) {
    if (n_batches < 0 || n_groups < 1 || n_groups > kMaxGroups || ld < n_groups || !(factor > 0.0))
        return FALCON_EINVAL;
    if (n_batches == 0) return FALCON_OK;
    if (!times_dev || !flags_dev || n_batches > 0x7FFFFFFF) return FALCON_EINVAL;
    int n2 = 1;
    while (n2 < n_groups) n2 <<= 1;
    const size_t smem = size_t(n2) * sizeof(double);
    const int threads = n2 >= 2048 ? 1024 : (n2 / 2 >= 32 ? n2 / 2 : 32);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(classify_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return FALCON_ECUDA;
    classify_kernel<<<unsigned(n_batches), threads, smem, static_cast<cudaStream_t>(stream)>>>(
        times_dev, n_groups, ld, factor, flags_dev, median_dev);
    return cudaGetLastError() == cudaSuccess ? FALCON_OK : FALCON_ECUDA;
}
