// tracegen.cu — device twin of paper_2410_12588_b200/tracegen.py (input generator only;
// none of the BOCD arithmetic lives here).  See include/falcon_trace.h.
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/falcon_trace.h"

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double uniform01(uint64_t k1, uint64_t t, uint64_t stream) {
    const uint64_t h = splitmix64(k1 ^ (t * 2ull + stream));
    return (double(h >> 11) + 0.5) * 0x1.0p-53;
}

__device__ __forceinline__ double std_normal(uint64_t k1, uint64_t t) {
    const double u1 = uniform01(k1, t, 0), u2 = uniform01(k1, t, 1);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

struct GenArgs {
    falcon_trace_spec spec;
    double* x;
    int64_t ld, s0, count, t0, T;
};

// One CTA per (series, column block); threads walk columns.  Episodes of the
// series are scanned per element (a handful per series).
__global__ void trace_kernel(const GenArgs a) {
    const int64_t i = blockIdx.y;
    const int64_t s = a.s0 + i;
    if (i >= a.count) return;
    const uint64_t k0 = splitmix64(a.spec.seed);
    const uint64_t k1 = splitmix64(k0 ^ uint64_t(s));
    const uint64_t ke = splitmix64(k0 ^ 0xFFFFFFFFFFFFFFFFull);
    const double b = a.spec.b[s], sg = a.spec.sigma[s];
    const int64_t e0 = a.spec.ep_off[s], e1 = a.spec.ep_off[s + 1];
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < a.T;
         j += int64_t(gridDim.x) * blockDim.x) {
        const int64_t t = a.t0 + j;
        double e = sg * std_normal(k1, uint64_t(t));
        if (a.spec.gamma != 0.0) e += a.spec.gamma * std_normal(ke, uint64_t(t));
        for (int64_t k = e0; k < e1; ++k)
            if (t >= a.spec.ep_start[k] && t < a.spec.ep_end[k]) e += a.spec.ep_logsev[k];
        a.x[i * a.ld + j] = b * exp(e);
    }
}

}  // namespace

extern "C" int falcon_trace_generate(const falcon_trace_spec* spec, double* x_dev, int64_t ld, int64_t s0,
                                     int64_t count, int64_t t0, int64_t T, void* stream) {
    if (!spec || (!x_dev && count > 0 && T > 0) || ld < T || s0 < 0 || count < 0 || t0 < 0 || T < 0 ||
        s0 + count > spec->n_series)
        return -1;
    if (count == 0 || T == 0) return 0;
    GenArgs a{*spec, x_dev, ld, s0, count, t0, T};
    dim3 block(256);
    int64_t gx = (T + 255) / 256;
    if (gx > 64) gx = 64;
    const dim3 grid = dim3(unsigned(gx), unsigned(count), 1u);
    if (count > 65535) {
        // split over series in slabs of 65535 rows (grid.y limit)
        for (int64_t c0 = 0; c0 < count; c0 += 65535) {
            GenArgs b = a;
            b.s0 = s0 + c0;
            b.count = (count - c0) < 65535 ? (count - c0) : 65535;
            b.x = x_dev + c0 * ld;
            trace_kernel<<<dim3(unsigned(gx), unsigned(b.count)), block, 0, (cudaStream_t)stream>>>(b);
        }
    } else {
        trace_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(a);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
