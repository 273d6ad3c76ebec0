// Microbenchmark: latency of a warp-wide fp64 sum, (a) xor butterfly of SHFL + DADD (the
// update kernel's), (b) exact fixed-point sum with REDUX (max exponent, scale, F2I.S64, three
// 21-bit REDUX.SUM, recombine, I2F.S64).  One warp per SM, a dependent chain of kIter sums;
// clock64 per iteration.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int kIter = 4096;

__device__ __forceinline__ double sum_bfly(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double sum_redux(double v) {
    // v > 0 assumed; common scale from the warp's largest binary exponent
    const unsigned e = (unsigned(__double2hiint(v)) >> 20) & 0x7FF;
    const unsigned em = __reduce_max_sync(0xffffffffu, e);
    // scale by 2^(56 - (em - 1023)) exactly (exponent field add), convert
    const int sh = 56 - (int(em) - 1023);
    const double s = __hiloint2double(__double2hiint(v) + (sh << 20), __double2loint(v));
    const long long q = __double2ll_rn(s);
    const unsigned c0 = unsigned(q) & 0x1FFFFF, c1 = unsigned(q >> 21) & 0x1FFFFF, c2 = unsigned(q >> 42);
    const unsigned s0 = __reduce_add_sync(0xffffffffu, c0);
    const unsigned s1 = __reduce_add_sync(0xffffffffu, c1);
    const unsigned s2 = __reduce_add_sync(0xffffffffu, c2);
    const long long t = (long long)s0 + ((long long)s1 << 21) + ((long long)s2 << 42);
    const double r = __ll2double_rn(t);
    return __hiloint2double(__double2hiint(r) - (sh << 20), __double2loint(r));
}
template <int MODE>
__global__ void k(double* out, long long* cyc) {
    double v = 1.0 + threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < kIter; ++i) {
        const double s = MODE == 0 ? sum_bfly(v) : sum_redux(v);
        v = v + s * 1e-9;  // dependent chain
    }
    long long t1 = clock64();
    out[blockIdx.x * 32 + threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double* o; long long* c; long long h[148];
    cudaMalloc(&o, 148 * 32 * 8); cudaMalloc(&c, 148 * 8);
    for (int m = 0; m < 2; ++m) {
        for (int rep = 0; rep < 2; ++rep) {
            if (m == 0) k<0><<<148, 32>>>(o, c); else k<1><<<148, 32>>>(o, c);
            cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
        }
        printf("%s: %.1f clock64 ticks per warp sum\n", m == 0 ? "butterfly" : "redux", double(h[0]) / kIter);
    }
    return 0;
}
