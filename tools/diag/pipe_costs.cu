// Microbenchmark: issue cost of I2F.F64 / SHFL.BFLY next to DFMA on sm_100a.
// Each kernel runs kIter iterations over 8 independent chains per thread; time with
// CUDA events, and run under ncu for pipe utilisation and shared-pipe wavefronts.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIter = 2048;
template <int MODE>
__global__ void __launch_bounds__(512) pipe_kernel(double* out, int salt) {
    double a[8];
    int k[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) { a[c] = 1.0 + (threadIdx.x + c) * 1e-9; k[c] = salt + c + threadIdx.x; }
    const double m = 0.999999, s = 1e-12;
#pragma unroll 2
    for (int it = 0; it < kIter; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (MODE == 0) {  // DFMA only
                a[c] = fma(a[c], m, s);
            } else if (MODE == 1) {  // I2F.F64 only (dependent through k)
                double f = __int2double_rn(k[c]);
                k[c] += __double2hiint(f) & 1;
                a[c] += 0.0;  // keep shape
            } else if (MODE == 2) {  // 1 I2F.F64 per 8 DFMA
                a[c] = fma(a[c], m, s);
                if (c == 0) a[c] = fma(__int2double_rn(k[c] + it), s, a[c]);
            } else if (MODE == 3) {  // SHFL.BFLY of a double per 8 DFMA
                a[c] = fma(a[c], m, s);
                if (c == 0) a[c] += __shfl_xor_sync(0xffffffffu, a[c], 1) * s;
            } else if (MODE == 4) {  // 2 I2F.F64 per DFMA (cell-like ratio x4)
                a[c] = fma(__int2double_rn(k[c] + it), s, a[c]);
            }
        }
    }
    double r = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) r += a[c] + k[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int MODE>
float run(double* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    pipe_kernel<MODE><<<148 * 2, 512>>>(out, 1);
    cudaEventRecord(e0);
    pipe_kernel<MODE><<<148 * 2, 512>>>(out, 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 2 * 512 * sizeof(double));
    const double warp_iters = 148.0 * 2 * 16 * kIter * 8;  // warp-level chain steps
    float t0 = run<0>(out), t1 = run<1>(out), t2 = run<2>(out), t3 = run<3>(out), t4 = run<4>(out);
    printf("ms dfma %.3f i2f %.3f dfma+i2f/8 %.3f dfma+shfl/8 %.3f i2f+dfma %.3f\n", t0, t1, t2, t3, t4);
    printf("ns per warp-op per SM: dfma %.4f i2f %.4f\n", t0 * 1e6 / (warp_iters / 148),
           t1 * 1e6 / (warp_iters / 148));
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
