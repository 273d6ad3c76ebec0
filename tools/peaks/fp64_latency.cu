// Microbenchmark: dependent DFMA latency and LDS latency on this B200 (one warp, clock64).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void dfma_lat(double* out, long long* cyc, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) x[k] = threadIdx.x + k;
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CH; ++k) x[k] = fma(x[k], a, b);
    }
    long long c1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; ++k) s += x[k];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
}
__global__ void lds_lat(double* out, long long* cyc, int iters) {
    __shared__ int buf[1024];
    for (int k = threadIdx.x; k < 1024; k += blockDim.x) buf[k] = (k + 1) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) p = buf[p];
    long long c1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
}
int main() {
    double* out; long long* cyc; long long h;
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
    const int it = 100000;
#define RUN(CH) dfma_lat<CH><<<1, 32>>>(out, cyc, it, 0.999999, 1e-9); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); \
    printf("DFMA chains/warp=%d: %.2f cycles per iteration (%.2f per DFMA)\n", CH, double(h) / it, double(h) / it / CH);
    RUN(1) RUN(2) RUN(4) RUN(8) RUN(16)
    lds_lat<<<1, 32>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS dependent chain: %.2f cycles per load\n", double(h) / it);
    return 0;
}
