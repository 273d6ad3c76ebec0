// P0 microbenchmark: FP64 pipe peak on this B200 (DFMA throughput with every SM saturated),
// plus the throughput of libdevice log/exp in fp64.  Output: one JSON object on stdout.
// The SM clock during the DFMA loop is sampled by nvidia-smi (tools/peaks/p0.py), which
// turns the rate into DFMA per clock per SM (clock64 deltas do not give the SM clock here).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

// 8 independent DFMA chains per thread, ITERS iterations each.
__global__ void dfma_kernel(double* out, int iters, double a, double b,
                            unsigned long long* cyc) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  unsigned long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  unsigned long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

template <int OP>
__global__ void transc_kernel(double* out, int iters, double seed) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = seed + 1e-3 * (threadIdx.x + k);
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double y = OP == 0 ? log(x[k]) : exp(-x[k]);
      acc += y;
      x[k] += 1e-9;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  const int threads = 512, blocks = sms * 4, iters = 20000;
  double* out; unsigned long long* cyc;
  CK(cudaMalloc(&out, sizeof(double) * threads * blocks));
  CK(cudaMalloc(&cyc, sizeof(unsigned long long) * blocks));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  // warm-up (also lets the clock settle)
  for (int w = 0; w < 3; ++w) dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7, cyc);
  CK(cudaDeviceSynchronize());
  float best_ms = 1e30f; unsigned long long* hc = (unsigned long long*)malloc(8 * blocks);
  double cyc_med = 0;
  const int reps = argc > 1 ? atoi(argv[1]) : 60;  // ~3 s of saturated FP64 pipe for the sampler
  for (int rep = 0; rep < reps; ++rep) {
    CK(cudaEventRecord(e0));
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7, cyc);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best_ms) {
      best_ms = ms;
      CK(cudaMemcpy(hc, cyc, 8 * blocks, cudaMemcpyDeviceToHost));
      double s = 0; for (int i = 0; i < blocks; ++i) s += hc[i]; cyc_med = s / blocks;
    }
  }
  double dfma = (double)threads * blocks * iters * 16 * 8;
  double dfma_per_s = dfma / (best_ms * 1e-3);
  (void)cyc_med;
  // transcendentals
  float tl = 1e30f, te = 1e30f; const int titers = 2000;
  for (int rep = 0; rep < 5; ++rep) {
    float ms;
    CK(cudaEventRecord(e0)); transc_kernel<0><<<blocks, threads>>>(out, titers, 1.5);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < tl) tl = ms;
    CK(cudaEventRecord(e0)); transc_kernel<1><<<blocks, threads>>>(out, titers, 1.5);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < te) te = ms;
  }
  double nt = (double)threads * blocks * titers * 8;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"attr_clock_mhz\": %.1f, "
         "\"dfma_per_s\": %.6e, \"best_rep_ms\": %.3f, "
         "\"fp64_tflops_fma\": %.3f, \"log_per_s\": %.6e, \"exp_per_s\": %.6e}\n",
         p.name, sms, clk_khz / 1e3, dfma_per_s, best_ms,
         2 * dfma_per_s / 1e12, nt / (tl * 1e-3), nt / (te * 1e-3));
  return 0;
}
