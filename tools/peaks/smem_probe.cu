// smem_probe.cu — shared-memory wavefront cost of the access patterns the BOCD cell loop
// can use (which lanes share a table entry, 64- vs 128-bit entries).  Each kernel issues
// kIters loads per thread of one pattern; the time per warp-load (SM cycles) over the
// whole SM gives the wavefronts per request (1 wavefront / clk / SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_probe smem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kThreads = 512;

template <int PAT>
__device__ __forceinline__ unsigned entry(unsigned lane, unsigned it) {
    switch (PAT) {
        case 0: return lane;                        // 32 distinct consecutive
        case 1: return lane & 15;                   // halves share (l, l+16)
        case 2: return lane >> 1;                   // adjacent pairs share
        case 3: return lane & 7;                    // 8 distinct, 4 copies
        case 4: return lane >> 2;                   // adjacent quads share
        case 5: return 0;                           // uniform
        default: {                                  // pseudo-random over 256 entries
            unsigned h = (lane * 0x9E3779B9u) ^ (it * 0x85EBCA6Bu);
            h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
            return h & 255u;
        }
    }
}

template <int PAT, int BYTES>
__global__ void probe(unsigned* out) {
    __shared__ __align__(16) double tab[4096];
    for (int k = threadIdx.x; k < 4096; k += blockDim.x) tab[k] = 1.0 + k;
    __syncthreads();
    const unsigned lane = threadIdx.x & 31;
    // 8 lane patterns (loop-invariant byte addresses); immediate offsets keep the loop free of
    // address arithmetic, so the time per warp-load is the shared-memory wavefront count
    unsigned addr[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
        addr[k] = unsigned(__cvta_generic_to_shared(tab)) + ((entry<PAT>(lane, k) + 32u * k) & 127u) * BYTES;
    unsigned acc = 0;
    for (int it = 0; it < kIters / 64; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                unsigned w;
                if (BYTES == 16) {
                    double x, y;
                    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr[k] + unsigned(u * 512) % 2048u));
                    w = __double2loint(x) ^ __double2hiint(x) ^ __double2loint(y) ^ __double2hiint(y);
                } else {
                    double x;
                    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(addr[k] + unsigned(u * 256) % 2048u));
                    w = __double2loint(x) ^ __double2hiint(x);
                }
                acc ^= w;
            }
        }
    }
    if (acc == 0x12345u) out[0] = acc;
}

template <int PAT, int BYTES>
float run(const char* name, unsigned* d) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 4;
    probe<PAT, BYTES><<<grid, kThreads>>>(d);
    cudaEventRecord(a);
    probe<PAT, BYTES><<<grid, kThreads>>>(d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_loads_per_sm = double(grid / sms) * (kThreads / 32) * kIters;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("{\"pattern\": \"%s\", \"bytes\": %d, \"cycles_per_warp_load\": %.3f}\n", name, BYTES,
           cyc / warp_loads_per_sm);
    return ms;
}

int main() {
    unsigned* d;
    cudaMalloc(&d, 8);
    run<0, 16>("32 distinct consecutive", d);
    run<1, 16>("halves share (l, l+16)", d);
    run<2, 16>("adjacent pairs share", d);
    run<3, 16>("8 distinct", d);
    run<4, 16>("adjacent quads share", d);
    run<5, 16>("uniform", d);
    run<6, 16>("random of 256", d);
    run<0, 8>("32 distinct consecutive", d);
    run<1, 8>("halves share (l, l+16)", d);
    run<2, 8>("adjacent pairs share", d);
    run<3, 8>("8 distinct", d);
    run<5, 8>("uniform", d);
    run<6, 8>("random of 256", d);
    return 0;
}
