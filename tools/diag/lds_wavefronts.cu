// Microbenchmark: shared-memory wavefronts per warp-level LDS of various widths and
// address patterns (uniform / per-lane / single active lane).  Run under ncu with
//   --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum
// one kernel per pattern, 1 warp per CTA, kIter loads per thread.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIter = 4096;
template <int MODE>
__global__ void lds_kernel(double* out, int salt) {
    __shared__ __align__(16) double tab[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = i * 0.5;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    int base = salt & 7;
#pragma unroll 8
    for (int it = 0; it < kIter; ++it) {
        int idx = (base + it) & 255;  // uniform across the warp
        if (MODE == 0) {  // LDS.32 uniform
            acc += __int_as_float(reinterpret_cast<const int*>(tab)[idx]);
        } else if (MODE == 1) {  // LDS.64 uniform
            acc += tab[idx];
        } else if (MODE == 2) {  // LDS.128 uniform
            double2 v = reinterpret_cast<const double2*>(tab)[idx];
            acc += v.x + v.y;
        } else if (MODE == 3) {  // LDS.64 per-lane consecutive
            acc += tab[(idx + lane) & 1023];
        } else if (MODE == 4) {  // LDS.128 per-lane consecutive
            double2 v = reinterpret_cast<const double2*>(tab)[(idx + lane) & 511];
            acc += v.x + v.y;
        } else if (MODE == 5) {  // LDS.64, lane 0 only
            if (lane == 0) acc += tab[idx];
        } else if (MODE == 6) {  // LDS.64, lanes 0..3 distinct
            if (lane < 4) acc += tab[(idx + lane) & 1023];
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 32 * sizeof(double));
    lds_kernel<0><<<148, 32>>>(out, 1);
    lds_kernel<1><<<148, 32>>>(out, 1);
    lds_kernel<2><<<148, 32>>>(out, 1);
    lds_kernel<3><<<148, 32>>>(out, 1);
    lds_kernel<4><<<148, 32>>>(out, 1);
    lds_kernel<5><<<148, 32>>>(out, 1);
    lds_kernel<6><<<148, 32>>>(out, 1);
    cudaError_t e = cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(e));
    return 0;
}
