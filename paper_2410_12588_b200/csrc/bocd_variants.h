// bocd_variants.h — host-side description of the compiled kernel variants.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace fbocd {

struct Variant {
    const void* fn = nullptr;        // __global__ void(KParams), MAP on demand
    const void* fn_eager = nullptr;  // MAP reduced every step
    const void* fn_p = nullptr;        // persistent twins (streaming calls: few steps per call)
    const void* fn_eager_p = nullptr;
    int nt = 0;                // threads per series group
    int j = 0;                 // cells per thread
    int spb = 0;               // series groups per CTA
    bool full = false;         // R == nt * j at compile time
    bool tab2 = false;         // doubled per-r tables
    size_t group_smem = 0;     // bytes of GroupSmem (one-unit kernels)
    size_t group_smem_p = 0;   // of the persistent kernels' GroupSmem (64-step tiles); + PREF buffer
    bool pref = false;         // the persistent kernels prefetch the next unit's state (TMA)
    // one-CTA-per-SM twins of the one-unit kernels (spb_w = spb * MINB series groups per CTA,
    // launched as one balanced wave when the batch fits one wave unevenly); null if none
    const void* fn_w = nullptr;
    const void* fn_eager_w = nullptr;
    int spb_w = 0;
};

int select_variant(int R, int mode, double alpha0, Variant* out);  // mode: FALCON_TRUNC_MERGE / _DROP
// dynamic shared memory of one CTA of variant v at ring size R (persistent or one-unit kernels)
size_t variant_smem(const Variant& v, int R, bool persistent);
size_t variant_smem_wide(const Variant& v, int R);  // of the fn_w / fn_eager_w kernels

struct FastMathTables;
struct CellTables;
int upload_fastmath_constants();  // once per device, before any kernel that uses fast_log2/exp2
int launch_fastmath_probe(int which, const double* in, double* out, int64_t n, const FastMathTables* tab,
                          const CellTables* ct, cudaStream_t st);

}  // namespace fbocd
