// bocd_variants.h — host-side description of the compiled kernel variants.
#pragma once

#include <cstddef>

namespace fbocd {

struct Variant {
    const void* fn = nullptr;  // __global__ void(KParams)
    int nt = 0;                // threads per series group
    int j = 0;                 // cells per thread
    int spb = 0;               // series groups per CTA
    bool full = false;         // R == nt * j at compile time
    size_t group_smem = 0;     // bytes of per-group shared memory
};

int select_variant(int R, Variant* out);

}  // namespace fbocd
