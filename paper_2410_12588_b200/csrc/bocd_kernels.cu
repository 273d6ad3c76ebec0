// bocd_kernels.cu — instantiations of the resident BOCD kernel and the variant table.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "bocd_kernel.cuh"
#include "bocd_variants.h"

namespace fbocd {

template <int NT, int J, bool FULL, bool TAB2, int SPB, int MINB, int MODE>
static void make_variant_mode(Variant* out) {
    Variant v;
    v.fn = reinterpret_cast<const void*>(&bocd_update_kernel<NT, J, FULL, TAB2, false, SPB, MINB, false, MODE>);
    v.fn_eager = reinterpret_cast<const void*>(&bocd_update_kernel<NT, J, FULL, TAB2, true, SPB, MINB, false, MODE>);
    v.fn_p = reinterpret_cast<const void*>(&bocd_update_kernel<NT, J, FULL, TAB2, false, SPB, MINB, true, MODE>);
    v.fn_eager_p = reinterpret_cast<const void*>(&bocd_update_kernel<NT, J, FULL, TAB2, true, SPB, MINB, true, MODE>);
    v.pref = kPrefOk<NT, J, FULL>;
    v.nt = NT;
    v.j = J;
    v.spb = SPB;
    v.full = FULL;
    v.tab2 = TAB2;
    v.group_smem = sizeof(GroupSmem<NT, kTile>);
    v.group_smem_p = sizeof(GroupSmem<NT, kPrefOk<NT, J, FULL> ? kTileP : kTile>);  // (+ PREF buffer): group_bytes
    *out = v;
}
// the truncation mode is a template parameter of the kernels (MERGE / DROP specialised tails);
// MODE bit 1 (FULL kernels only): 2 alpha0 has a fractional part f2, added to the exact
// integer conversion of 2 alpha0 + r + 1 - f2 (one DADD per cell)
template <int NT, int J, bool FULL, bool TAB2, int SPB, int MINB>
static void make_variant(int mode, Variant* out, bool frac = false) {
    if constexpr (FULL) {
        if (frac) {
            if (mode == 0)
                make_variant_mode<NT, J, FULL, TAB2, SPB, MINB, 2>(out);
            else
                make_variant_mode<NT, J, FULL, TAB2, SPB, MINB, 3>(out);
            return;
        }
    }
    if (mode == 0)
        make_variant_mode<NT, J, FULL, TAB2, SPB, MINB, 0>(out);
    else
        make_variant_mode<NT, J, FULL, TAB2, SPB, MINB, 1>(out);
}
// + the one-CTA-per-SM twins (SPB * MINB groups, MINB = 1) of the one-unit kernels, for a
// batch that fits one wave unevenly (C2: 1,024 series of R = 512 on 148 SMs are 8 on most SMs
// in CTAs of 4, at most 7 in balanced CTAs of 8)
template <int NT, int J, bool FULL, bool TAB2, int SPB, int MINB, int MODE>
static void set_wide(Variant* out) {
    constexpr int W = SPB * MINB;
    out->fn_w = reinterpret_cast<const void*>(&bocd_update_kernel<NT, J, FULL, TAB2, false, W, 1, false, MODE>);
    out->fn_eager_w = reinterpret_cast<const void*>(&bocd_update_kernel<NT, J, FULL, TAB2, true, W, 1, false, MODE>);
    out->spb_w = W;
}
template <int NT, int J, bool FULL, bool TAB2, int SPB, int MINB>
static void make_variant_w(int mode, Variant* out, bool frac = false) {
    make_variant<NT, J, FULL, TAB2, SPB, MINB>(mode, out, frac);
    const int m = mode + (FULL && frac ? 2 : 0);
    if (m == 0) set_wide<NT, J, FULL, TAB2, SPB, MINB, 0>(out);
    else if (m == 1) set_wide<NT, J, FULL, TAB2, SPB, MINB, 1>(out);
    else if (m == 2) set_wide<NT, J, FULL, TAB2, SPB, MINB, 2>(out);
    else set_wide<NT, J, FULL, TAB2, SPB, MINB, 3>(out);
}

// Variant choice: FULL kernels (R = NT*J, compile-time ring arithmetic) for the
// power-of-two R of the BASELINE configs; generic kernels (runtime R, masked
// cells) for any other 2 <= R <= 4096.  Each variant has a lazy-MAP and an
// EAGER-MAP kernel (bocd_kernel.cuh), one-unit and persistent, per truncation mode.
// (Shapes measured slower for R = 1024 and removed: 128x8 with 3-4 series per CTA, 64x16
// (J = 16: > 168 registers), 256x4.)
int select_variant(int R, int mode, double alpha0, Variant* out) {
    // FULL kernels form 2 alpha_{r+1} = 2 alpha0 + r + 1 as the exact integer conversion of
    // floor(2 alpha0) + 1 + r, plus the fractional part of 2 alpha0 when it has one (MODE bit
    // 1: one DADD per cell; the default alpha0 = 1 and every half-integer need none)
    const double a2 = 2.0 * alpha0;
    const bool full_ok = a2 > 0.0 && a2 <= double(1 << 20);
    const bool frac = a2 != std::floor(a2);
    switch (full_ok ? R : -1) {
        case 256: make_variant<32, 8, true, true, 8, 2>(mode, out, frac); return 0;
        case 512: make_variant_w<64, 8, true, true, 4, 2>(mode, out, frac); return 0;
        case 1024: make_variant_w<128, 8, true, true, 2, 2>(mode, out, frac); return 0;
        case 2048: make_variant<256, 8, true, false, 1, 2>(mode, out, frac); return 0;
        case 4096: make_variant<512, 8, true, false, 1, 1>(mode, out, frac); return 0;
        default: break;
    }
    if (R < 2 || R > 4096) return -1;
    if (!full_ok && (R == 256 || R == 512 || R == 1024 || R == 2048 || R == 4096)) {
        // the generic kernels of the same shape (TAB2 up to 2048)
        if (R == 256) { make_variant<32, 8, false, true, 8, 2>(mode, out); return 0; }
        if (R == 512) { make_variant<64, 8, false, true, 4, 2>(mode, out); return 0; }
        if (R == 1024) { make_variant<128, 8, false, true, 2, 2>(mode, out); return 0; }
        if (R == 2048) { make_variant<256, 8, false, false, 1, 2>(mode, out); return 0; }
        make_variant<512, 8, false, false, 1, 1>(mode, out);
        return 0;
    }
    if (R <= 32) { make_variant<32, 1, false, true, 8, 2>(mode, out); return 0; }
    if (R <= 256) { make_variant<32, 8, false, true, 8, 2>(mode, out); return 0; }
    if (R <= 512) { make_variant<64, 8, false, true, 4, 2>(mode, out); return 0; }
    if (R <= 1024) { make_variant<128, 8, false, true, 2, 2>(mode, out); return 0; }
    if (R <= 2048) { make_variant<256, 8, false, false, 1, 2>(mode, out); return 0; }
    make_variant<512, 8, false, false, 1, 1>(mode, out);
    return 0;
}

size_t variant_smem(const Variant& v, int R, bool persistent) {
    const int rows = v.full ? R + v.nt : (v.tab2 ? 2 * R : R);  // table_entries
    const bool pref = persistent && v.pref;  // only the persistent kernels carry the prefetch buffer
    const size_t grp = (pref ? v.group_smem_p : v.group_smem) +
                       (pref ? ((3 * size_t(R) * sizeof(double) + sizeof(SeriesScalars) + 15) & ~size_t(15)) : 0);
    return bocd_fm_bytes(cell_ec(v.full, v.nt * v.j, pref), cell_logbits(v.full, v.nt * v.j)) + table_bytes(rows, v.full) +
           size_t(v.spb) * grp;
}

size_t variant_smem_wide(const Variant& v, int R) {
    Variant w = v;
    w.spb = v.spb_w;
    return variant_smem(w, R, false);
}

// Test hook: elementwise fast_log2 / fast_exp2 (which 0 / 1) and the cell loop's cell_log2 /
// cell_exp2 (which 2 / 3; tables at the BOCD kernel's addresses) over device arrays.
__global__ void fastmath_probe_kernel(int which, const double* in, double* out, int64_t n,
                                      const FastMathTables* tab, const CellTables* ct) {
    extern __shared__ __align__(16) unsigned char dyn[];
    const unsigned fmb = fm_setup(dyn, tab);
    const bool at_base = smem_addr(dyn) == kDynBase && fmb == kFmBase;
    double* ex = reinterpret_cast<double*>(dyn + (kCellExpBase - kDynBase));
    constexpr int EC = cell_ec(true, 1024, false);
    for (int k = threadIdx.x; k < kCellExpTab * EC; k += blockDim.x) ex[k] = ct->exptab[k / EC];
    double2* lg = reinterpret_cast<double2*>(dyn + (cell_log_base<EC>() - kDynBase));
    const double2* src = which == 4 ? ct->log10 : ct->log8;
    for (int k = threadIdx.x; k < (which == 4 ? 1024 : 256); k += blockDim.x) lg[k] = src[k];
    __syncthreads();
    const double C7 = __hiloint2double(0x43380000, int(0x80000000u));  // Dc = 0
    const unsigned lbe = 8u * (threadIdx.x & unsigned(EC - 1));
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        double v;
        switch (which) {
            case 0: v = fast_log2(in[k], fmb); break;
            case 1: v = fast_exp2(in[k], fmb); break;
            case 2: v = cell_log2<EC, 8>(in[k]); break;
            case 4: v = cell_log2<EC, 10>(in[k]); break;
            default: v = cell_exp2<EC>(in[k], C7, lbe); break;
        }
        out[k] = at_base ? v : __longlong_as_double(0x7FF8000000000000ll);  // NaN: layout check failed
    }
}

int launch_fastmath_probe(int which, const double* in, double* out, int64_t n, const FastMathTables* tab,
                          const CellTables* ct, cudaStream_t st) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    if (blocks < 1) blocks = 1;
    const size_t smem = bocd_fm_bytes(cell_ec(true, 1024, false), 10);
    if (cudaFuncSetAttribute(fastmath_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) !=
        cudaSuccess)
        return -1;
    fastmath_probe_kernel<<<unsigned(blocks), 256, smem, st>>>(which, in, out, n, tab, ct);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// The constant bank is per translation unit: this is the copy the kernels above read.
int upload_fastmath_constants() {
    if (cudaMemcpyToSymbol(c_fm, kFastMathConstants, sizeof(kFastMathConstants)) != cudaSuccess) return -1;
    return cudaMemcpyToSymbol(c_cell, kCellConstants, sizeof(kCellConstants)) == cudaSuccess ? 0 : -1;
}

}  // namespace fbocd
