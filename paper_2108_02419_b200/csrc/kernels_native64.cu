// kernels_native64.cu -- the NATIVE64 race-kernel instantiations (native64_kernel.cuh) and their
// selectors.  Compiled once per part so the objects build in parallel:
//   BBE_N64_SCAN = 0: the scan-free layouts (theta = 0 everywhere): K = 1-4, 8- and 16-tick blocks,
//                     with and without a lognormal competitor;
//   BBE_N64_SCAN = 1: layouts with a front-runner scan, BBE_N64_SCAN_NT-tick blocks, CH = 1-8 key chunks, one part
//                     per (BBE_N64_K1: K = 1 or K = 2-4) x (BBE_N64_LN: lognormal competitor or not).
#include "kernels.h"
#include "native64_kernel.cuh"

#ifndef BBE_N64_SCAN
#define BBE_N64_SCAN 1
#endif
#ifndef BBE_N64_K1
#define BBE_N64_K1 1
#endif
#ifndef BBE_N64_LN
#define BBE_N64_LN 0
#endif
#define BBE_CAT2(a, b) a##b
#define BBE_CAT(a, b) BBE_CAT2(a, b)

namespace bbe {
namespace {

#if BBE_N64_SCAN
constexpr bool LN = BBE_N64_LN != 0;
template <int K>
KernelFn n64_scan_for_ch(int ch) {
    switch (ch) {
        case 1: return native64_kernel<K, 1, true, LN, BBE_N64_SCAN_NT>;
        case 2: return native64_kernel<K, 2, true, LN, BBE_N64_SCAN_NT>;
        case 3: return native64_kernel<K, 3, true, LN, BBE_N64_SCAN_NT>;
        case 4: return native64_kernel<K, 4, true, LN, BBE_N64_SCAN_NT>;
        case 5: return native64_kernel<K, 5, true, LN, BBE_N64_SCAN_NT>;
        case 6: return native64_kernel<K, 6, true, LN, BBE_N64_SCAN_NT>;
        case 7: return native64_kernel<K, 7, true, LN, BBE_N64_SCAN_NT>;
        case 8: return native64_kernel<K, 8, true, LN, BBE_N64_SCAN_NT>;
    }
    return nullptr;
}
#else
template <bool LN, int NT>
KernelFn n64_free_for(int k) {
    switch (k) {
        case 1: return native64_kernel<1, 1, false, LN, NT>;
        case 2: return native64_kernel<2, 1, false, LN, NT>;
        case 3: return native64_kernel<3, 1, false, LN, NT>;
        case 4: return native64_kernel<4, 1, false, LN, NT>;
    }
    return nullptr;
}
#endif

}  // namespace

#if BBE_N64_SCAN
// pick_native64_scan_k1_ln0 / _k1_ln1 (K = 1) and _kn_ln0 / _kn_ln1 (K = 2-4)
#if BBE_N64_K1
KernelFn BBE_CAT(pick_native64_scan_k1_ln, BBE_N64_LN)(int k, int ch) { return k == 1 ? n64_scan_for_ch<1>(ch) : nullptr; }
#else
KernelFn BBE_CAT(pick_native64_scan_kn_ln, BBE_N64_LN)(int k, int ch) {
    switch (k) {
        case 2: return n64_scan_for_ch<2>(ch);
        case 3: return n64_scan_for_ch<3>(ch);
        case 4: return n64_scan_for_ch<4>(ch);
    }
    return nullptr;
}
#endif
#else
KernelFn pick_native64_free(int k, bool ln, int nt) {
    if (nt == 16) return ln ? n64_free_for<true, 16>(k) : n64_free_for<false, 16>(k);
    if (nt == 8) return ln ? n64_free_for<true, 8>(k) : n64_free_for<false, 8>(k);
    return nullptr;
}
#endif

}  // namespace bbe
