// kernels_native.cu -- the NATIVE race-kernel instantiations (native_kernel.cuh) and their selectors.
// Compiled once per (half, ticks per block): BBE_NATIVE_K1 selects the K = 1 half (one competitor per
// lane, the common layouts) or the K = 2-4 half, BBE_NATIVE_NT the block length, so the objects
// build in parallel.  K = 1 is built for NT = 8 and 16, K = 2 without a scan for 4 and 16, every other
// layout for NT = 4 only (longer blocks spill there).
#include "kernels.h"
#include "native_kernel.cuh"

#ifndef BBE_NATIVE_NT
#define BBE_NATIVE_NT 4
#endif
#define BBE_CAT2(a, b) a##b
#define BBE_CAT(a, b) BBE_CAT2(a, b)

namespace bbe {
namespace {

constexpr int NT = BBE_NATIVE_NT;

template <int K, bool SCAN>
KernelFn native_for_ch(int ch) {
    switch (ch) {
        case 1: return native_kernel<K, 1, SCAN, 4, NT>;
        case 2: return native_kernel<K, 2, SCAN, 4, NT>;
        case 3: return native_kernel<K, 3, SCAN, 4, NT>;
        case 4: return native_kernel<K, 4, SCAN, 4, NT>;
        case 5: return native_kernel<K, 5, SCAN, 4, NT>;
        case 6: return native_kernel<K, 6, SCAN, 4, NT>;
        case 7: return native_kernel<K, 7, SCAN, 4, NT>;
        case 8: return native_kernel<K, 8, SCAN, 4, NT>;
    }
    return nullptr;
}

template <int K>
KernelFn native_for(int ch, bool scan) {
    return scan ? native_for_ch<K, true>(ch) : native_for_ch<K, false>(ch);
}

#ifdef BBE_NATIVE_K1
// K = 1 with a scan and W = 4m+1 or 4m+2: rows read 2 words at a time (at most one padding key)
KernelFn native_vec2_for(int ch) {
    switch (ch) {
        case 1: return native_kernel<1, 1, true, 2, NT>;
        case 3: return native_kernel<1, 3, true, 2, NT>;
        case 5: return native_kernel<1, 5, true, 2, NT>;
        case 7: return native_kernel<1, 7, true, 2, NT>;
        case 9: return native_kernel<1, 9, true, 2, NT>;
        case 11: return native_kernel<1, 11, true, 2, NT>;
        case 13: return native_kernel<1, 13, true, 2, NT>;
        case 15: return native_kernel<1, 15, true, 2, NT>;
    }
    return nullptr;
}
#endif

}  // namespace

#ifdef BBE_NATIVE_K1
KernelFn BBE_CAT(pick_native_k1_nt, BBE_NATIVE_NT)(int ch, bool scan, int vec) {
    return vec == 2 ? (scan ? native_vec2_for(ch) : nullptr) : native_for<1>(ch, scan);
}
#else
KernelFn BBE_CAT(pick_native_kn_nt, BBE_NATIVE_NT)(int k, int ch, bool scan) {
#if BBE_NATIVE_NT == 4
    switch (k) {
        case 2: return native_for<2>(ch, scan);
        case 3: return native_for<3>(ch, scan);
        case 4: return native_for<4>(ch, scan);
    }
    return nullptr;
#else
    // K = 2 with a scan stays at 4: 8 and 16 measured slower there (derby20: 12.3 -> 13.1 / 19.4 ms,
    // and 12.8 ms with the 16 ticks run as a loop of 4-tick groups)
    return (k == 2 && !scan) ? native_for_ch<2, false>(ch) : nullptr;
#endif
}
#endif

}  // namespace bbe
