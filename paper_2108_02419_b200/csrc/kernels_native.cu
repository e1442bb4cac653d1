// kernels_native.cu -- the NATIVE race-kernel instantiations (native_kernel.cuh) and their selector.
// Compiled twice: with BBE_NATIVE_K1 (one competitor per lane, the common layouts) and without
// (2-4 competitors per lane), so the two halves build in parallel.
#include "kernels.h"
#include "native_kernel.cuh"

namespace bbe {
namespace {

template <int K, bool SCAN>
KernelFn native_for_ch(int ch) {
    switch (ch) {
        case 1: return native_kernel<K, 1, SCAN>;
        case 2: return native_kernel<K, 2, SCAN>;
        case 3: return native_kernel<K, 3, SCAN>;
        case 4: return native_kernel<K, 4, SCAN>;
        case 5: return native_kernel<K, 5, SCAN>;
        case 6: return native_kernel<K, 6, SCAN>;
        case 7: return native_kernel<K, 7, SCAN>;
        case 8: return native_kernel<K, 8, SCAN>;
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
        case 1: return native_kernel<1, 1, true, 2>;
        case 3: return native_kernel<1, 3, true, 2>;
        case 5: return native_kernel<1, 5, true, 2>;
        case 7: return native_kernel<1, 7, true, 2>;
        case 9: return native_kernel<1, 9, true, 2>;
        case 11: return native_kernel<1, 11, true, 2>;
        case 13: return native_kernel<1, 13, true, 2>;
        case 15: return native_kernel<1, 15, true, 2>;
    }
    return nullptr;
}
#endif

}  // namespace

#ifdef BBE_NATIVE_K1
KernelFn pick_native_k1(int ch, bool scan, int vec) {
    return vec == 2 ? (scan ? native_vec2_for(ch) : nullptr) : native_for<1>(ch, scan);
}
#else
KernelFn pick_native_kn(int k, int ch, bool scan) {
    switch (k) {
        case 2: return native_for<2>(ch, scan);
        case 3: return native_for<3>(ch, scan);
        case 4: return native_for<4>(ch, scan);
    }
    return nullptr;
}

KernelFn pick_native(int k, int ch, bool scan, int vec) {
    if (k == 1) return pick_native_k1(ch, scan, vec);
    return vec == 4 ? pick_native_kn(k, ch, scan) : nullptr;
}
#endif

}  // namespace bbe
