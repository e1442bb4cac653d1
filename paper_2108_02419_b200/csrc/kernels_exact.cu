// kernels_exact.cu -- the bit-exact race kernels (exact_kernel.cuh: INJECT and MT), the MT seeding
// kernel, and the MT __constant__ tables they read.
#include "exact_kernel.cuh"
#include "kernels.h"

namespace bbe {

KernelFn pick_exact(int mode, int k, bool ln, bool lean) {
    if (mode == MT) {
        switch (k) {
            case 1:
                if (lean) return ln ? exact_kernel<1, MT, true, true> : exact_kernel<1, MT, false, true>;
                return ln ? exact_kernel<1, MT, true> : exact_kernel<1, MT, false>;
            case 2: return ln ? exact_kernel<2, MT, true> : exact_kernel<2, MT, false>;
            case 3: return ln ? exact_kernel<3, MT, true> : exact_kernel<3, MT, false>;
            case 4: return ln ? exact_kernel<4, MT, true> : exact_kernel<4, MT, false>;
        }
    } else if (mode == INJECT) {
        switch (k) {
            case 1: return exact_kernel<1, INJECT>;
            case 2: return exact_kernel<2, INJECT>;
            case 3: return exact_kernel<3, INJECT>;
            case 4: return exact_kernel<4, INJECT>;
        }
    }
    return nullptr;
}

cudaError_t upload_mt_tables(const uint32_t* init624, int exp_ok, const uint64_t* exp_tab256, const double* exp_c8) {
    cudaError_t e = cudaMemcpyToSymbol(c_mt_init, init624, sizeof(uint32_t) * kMtN);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_exp_ok, &exp_ok, sizeof(int));
    if (e == cudaSuccess && exp_ok) e = cudaMemcpyToSymbol(c_exp_tab, exp_tab256, sizeof(uint64_t) * 256);
    if (e == cudaSuccess && exp_ok) e = cudaMemcpyToSymbol(c_exp_c, exp_c8, sizeof(double) * 8);
    return e;
}

cudaError_t launch_mt_seed(cudaStream_t stream, const uint64_t* seeds, uint64_t h_run, int64_t sim_offset, int64_t n,
                           uint32_t* states) {
    mt_seed_kernel<<<(unsigned)((n + 127) / 128), 128, 0, stream>>>(seeds, h_run, sim_offset, n, states);
    return cudaGetLastError();
}

uint64_t splitmix64_host(uint64_t x) { return splitmix64_dev(x); }

}  // namespace bbe
