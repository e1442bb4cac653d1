// kernels.h -- the kernel translation units' interface to the host code (bbe_sim.cu).
//
// The race kernels are compiled in their own translation units (kernels_native.cu, kernels_exact.cu)
// so the three objects build in parallel; the host picks a kernel through these functions and
// launches it through the returned pointer.  MT tables live in __constant__ memory of the exact
// translation unit, so they are uploaded from there.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace bbe {

typedef void (*KernelFn)(LaunchArgs);

// NATIVE: K competitors per lane, CH key chunks of VEC (4 or 2) words, SCAN = some theta > 0, NT
// ticks per block; nullptr where that combination is not built (see kernels_native.cu)
KernelFn pick_native(int k, int ch, bool scan, int vec, int nt);
// the per-translation-unit halves (kernels_native.cu built once per K half and NT)
KernelFn pick_native_k1_nt8(int ch, bool scan, int vec);
KernelFn pick_native_k1_nt16(int ch, bool scan, int vec);
KernelFn pick_native_kn_nt4(int k, int ch, bool scan);
KernelFn pick_native_kn_nt16(int k, int ch, bool scan);
// NATIVE64 (FP64 state): with a front-runner scan (BBE_N64_SCAN_NT = 16-tick blocks), or scan-free (NT = 8 or 16);
// LN = some lognormal competitor
KernelFn pick_native64_scan(int k, int ch, bool ln);  // bbe_sim.cu: dispatches to the four parts
KernelFn pick_native64_scan_k1_ln0(int k, int ch);
KernelFn pick_native64_scan_k1_ln1(int k, int ch);
KernelFn pick_native64_scan_kn_ln0(int k, int ch);
KernelFn pick_native64_scan_kn_ln1(int k, int ch);
KernelFn pick_native64_free(int k, bool ln, int nt);
// INJECT / MT (mode: INJECT or MT), K competitors per lane, LN = some lognormal competitor (MT)
KernelFn pick_exact(int mode, int k, bool ln, bool lean);  // lean: MT, K = 1, <= 2 segments per warp
// c_mt_init (init_genrand(19650218)), and the host libm's exp table for MT lognormal steps
cudaError_t upload_mt_tables(const uint32_t* init624, int exp_ok, const uint64_t* exp_tab256, const double* exp_c8);
// random.Random(seed) for n sims (per-sim seeds, or derive_seed(master, "run", offset + i) via h_run)
cudaError_t launch_mt_seed(cudaStream_t stream, const uint64_t* seeds, uint64_t h_run, int64_t sim_offset, int64_t n,
                           uint32_t* states);
// splitmix64 (seeding.py:24-28), shared with the device code
uint64_t splitmix64_host(uint64_t x);

}  // namespace bbe
