// issue_peak.cu -- measured per-SM issue rates of the instruction classes the race kernels use
// (SURVEY.md §8d asks to re-measure the FFMA / IMAD / LOP3 peaks on the box).
//
// Each thread runs 8 independent dependency chains of one operation; the grid fills every SM.
// Reports lane-ops/s and the fraction of 148 SMs x 128 lanes x f_SM (the roofline peak bench.py uses).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o issue_peak tools/issue_peak.cu && ./issue_peak
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

constexpr int kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(256) chains(uint32_t* out, uint32_t seed) {
    uint32_t a[8];
    float f[8];
    double g[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = seed * (threadIdx.x + 1) + i;
        f[i] = (float)a[i] * 1e-9f;
        g[i] = (double)a[i] * 1e-9;
    }
    const double gb = 1.0000000001, gc = 1e-12;
    const uint32_t b = seed ^ 0x9E3779B9u, c = seed * 3u + 7u;
    const float fb = 1.0000001f, fc = 1e-7f;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if constexpr (OP == 0) f[i] = fmaf(f[i], fb, fc);                    // FFMA
            if constexpr (OP == 1) a[i] = a[i] * b + c;                          // IMAD
            if constexpr (OP == 2) a[i] = (a[i] ^ b) & (c | a[i]);               // LOP3
            if constexpr (OP == 3) a[i] = min(a[i] + b, c + (uint32_t)i);        // VIADDMNMX
            if constexpr (OP == 4) a[i] = a[i] < b + (uint32_t)i ? a[i] + 1u : a[i] - c;  // ISETP+SEL
            if constexpr (OP == 5) g[i] = fma(g[i], gb, gc);                     // DFMA
            if constexpr (OP == 6) g[i] = __dadd_rn(g[i], gc);                   // DADD
            if constexpr (OP == 7) g[i] = __dmul_rn(g[i], gb);                   // DMUL
            if constexpr (OP == 8) g[i] = g[i] < gb ? __dadd_rn(g[i], gc) : __dmul_rn(g[i], gc);  // DSETP+DADD/DMUL
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i] + __float_as_uint(f[i]) + (uint32_t)__double2loint(g[i]);
    if (s == 0x12345678u) out[0] = s;  // keep the chains alive
}

template <int OP>
double run(const char* name, int sms, double f_mhz, int ops_per_step) {
    uint32_t* out;
    cudaMalloc(&out, 4);
    const int blocks = sms * 8, threads = 256;
    chains<OP><<<blocks, threads>>>(out, 1u);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) chains<OP><<<blocks, threads>>>(out, 2u + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 5.0 * blocks * threads * (double)kIters * 8 * ops_per_step;
    const double rate = ops / (ms * 1e-3);
    const double peak = sms * 128.0 * f_mhz * 1e6;
    printf("%-26s %8.2f T lane-op/s  %5.1f %% of %d SMs x 128 lanes x %.0f MHz\n", name, rate / 1e12, 100 * rate / peak,
           sms, f_mhz);
    cudaFree(out);
    return rate;
}

int main() {
    int dev = 0, sms = 0, khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    const double mhz = khz / 1000.0;
    run<0>("FFMA (fma pipe)", sms, mhz, 1);
    run<1>("IMAD (fma pipe)", sms, mhz, 1);
    run<2>("LOP3 (alu pipe)", sms, mhz, 1);
    run<3>("VIADDMNMX (alu pipe)", sms, mhz, 1);
    run<4>("ISETP + SEL (alu pipe)", sms, mhz, 2);
    run<5>("DFMA (fp64)", sms, mhz, 1);
    run<6>("DADD (fp64)", sms, mhz, 1);
    run<7>("DMUL (fp64)", sms, mhz, 1);
    run<8>("DSETP + DADD|DMUL (fp64)", sms, mhz, 2);
    return 0;
}
