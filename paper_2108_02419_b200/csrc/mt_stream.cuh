// mt_stream.cuh -- CPython's random.Random (MT19937) on the GPU, for BBE_MODE_MT.
//
// The reference seeds every dry run with make_rng(seed) = random.Random(seed & (2^64-1))
// (seeding.py:62-64, agents.py:164, batch.py:117-119) and draws steps with uniform() and
// lognormvariate() (race.py:46-47, 68-69).  Reproducing that stream per simulation makes the GPU
// result identical to the reference's for the same seeds.  Algorithms restated from CPython 3.12
// Modules/_randommodule.c (init_genrand, init_by_array, genrand_uint32, random_random) and
// Lib/random.py (uniform, normalvariate, lognormvariate).
//
// Layout: (1) mt_seed_kernel, one thread per sim, runs init_by_array's two serial passes (pass 1
// twice, the second time in lockstep with pass 2, so nothing but the final state is stored) and
// writes the seeded 624-word state sim-major through a 32x32 shared-memory transpose; (2) the race kernel keeps
// each segment's state in shared memory and regenerates it in place, W lanes per 624-word twist.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bbe {

constexpr int kMtN = 624;
constexpr int kMtM = 397;

// init_genrand(19650218): the table every init_by_array starts from (host-computed).
__constant__ uint32_t c_mt_init[kMtN];

// lognormvariate = exp(normalvariate): CPython calls the host libm's exp.  glibc's exp is the
// table-driven algorithm of sysdeps/ieee754/dbl-64/e_exp.c (N = 128, degree-5 polynomial); the host
// reads its constants and table out of the very libm CPython uses (bbe_sim.cu: load_libm_exp) and
// the kernel evaluates it in the order the FMA build of that code does, which reproduces exp()
// bit-for-bit (tools/glibc_exp_probe.c: 0 mismatches in 4e7 arguments).  If the table was not found,
// c_exp_ok = 0 and CUDA's exp is used (last-bit differences possible).
__constant__ uint64_t c_exp_tab[256];
__constant__ double c_exp_c[8];  // invln2N, shift, negln2hiN, negln2loN, C2, C3, C4, C5
__constant__ int c_exp_ok;

__device__ __forceinline__ double libm_exp(double x) {
    const uint64_t ux = __double_as_longlong(x);
    const uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ffu;
    if (!c_exp_ok || abstop >= 0x408u) return exp(x);  // |x| >= 512 (never reached by the step laws)
    if (abstop < 0x3c9u) return __dadd_rn(1.0, x);      // |x| < 2^-54: glibc returns 1.0 + x
    double kd = __fma_rn(c_exp_c[0], x, c_exp_c[1]);
    const uint64_t ki = __double_as_longlong(kd);
    kd = __dsub_rn(kd, c_exp_c[1]);
    const double r = __fma_rn(kd, c_exp_c[3], __fma_rn(kd, c_exp_c[2], x));
    const int idx = 2 * (int)(ki % 128u);
    const uint64_t top = ki << 45;
    const double tail = __longlong_as_double(c_exp_tab[idx]);
    const double scale = __longlong_as_double(c_exp_tab[idx + 1] + top);
    const double r2 = __dmul_rn(r, r);
    const double tmp = __fma_rn(__dmul_rn(r2, r2), __fma_rn(r, c_exp_c[7], c_exp_c[6]),
                                __fma_rn(r2, __fma_rn(r, c_exp_c[5], c_exp_c[4]), __dadd_rn(tail, r)));
    return __fma_rn(scale, tmp, scale);
}

__host__ __device__ inline uint64_t splitmix64_dev(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// derive_seed(master, "run", i) (seeding.py:50-59); h_run = splitmix64(splitmix64(master) ^ fnv("s:run"))
__device__ __forceinline__ uint64_t derive_seed_run_dev(uint64_t h_run, uint64_t i) {
    uint64_t h = 0xCBF29CE484222325ull;
    h = (h ^ (uint64_t)'i') * 0x100000001B3ull;
    h = (h ^ (uint64_t)':') * 0x100000001B3ull;
#pragma unroll
    for (int k = 0; k < 8; ++k) h = (h ^ ((i >> (56 - 8 * k)) & 0xffu)) * 0x100000001B3ull;
    return splitmix64_dev(h_run ^ h);
}

__device__ __forceinline__ uint32_t mt_temper(uint32_t y) {
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    return y ^ (y >> 18);
}

__device__ __forceinline__ uint32_t mt_mix(uint32_t a, uint32_t b, uint32_t m) {
    const uint32_t y = (a & 0x80000000u) | (b & 0x7fffffffu);
    return m ^ (y >> 1) ^ ((0u - (y & 1u)) & 0x9908b0dfu);
}

// Kinderman-Monahan acceptance of one normalvariate trial (Lib/random.py): u1 = random(), u2 =
// 1 - random() from the tempered words (w0, w1), (w2, w3); z = NV_MAGICCONST * (u1 - 0.5) / u2;
// accept iff z*z/4 <= -log(u2).  Decided in FP32 when the two sides are apart by more than 4x a
// bound on the FP32 error, else in FP64 exactly as CPython does -- the same decision either way.
// FP32 error bound (a = u1 - 0.5, |l| = -log u2):
//   a from w0 alone: I2F + FMA rounding + the dropped w1 bits, |da| <= 2^-24 + 2^-27;
//   u2 = c 2^-27 - (w3>>6) 2^-53 with c = 2^27 - (w2>>5) >= 2 (c = 1 goes to FP64): rel <= 2^-22;
//   z: rel <= |da|/|a| + 2.5 2^-22;  z*z/4: rel <= 1.34e-7/|a| + 1.4e-6;
//   __logf: abs <= 2^-21.41 on [0.5, 2], else 3 ulp, plus u2's rel error: <= 6e-7 + 3.6e-7 |l|.
// The test below is |gap| > 4x that sum, multiplied through by |a| (no division).
// w1 is passed RAW (untempered): only the FP64 path needs it, so it is tempered there.
__device__ __forceinline__ bool km_accept(uint32_t w0, uint32_t w1_raw, uint32_t w2, uint32_t w3, double nv) {
    const float a = __fmaf_rn((float)(w0 >> 5), 0x1p-27f, -0.5f);
    const uint32_t c = 0x8000000u - (w2 >> 5);
    const float u2 = __fmaf_rn(-(float)(w3 >> 6), 0x1p-53f, (float)c * 0x1p-27f);
    const float z = __fdividef((float)nv * a, u2);
    const float zz = 0.25f * z * z;
    const float lg = -__logf(u2);
    const float gap = zz - lg;
    const float aa = fabsf(a);
    if (c >= 2u && fabsf(gap) * aa > zz * (5.4e-7f + 5.6e-6f * aa) + (2.4e-6f + 1.5e-6f * lg) * aa) return gap < 0.0f;
    const double u1 = random53(w0, mt_temper(w1_raw));
    const double u2d = __dsub_rn(1.0, random53(w2, w3));
    const double zx = __ddiv_rn(__dmul_rn(nv, __dsub_rn(u1, 0.5)), u2d);
    return __dmul_rn(__dmul_rn(zx, zx), 0.25) <= -log(u2d);  // z*z/4.0 (exact scaling)
}

// One thread per sim: random.Random(seed) for a u64 seed = init_by_array(key = 32-bit LE words of
// the seed, one word when seed < 2^32), CPython _randommodule.c.  states: [n][624] u32.
//   pass 1 (624 steps):  mt[i] = (mt[i] ^ ((mt[i-1] ^ (mt[i-1] >> 30)) * 1664525)) + key[j] + j,
//                        i = 1..623, then mt[0] = mt[623] and i = 1 once more (-> m1);
//   pass 2 (623 steps):  mt[i] = (mt[i] ^ ((mt[i-1] ^ (mt[i-1] >> 30)) * 1566083941)) - i,
//                        i = 2..623 reading pass 1's mt[i], then the wrap and i = 1; mt[0] = 2^31.
// Pass 2 starts from m1, which needs all of pass 1, and then reads pass 1's words in order -- so
// pass 1 runs twice: once for m1, then again in lockstep with pass 2 (two independent chains per
// thread).  Nothing is stored but the final state, which leaves through a 32x32 shared-memory
// transpose so every store is coalesced.
__global__ void __launch_bounds__(128) mt_seed_kernel(const uint64_t* seeds, uint64_t h_run, int64_t sim_offset,
                                                      int64_t n, uint32_t* states) {
    __shared__ uint32_t tile[4][32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t warp_base = s - lane;
    const bool on = s < n;
    const uint64_t seed = on ? (seeds ? seeds[s] : derive_seed_run_dev(h_run, (uint64_t)(sim_offset + s))) : 0ull;
    // key[j] + j of pass 1's step at i: j = (i - 1) % keylen, so odd i add ka and even i add kb
    const uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);
    const uint32_t ka = key0, kb = key1 ? key1 + 1u : key0;
    auto step1 = [&](uint32_t init_i, uint32_t prev, uint32_t kj) { return (init_i ^ ((prev ^ (prev >> 30)) * 1664525u)) + kj; };

    // pass 1, first run: only its last word and the extra step at i = 1 (m1) are kept
    const uint32_t p1_1 = step1(c_mt_init[1], c_mt_init[0], ka);  // pass 1's word 1 (read again below)
    uint32_t prev = p1_1;
#pragma unroll 2
    for (int i = 2; i < kMtN; ++i) prev = step1(c_mt_init[i], prev, (i & 1) ? ka : kb);
    const uint32_t m1 = step1(p1_1, prev, kb);  // mt[0] = mt[623]; i = 1 with j = 623 % keylen

    // pass 1 again (q, its word i) in lockstep with pass 2 (prev2), 32 words at a time
    uint32_t q = p1_1;
    uint32_t prev2 = m1;
    for (int blk0 = 0; blk0 < kMtN; blk0 += 32) {
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            const int i = blk0 + t;
            if (i >= 2 && i < kMtN) {
                q = step1(c_mt_init[i], q, (i & 1) ? ka : kb);
                prev2 = (q ^ ((prev2 ^ (prev2 >> 30)) * 1566083941u)) - (uint32_t)i;
                tile[warp][t][lane] = prev2;
            }
        }
        __syncwarp();
        const int w = blk0 + lane;  // this lane writes word w of each of the warp's 32 sims
        for (int r = 0; r < 32; ++r) {
            const int64_t sr = warp_base + r;
            if (sr < n && w >= 2 && w < kMtN) states[sr * kMtN + w] = tile[warp][lane][r];
        }
        __syncwarp();
    }
    const uint32_t f1 = (m1 ^ ((prev2 ^ (prev2 >> 30)) * 1566083941u)) - 1u;
    if (on) {
        states[s * kMtN + 0] = 0x80000000u;
        states[s * kMtN + 1] = f1;
    }
}

}  // namespace bbe
