// common.cuh -- shared definitions of the race kernels (parameter blocks, tally layout, launch
// arguments, Philox4x32-10, warp helpers).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

// BBE_CHECKS builds (tools/ab_build.sh checks "-DBBE_CHECKS"): device-side bounds asserts on every
// shared-memory index the kernels compute (MT stream window, key rows, staged draws, histograms) --
// the bounds evidence on a pool where compute-sanitizer is closed.  Off in the product build.
#ifdef BBE_CHECKS
#include <cassert>
#define BBE_CHECK(cond) assert(cond)
#else
#define BBE_CHECK(cond) ((void)0)
#endif

namespace bbe {

// the block's dynamic shared memory size in bytes (%dynamic_smem_size), for BBE_CHECK
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
    uint32_t v;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
    return v;
}
template <typename T>
__device__ __forceinline__ bool in_dyn_smem(const T* p, const void* base) {
    const char* c = reinterpret_cast<const char*>(p);
    const char* b = reinterpret_cast<const char*>(base);
    return c >= b && c + sizeof(T) <= b + dyn_smem_bytes();
}

constexpr int kWarp = 32;
constexpr int kBlockThreads = 128;
constexpr int kWarpsPerBlock = kBlockThreads / kWarp;
#ifndef BBE_EXACT_TICKS
#define BBE_EXACT_TICKS 8  // C2 MT: 4 -> 2.54 ms, 8 -> 2.43, 16 -> 2.42 (bit-identical; 8 idles less on short races)
#endif
#ifndef BBE_N64_SCAN_NT
#define BBE_N64_SCAN_NT 16  // NATIVE64 layouts with a front-runner scan: ticks per block (A/B, ms:
                            // 8 -> 16: C2 0.667 -> 0.653, derby20 29.25 -> 28.12, derby12 17.85 -> 15.25)
#endif
constexpr int kTicksPerBlock = BBE_EXACT_TICKS;  // exact kernels: ticks between finalize/refill boundaries

// Parameter block fields (SoA, stride n), host-packed in double (see bbe_sim.cu: pack_params).
enum Field {
    F_LO = 0, F_SPAN, F_LMU, F_SIGMA, F_SCALE, F_MU, F_RP_EARLY, F_RP_LATE, F_EARLY, F_LATE, F_BP,
    F_THETA, F_POS0, F_PREV0, F_FIN0, F_FAMILY,
    F_FINREL,  // finish tick relative to the state's tick, order-compressed to int32 (racing: unused)
    F_COUNT
};

// NATIVE-only FP32 parameter block (SoA, stride n), derived on the host from the double block.
enum FieldF {
    NF_LO_MINUS_SPAN = 0,  // uniform: lo + span*u == (lo - span) + span*(1 + u), u from the exponent trick
    NF_SPAN, NF_SG2, NF_LMU2,  // lognormal: exp2(sg2 * z + lmu2) == scale * exp(mu + sigma z)
    NF_RP_EARLY, NF_RP_LATE, NF_EARLY, NF_LATE, NF_BP, NF_THETA, NF_POS0, NF_PREV0, NF_COUNT
};

enum Mode { NATIVE = 0, INJECT = 1, MT = 2, NATIVE64 = 3 };

// "First failing sim" tally fields hold (2^63 - 1) - index (0 = none): a MAX reduction -- atomicMax
// in a kernel, or a signed int64 all-reduce across ranks -- then keeps the smallest index.
__host__ __device__ inline unsigned long long encode_first(int64_t index) {
    return 0x7fffffffffffffffull - (unsigned long long)index;
}
__host__ __device__ inline int64_t decode_first(unsigned long long v) {
    return v ? (int64_t)(0x7fffffffffffffffull - v) : -1;
}

// Tally layout in u64 (see bbe_tally_offset in bbe_sim.h).
struct TallyLayout {
    int n, nperm;
    __host__ __device__ int wins() const { return 0; }
    __host__ __device__ int ranks() const { return n; }
    __host__ __device__ int perms() const { return n + n * n; }
    __host__ __device__ int ct() const { return n + n * n + nperm; }
    __host__ __device__ int blocked() const { return ct() + 1; }
    __host__ __device__ int n_div() const { return ct() + 2; }
    __host__ __device__ int n_bad() const { return ct() + 3; }
    __host__ __device__ int first_div() const { return ct() + 4; }
    __host__ __device__ int first_bad() const { return ct() + 5; }
    __host__ __device__ int len() const { return ct() + 6; }
    __host__ __device__ int hist_len() const { return n + n * n + nperm; }  // shared-memory histograms
};

struct LaunchArgs {
    const double* P;  // [F_COUNT][n] parameter block
    const float* Pf;  // [NF_COUNT][n] (NATIVE)
    uint32_t rk[20];  // Philox4x32-10 round keys of the seed (NATIVE)
    float shift;      // NATIVE: positions, L and breakpoints are offset by this (the front-runner frame)
    uint32_t key_base;  // NATIVE: front-runner key = float bits of a position - key_base
    int key_bits;       // NATIVE: index bits packed under the key
    double key_c64;       // NATIVE64: coarse front-runner key = mantissa bits 51..26 of (pos + key_c64)
    uint32_t key_sub64;   //   (the constant exponent bit the 32-bit key window drags in, subtracted)
    int n64_flags;        // NATIVE64: kN64RespVar | kN64Guard (bbe_sim.cu native64_flags)
    uint32_t key_mul, key_nmul;  // NATIVE: 2^key_bits and -2^key_bits (runtime values: IMAD, not shifts)
    int n, W, S, WP, from_start, scan, perms;
    double L;
    int64_t tick0;
    int32_t limit;  // tick_limit clamped to int32 (ticks run per sim)
    int64_t n_sims, sim_offset;
    uint64_t seed;
    const double* draws;          // INJECT
    const int64_t* draw_offsets;  // INJECT [n_sims+1]
    const uint32_t* mt_states;    // MT: [n_sims][624] seeded MT19937 states
    double nv_magic;              // MT: random.NV_MAGICCONST = 4*exp(-0.5)/sqrt(2.0), host libm
    double* traj_pos;             // exact modes, optional: [n_sims][traj_cap+1][n] positions per tick
    double* traj_prev;            //   and previous steps (run_race(record=True), race.py:378-389)
    int32_t traj_cap;             //   ticks recorded per sim (longer sims are reported via n_ticks)
    uint64_t* tally;              // device, TallyLayout
    unsigned long long* work;     // [0] sims claimed after the first round, [1] blocks done (zeroed)
    int32_t* winner;              // optional per-sim outputs
    int32_t* order;
    int64_t* finish_ticks;
    double* final_pos;
    int64_t* blocked;
    int64_t* draws_used;
    unsigned long long* group_wins;  // optional [groups][n]: winners of sims (group_base + s) / group_size
    int64_t group_size, group_base;
};

// ---- dynamic shared memory ----
// NATIVE key rows: a segment's row holds WP = VEC*CH keys (W rounded up to the load width VEC, 4 or
// 2 words).  The slot stride is compile-time: the largest S*WP any W in (VEC(CH-1), VEC*CH] needs,
// +4 for a padding word group at the end of every slot row (where lanes without a segment write).
__host__ __device__ constexpr int swp_max(int VEC, int CH) {
    int m = 0;
    for (int w = VEC * (CH - 1) + 1; w <= VEC * CH && w <= 32; ++w) m = (32 / w) * VEC * CH > m ? (32 / w) * VEC * CH : m;
    return m;
}
__host__ __device__ constexpr int native_slot_words(int VEC, int CH) { return swp_max(VEC, CH) + 4; }
__host__ __device__ constexpr int native_warp_words(int K, int VEC, int CH) { return 2 * K * native_slot_words(VEC, CH); }
constexpr int kMtWords = 624;
// MT trial-evaluation pass (K = 1): a pending lognormal draw evaluates up to this many speculative
// Kinderman-Monahan trials at once, on otherwise idle lanes of its segment
constexpr int kMtMaxTrials = 8;
// side buffer: >= one round's reads -- 4 words x 32 lanes x K slots, + the trial window's overhang
__host__ __device__ constexpr int mt_side_words(int K) { return 128 * K + 4 * kMtMaxTrials; }
__host__ __device__ constexpr int mt_seg_words(int K) { return kMtWords + mt_side_words(K); }
constexpr int kXSlot = 66;         // exact modes: doubles per position row (S*round_up(W,2) <= 64, + pad)
// NATIVE64 host flags
constexpr int kN64RespVar = 1;  // some competitor's early and late multipliers differ
constexpr int kN64Guard = 2;    // fl(pos + step) == pos is possible: keep the nextafter guard
constexpr int kN64NoTie = 4;    // no blocked lane can face a gap-rounding tie (every racing position > 2 max theta)
__host__ __device__ inline size_t smem_bytes(int mode, int hist_len_even, int K, int S, int WP, int nt64 = 0) {
    size_t b = (size_t)hist_len_even * 8;
    if (mode == NATIVE || (mode == NATIVE64 && WP > 0)) {  // NATIVE64 scan-free kernels: no key rows (WP 0)
        const int vec = (WP % 4) ? 2 : 4;  // the host rounds W up to 2 (VEC 2) or 4 (VEC 4)
        b += (size_t)kWarpsPerBlock * native_warp_words(K, vec, WP / vec) * 4;
    }
    if (mode == NATIVE64) b += (size_t)kWarpsPerBlock * K * nt64 * kWarp * 8;  // staged draws
    if (mode == MT) b += (size_t)kWarpsPerBlock * S * mt_seg_words(K) * 4;
    if (mode == INJECT || mode == MT) b += (size_t)kWarpsPerBlock * 2 * K * kXSlot * 8;
    if (mode == MT) b += (size_t)kWarpsPerBlock * kWarp * 4;  // per-warp lognormal offsets (trial pass)
    return b;
}

// ---- Philox4x32-10 (Salmon et al., SC'11), in registers ----
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox_rk(U4 c, const uint32_t* rk) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = U4{hi1 ^ c.y ^ rk[2 * r], lo1, hi0 ^ c.w ^ rk[2 * r + 1], lo0};
    }
    return c;
}

// random_random(): m * 2^-53 with m = a*2^26 + b, a = w0>>5, b = w1>>6 -- an exact 53-bit fraction
// (CPython _randommodule.c), built from bits without integer->double conversions (bit 52 of m is bit
// 31 of w0).
__device__ __forceinline__ double random53(uint32_t w0, uint32_t w1) {
    const uint32_t lo = ((w0 << 21) & 0xFC000000u) | (w1 >> 6);  // m bits 0..31
    const uint32_t hi = w0 >> 11;                                  // m bits 32..52
    // as unit53: H = 0.5 + (m mod 2^52) 2^-53 from bits, m * 2^-53 = H - 0.5 + m_52 / 2: one exact DADD
    // (Sterbenz when m_52 = 0); equal to CPython's value on 2e6 random word pairs and the edge words
    return __dadd_rn(__hiloint2double((int)(0x3FE00000u | (hi & 0xFFFFFu)), (int)lo), (w0 >> 31) ? 0.0 : -0.5);
}

// NATIVE64 draws: u = m * 2^-53, m = the top 53 bits of the 64-bit word pair (w0:w1) -- uniform on
// the reference's grid k * 2^-53 (random.random()'s resolution), with fewer operations than
// random53: H = 0.5 + (m mod 2^52) * 2^-53 is built from bits, and u = H - 0.5 + m_52 / 2 is one
// exact DADD (Sterbenz when m_52 = 0).  oracle/bbe_oracle.c unit53 is the same formula.
__device__ __forceinline__ double unit53(uint32_t w0, uint32_t w1) {
    const uint32_t lo = __funnelshift_r(w1, w0, 11);            // m bits 0..31
    const uint32_t hi = 0x3FE00000u | ((w0 >> 11) & 0xFFFFFu);  // m bits 32..51 under 2^-1
    return __dadd_rn(__hiloint2double((int)hi, (int)lo), (w0 >> 31) ? 0.0 : -0.5);
}

template <typename T>
__device__ __forceinline__ T shfl(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// Finish-tick sentinels of the NATIVE kernels (int32 finish ticks relative to the state's tick).
constexpr int32_t kRacing = 0x7fffffff;
constexpr int32_t kDiverged = 0x7ffffffe;
constexpr int32_t kIdle = 0x7ffffffd;  // slot without a competitor / segment without a sim

// ---- dynamic sim assignment (persistent kernels) ----
// Every segment starts on sim `slot` (< segs_total); later sims are claimed from work[0], so a
// segment that drew short races takes more of them.  Warp-uniform call: one atomic per warp for all
// its finishing segments (leader lane = the segment's first lane, `base`).
__device__ __forceinline__ int64_t claim_next_sim(bool seg_done, bool leader, int base, int64_t segs_total,
                                                  unsigned long long* work) {
    const unsigned lead = __ballot_sync(0xffffffffu, seg_done && leader);
    const int first = __ffs(lead) - 1;
    unsigned long long got = 0;
    if ((int)(threadIdx.x & 31) == first) got = atomicAdd(work, (unsigned long long)__popc(lead));
    got = __shfl_sync(0xffffffffu, got, first < 0 ? 0 : first);
    return segs_total + (int64_t)got + __popc(lead & ((1u << base) - 1u));
}
// After the block's last claim (call from thread 0 after a __syncthreads): the last block to finish
// re-zeroes the counters for the next launch that uses this pair.
__device__ __forceinline__ void release_work(unsigned long long* work) {
    __threadfence();
    if (atomicAdd(work + 1, 1ull) == gridDim.x - 1) {
        work[0] = 0ull;
        work[1] = 0ull;
    }
}

}  // namespace bbe
