// race_kernel.cuh -- sm_100a kernels for the batched Monte Carlo race continuation.
//
// Reference semantics (all /root/reference/pkg/src/racemarket/race.py):
//   :93-96   responsiveness: early_mult if pos < breakpoint*L else late_mult
//   :233-241 initial_state: positions 0, prev[c] = resp(0)*pref*draw (index order)   [from_start]
//   :244-264 _front_runner: nearest STILL-RACING rival STRICTLY ahead; equal gaps -> lowest index
//   :267-274 _resolve_step: free (no front, or gap > theta): (resp*pref)*draw, consumes a draw;
//            blocked: resp*min(prev_c, prev_front), consumes nothing
//   :287-320 advance_race: synchronous; p = pos+step; p==pos -> nextafter(p,+inf); prev = step;
//            finish tick = t if p >= L
//   :323-332 _finish_order: sort by (finish_tick, L - pos, index)
//   :381-386 / :402-404 tick-limit check before each advance (absolute / relative)
//
// Execution mapping (B200, 148 SMs, 32-lane warps):
//   * One race ("sim") occupies a SEGMENT of W consecutive lanes of a warp; each lane holds K
//     competitors ("slots"): competitor c = k*W + l lives in lane l, slot k.  S = 32/W segments
//     (independent sims) share a warp, so a 10-runner field packs 3 sims per warp.
//   * Front runner, NATIVE: every lane publishes an order-preserving u32 key of its start-of-tick
//     position to a per-warp shared-memory row (double-buffered by tick parity, one __syncwarp);
//     each lane then reads its segment's keys with 128-bit broadcast loads and keeps
//     min((key_r - key_c - 1) mod 2^32) -- one IADD + one IMNMX per rival: the wrap sends every
//     rival at or behind c (and every finished rival, key 0) above every rival ahead, so the
//     minimum is the nearest position strictly ahead.  The front's index (needed only for a
//     blocked step) is recovered by a second pass that runs only when some lane is blocked.
//   * Front runner, INJECT (FP64, bit-exact): the reference's own arithmetic -- gap = p_i - p_c
//     in double, strict compares in index order -- over __shfl_sync'd rival positions.
//   * Finish/termination: __ballot_sync over "still racing" masks; a finished segment is
//     re-filled with its next sim at a 4-tick block boundary (persistent grid, sims strided).
//   * Draws: NATIVE = Philox4x32-10 keyed by the request seed, counter = (tick block, competitor,
//     global sim index) -> 4 draws per call per lane, independent of grid shape or GPU count;
//     INJECT = recorded reference draws read from a CSR stream, per-lane offset = popc of free
//     slots before it in competitor-index order (exactly the reference's consumption order).
//   * Tallies: per-block shared-memory histograms (wins, ranks, perms), one atomic flush per block.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace bbe {

constexpr int kWarp = 32;
constexpr int kBlockThreads = 128;
constexpr int kWarpsPerBlock = kBlockThreads / kWarp;
constexpr int kTicksPerBlock = 4;  // Philox4x32 yields 4 words per call: one per tick

// Parameter block fields (SoA, stride n), host-packed in double (see bbe_sim.cu: pack_params).
enum Field {
    F_LO = 0, F_SPAN, F_LMU, F_SIGMA, F_SCALE, F_MU, F_RP_EARLY, F_RP_LATE, F_EARLY, F_LATE, F_BP,
    F_THETA, F_POS0, F_PREV0, F_FIN0, F_FAMILY,
    F_FINREL,  // finish tick relative to the state's tick, order-compressed to int32 (racing: unused)
    F_COUNT
};

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

// NATIVE-only FP32 parameter block (SoA, stride n), derived on the host from the double block.
enum FieldF {
    NF_LO_MINUS_SPAN = 0,  // uniform: lo + span*u == (lo - span) + span*(1 + u), u from the exponent trick
    NF_SPAN, NF_SG2, NF_LMU2,  // lognormal: exp2(sg2 * z + lmu2) == scale * exp(mu + sigma z)
    NF_RP_EARLY, NF_RP_LATE, NF_EARLY, NF_LATE, NF_BP, NF_THETA, NF_POS0, NF_PREV0, NF_COUNT
};

struct LaunchArgs {
    const double* P;  // [F_COUNT][n] parameter block
    const float* Pf;  // [NF_COUNT][n] (NATIVE)
    uint32_t rk[20];  // Philox4x32-10 round keys of the seed (NATIVE)
    float shift;      // NATIVE: positions, L and breakpoints are offset by this to keep positions >= 0
    int n, W, S, WP, from_start, scan, perms;
    double L;
    int64_t tick0;
    int32_t limit;  // tick_limit clamped to int32 (ticks run per sim)
    int64_t n_sims, sim_offset;
    uint64_t seed;
    const double* draws;          // INJECT
    const int64_t* draw_offsets;  // INJECT [n_sims+1]
    uint64_t* tally;              // device, TallyLayout
    int32_t* winner;              // optional per-sim outputs
    int32_t* order;
    int64_t* finish_ticks;
    double* final_pos;
    int64_t* blocked;
    int64_t* draws_used;
};

// Dynamic shared memory of one block: histograms, then (NATIVE) the key rows.
__host__ __device__ inline int key_row_words(int K, int S, int WP) { return K * S * WP; }
// NATIVE key rows use a compile-time slot stride: the largest S*WP any W in (4(CH-1), 4CH] needs.
__host__ __device__ constexpr int swp_max(int CH) {
    return CH == 1 ? 128 : (CH == 2 ? 48 : (CH == 3 ? 36 : (CH == 4 ? 32 : 4 * CH)));
}
// +4: a padding word group at the end of every slot row, where lanes without a segment write.
__host__ __device__ constexpr int native_slot_words(int CH) { return swp_max(CH) + 4; }
__host__ __device__ constexpr int native_warp_words(int K, int CH) { return 2 * K * native_slot_words(CH); }
__host__ __device__ inline size_t smem_bytes(int mode_native, int hist_len, int K, int S, int WP) {
    size_t b = (size_t)hist_len * 8;
    if (mode_native) b += (size_t)kWarpsPerBlock * native_warp_words(K, (WP + 3) / 4) * 4;
    return b;
}

// ------------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11), in registers.
// ------------------------------------------------------------------------------------------------
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// [0,1) with 23 random bits, via the exponent trick (no I2F on the hot path).
__device__ __forceinline__ float u01_23(uint32_t w) { return __uint_as_float(0x3f800000u | (w >> 9)) - 1.0f; }
// (0,1] for the Box-Muller log.
__device__ __forceinline__ float u01_open0(uint32_t w) { return 1.0f - u01_23(w); }

// Order-preserving float <-> u32 key (total order of non-NaN floats; key 0 is never a real position).
__device__ __forceinline__ uint32_t key_of(float x) {
    const uint32_t b = __float_as_uint(x);
    return b ^ ((uint32_t)((int32_t)b >> 31) | 0x80000000u);
}
__device__ __forceinline__ float float_of_key(uint32_t k) {
    return __uint_as_float(k ^ (((int32_t)k < 0) ? 0x80000000u : 0xffffffffu));
}

template <typename Real> struct RealOps;
template <> struct RealOps<float> {
    static __device__ __forceinline__ float inf() { return CUDART_INF_F; }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float next_up(float p) { return nextafterf(p, CUDART_INF_F); }
};
template <> struct RealOps<double> {
    static __device__ __forceinline__ double inf() { return CUDART_INF; }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double next_up(double p) { return nextafter(p, CUDART_INF); }
};

template <typename T>
__device__ __forceinline__ T shfl(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }

enum Mode { NATIVE = 0, INJECT = 1 };

// ------------------------------------------------------------------------------------------------
// The race kernel.  K = competitors per lane (slots); CH = 128-bit key chunks per segment row
// (NATIVE; W <= 4*CH).  Persistent: grid sized to residency, sims strided over segments.
// ------------------------------------------------------------------------------------------------
template <typename Real, int K, int MODE, int CH>
__global__ void __launch_bounds__(kBlockThreads, MODE == NATIVE ? (K == 1 ? 8 : (K == 2 ? 5 : 3)) : 1)
race_kernel(const LaunchArgs a) {
    using R = RealOps<Real>;
    extern __shared__ __align__(16) unsigned long long s_dyn[];
    const TallyLayout TL{a.n, a.perms};
    const int hist_len = TL.hist_len();
    unsigned long long* s_hist = s_dyn;
    for (int i = threadIdx.x; i < hist_len; i += blockDim.x) s_hist[i] = 0ull;

    const int n = a.n, W = a.W, S = a.S;
    const int lane = threadIdx.x & (kWarp - 1);
    const int warp = threadIdx.x >> 5;
    const int seg = lane / W;
    const bool lane_on = seg < S;
    const int base = lane_on ? seg * W : 0;
    const int l = lane - seg * W;
    const unsigned segmask = lane_on ? ((W == 32 ? 0xffffffffu : ((1u << W) - 1u)) << base) : 0u;
    const unsigned lt_mask = (1u << lane) - 1u;

    // NATIVE key rows: [warp][parity][slot][segment * WP + lane-in-segment]
    const int row_words = key_row_words(K, S, a.WP);
    uint32_t* s_keys = reinterpret_cast<uint32_t*>(s_dyn + ((hist_len + 1) & ~1));  // 16-B aligned
    uint32_t* my_rows = s_keys + warp * 2 * row_words;
    const int seg_off = lane_on ? seg * a.WP : 0;
    if (MODE == NATIVE) {
        for (int i = lane; i < 2 * row_words; i += kWarp) my_rows[i] = 0u;  // pads stay "behind"
    }
    __syncthreads();

    // ---- per-slot constants (loaded once: the lane->competitor map is fixed for the kernel) ----
    int cidx[K];
    bool has[K];
    Real lo[K], span[K], lmu[K], sigma[K], rp_early[K], rp_late[K], early[K], late[K], bp[K], theta[K];
    Real pos0[K], prev0[K];
    int64_t fin0[K];
    bool lognorm[K];
    const double* P = a.P;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int c = k * W + l;
        cidx[k] = c;
        has[k] = lane_on && c < n;
        const int cc = has[k] ? c : 0;
        lo[k] = (Real)P[F_LO * n + cc];
        span[k] = (Real)P[F_SPAN * n + cc];
        lmu[k] = (Real)P[F_LMU * n + cc];
        sigma[k] = (Real)P[F_SIGMA * n + cc];
        rp_early[k] = (Real)P[F_RP_EARLY * n + cc];
        rp_late[k] = (Real)P[F_RP_LATE * n + cc];
        early[k] = (Real)P[F_EARLY * n + cc];
        late[k] = (Real)P[F_LATE * n + cc];
        bp[k] = (Real)P[F_BP * n + cc];
        theta[k] = (Real)P[F_THETA * n + cc];
        pos0[k] = (Real)P[F_POS0 * n + cc];
        prev0[k] = (Real)P[F_PREV0 * n + cc];
        fin0[k] = has[k] ? (int64_t)P[F_FIN0 * n + cc] : INT64_MAX;
        lognorm[k] = P[F_FAMILY * n + cc] != 0.0;
    }
    const Real L = (Real)a.L;
    const Real NEG_INF = -R::inf();
    bool any_lognorm = false;
#pragma unroll
    for (int k = 0; k < K; ++k) any_lognorm |= has[k] && lognorm[k];
    any_lognorm = __any_sync(0xffffffffu, any_lognorm);

    // ---- segment bookkeeping (replicated in every lane of the segment) ----
    const int64_t warps_total = (int64_t)gridDim.x * kWarpsPerBlock;
    const int64_t gwarp = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
    const int64_t segs_total = warps_total * S;
    int64_t s = lane_on ? gwarp * S + seg : a.n_sims;  // local sim index
    const int64_t start = a.tick0;
    int32_t rt = 0;                      // ticks advanced in the current sim
    int64_t cursor = 0, cursor_end = 0;  // INJECT
    bool running = false, diverged = false, bad = false;
    const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);

    Real pos[K], prev[K], pv[K];
    int64_t fin[K];
    bool racing[K];
    Real rawd[K][kTicksPerBlock];
    uint32_t ct_sim = 0, blk_sim = 0;            // this lane's slots, current sim
    unsigned long long ct_tot = 0, blk_tot = 0;  // this lane, whole kernel
    unsigned long long n_div = 0, n_bad = 0;
    int64_t first_div = INT64_MAX, first_bad = INT64_MAX;

    // refill: load the (local) sim s into the segment
    auto load_sim = [&](bool do_it) {
        if (!do_it) return;
        running = lane_on && s < a.n_sims;
        diverged = false;
        bad = false;
        rt = 0;
        ct_sim = blk_sim = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            pos[k] = pos0[k];
            prev[k] = prev0[k];
            fin[k] = fin0[k];
            racing[k] = running && has[k] && fin0[k] < 0;
        }
        if (MODE == INJECT && running) {
            cursor = a.draw_offsets[s];
            cursor_end = a.draw_offsets[s + 1];
        }
        if (a.from_start && running) {
            // race.py:233-241: one free draw per competitor in index order, resp at position 0
            const uint64_t gs = (uint64_t)(a.sim_offset + s);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (!has[k]) continue;
                Real d;
                if (MODE == INJECT) {
                    const int64_t at = cursor + cidx[k];
                    d = at < cursor_end ? (Real)a.draws[at] : (Real)1;
                } else {
                    const U4 w = philox4x32_10(U4{0xFFFFFFFFu, (uint32_t)cidx[k], (uint32_t)gs, (uint32_t)(gs >> 32)},
                                               k0, k1);
                    if (lognorm[k]) {
                        const float r = sqrtf(-2.0f * __logf(u01_open0(w.x)));
                        const float z = r * __cosf(6.283185307f * u01_23(w.y));
                        d = (Real)__expf(fmaf((float)sigma[k], z, (float)lmu[k]));
                    } else {
                        d = lo[k] + span[k] * (Real)u01_23(w.x);
                    }
                }
                const Real rp = ((Real)0 < bp[k]) ? rp_early[k] : rp_late[k];
                prev[k] = R::mul(rp, d);
            }
            if (MODE == INJECT) {
                if (cursor + n > cursor_end) bad = true;  // stream shorter than the priming draws
                cursor += n;
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) pv[k] = racing[k] ? pos[k] : NEG_INF;
    };

    load_sim(true);

    while (true) {
        // ---------------- block boundary: finalize finished segments, refill, exit test ----------
        bool seg_live = false;
#pragma unroll
        for (int k = 0; k < K; ++k) seg_live |= racing[k];
        const unsigned live_mask = __ballot_sync(0xffffffffu, seg_live);
        const bool seg_done = running && ((live_mask & segmask) == 0u);
        if (__any_sync(0xffffffffu, seg_done)) {
            // ---- finalize (warp-uniform; results used only where seg_done) ----
            Real lp[K];
            int rank[K];
#pragma unroll
            for (int k = 0; k < K; ++k) { lp[k] = R::sub(L, pos[k]); rank[k] = 0; }
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
                for (int j = 0; j < W; ++j) {
                    const int64_t fr = shfl(fin[kk], base + j);
                    const Real dr = shfl(lp[kk], base + j);
                    const int i = kk * W + j;
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const bool less = fr < fin[k] || (fr == fin[k] && (dr < lp[k] || (dr == lp[k] && i < cidx[k])));
                        rank[k] += (i < n && less) ? 1 : 0;
                    }
                }
            }
            // per-sim blocked count: segment sum of the lanes' counters
            uint32_t seg_blk = 0;
            for (int j = 0; j < W; ++j) seg_blk += shfl(blk_sim, base + j);
            int64_t lehmer = 0;
            if (a.perms) {
                // Lehmer index of the finish order: sum_c #{c' < c : rank(c') > rank(c)} * (n-1-rank(c))!
                int cnt[K];
#pragma unroll
                for (int k = 0; k < K; ++k) cnt[k] = 0;
#pragma unroll
                for (int kk = 0; kk < K; ++kk)
                    for (int j = 0; j < W; ++j) {
                        const int rr = shfl(rank[kk], base + j);
                        const int i = kk * W + j;
#pragma unroll
                        for (int k = 0; k < K; ++k) cnt[k] += (i < n && i < cidx[k] && rr > rank[k]) ? 1 : 0;
                    }
                int64_t term = 0;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (!has[k]) continue;
                    int64_t f = 1;
                    for (int q = 2; q <= n - 1 - rank[k]; ++q) f *= q;
                    term += cnt[k] * f;
                }
                for (int j = 0; j < W; ++j) lehmer += shfl(term, base + j);
            }
            if (seg_done) {
                const int64_t gs = a.sim_offset + s;
                if (MODE == INJECT) bad = bad || cursor != cursor_end;
                if (diverged) {
                    if (l == 0) { n_div++; first_div = min(first_div, gs); }
                } else if (bad) {
                    if (l == 0) { n_bad++; first_bad = min(first_bad, gs); }
                } else {
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        if (!has[k]) continue;
                        if (rank[k] == 0) atomicAdd(&s_hist[TL.wins() + cidx[k]], 1ull);
                        atomicAdd(&s_hist[TL.ranks() + cidx[k] * n + rank[k]], 1ull);
                    }
                    if (a.perms && l == 0) atomicAdd(&s_hist[TL.perms() + lehmer], 1ull);
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (!has[k]) continue;
                    const int64_t o = s * n + cidx[k];
                    if (a.winner && rank[k] == 0) a.winner[s] = diverged ? -1 : cidx[k];
                    if (a.order) a.order[s * n + rank[k]] = cidx[k];
                    if (a.finish_ticks) a.finish_ticks[o] = fin[k] == INT64_MAX ? -1 : fin[k];
                    if (a.final_pos) a.final_pos[o] = (double)pos[k];
                }
                if (l == 0) {
                    if (a.blocked) a.blocked[s] = seg_blk;
                    if (MODE == INJECT && a.draws_used) a.draws_used[s] = cursor - a.draw_offsets[s];
                }
                ct_tot += ct_sim;
                blk_tot += blk_sim;
                s += segs_total;
            }
            load_sim(seg_done);
        }
        if (!__any_sync(0xffffffffu, running)) break;

        // ---------------- NATIVE: 4 draws per slot for this tick block (counter = tick block) ----
        if (MODE == NATIVE) {
            __syncwarp();  // key rows: reads of the previous block precede this block's writes
            const uint64_t gs = (uint64_t)(a.sim_offset + s);
            const uint32_t blk = (uint32_t)rt >> 2;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const U4 w = philox4x32_10(U4{blk, (uint32_t)cidx[k], (uint32_t)gs, (uint32_t)(gs >> 32)}, k0, k1);
                if (any_lognorm && lognorm[k]) {
                    const float r0 = sqrtf(-2.0f * __logf(u01_open0(w.x)));
                    const float r1 = sqrtf(-2.0f * __logf(u01_open0(w.z)));
                    float s0, c0, s1, c1;
                    __sincosf(6.283185307f * u01_23(w.y), &s0, &c0);
                    __sincosf(6.283185307f * u01_23(w.w), &s1, &c1);
                    const float sg = (float)sigma[k], mu = (float)lmu[k];
                    rawd[k][0] = (Real)__expf(fmaf(sg, r0 * c0, mu));
                    rawd[k][1] = (Real)__expf(fmaf(sg, r0 * s0, mu));
                    rawd[k][2] = (Real)__expf(fmaf(sg, r1 * c1, mu));
                    rawd[k][3] = (Real)__expf(fmaf(sg, r1 * s1, mu));
                } else {
                    rawd[k][0] = fmaf((float)span[k], u01_23(w.x), (float)lo[k]);
                    rawd[k][1] = fmaf((float)span[k], u01_23(w.y), (float)lo[k]);
                    rawd[k][2] = fmaf((float)span[k], u01_23(w.z), (float)lo[k]);
                    rawd[k][3] = fmaf((float)span[k], u01_23(w.w), (float)lo[k]);
                }
            }
        }

        // ---------------- 4 synchronous ticks -------------------------------------------------------
#pragma unroll
        for (int tj = 0; tj < kTicksPerBlock; ++tj) {
            bool any_racing = false;
#pragma unroll
            for (int k = 0; k < K; ++k) any_racing |= racing[k];
            const unsigned rmask = __ballot_sync(0xffffffffu, any_racing);
            const bool seg_running = (rmask & segmask) != 0u;
            if (rmask == 0u) break;  // every segment finished inside this block

            // tick-limit check before the advance (race.py:381-386, 402-404)
            if (seg_running && rt >= a.limit) {
                diverged = true;
#pragma unroll
                for (int k = 0; k < K; ++k) { racing[k] = false; pv[k] = NEG_INF; }
            }

            // ---- front runner (race.py:244-264) ----
            Real gap[K];
            int bi[K];
            uint32_t fkey[K];
#pragma unroll
            for (int k = 0; k < K; ++k) { gap[k] = R::inf(); bi[k] = 0; fkey[k] = 0u; }
            if (a.scan) {
                if constexpr (MODE == NATIVE) {
                    uint32_t* row = my_rows + (tj & 1) * row_words;
                    uint32_t kp[K], nk[K], best[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        kp[k] = key_of((float)pos[k]);
                        nk[k] = ~kp[k];
                        best[k] = 0xffffffffu;
                        if (lane_on) row[k * S * a.WP + seg_off + l] = racing[k] ? kp[k] : 0u;
                    }
                    __syncwarp();
#pragma unroll
                    for (int kk = 0; kk < K; ++kk) {
                        const uint4* r4 = reinterpret_cast<const uint4*>(row + kk * S * a.WP + seg_off);
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            const uint4 v = r4[c];
#pragma unroll
                            for (int k = 0; k < K; ++k) {
                                best[k] = min(best[k], v.x + nk[k]);
                                best[k] = min(best[k], v.y + nk[k]);
                                best[k] = min(best[k], v.z + nk[k]);
                                best[k] = min(best[k], v.w + nk[k]);
                            }
                        }
                    }
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const uint32_t fk = best[k] - nk[k];  // = best + key_c + 1 (mod 2^32)
                        const bool ahead = fk > kp[k];        // no wrap <=> a rival strictly ahead
                        fkey[k] = ahead ? fk : 0u;
                        gap[k] = ahead ? R::sub((Real)float_of_key(fk), pos[k]) : R::inf();
                    }
                } else {
                    // exact reference arithmetic: gap = p_i - p_c, strict compares in index order
#pragma unroll
                    for (int kk = 0; kk < K; ++kk) {
#pragma unroll 2
                        for (int j = 0; j < W; ++j) {
                            const Real pr = shfl(pv[kk], base + j);
#pragma unroll
                            for (int k = 0; k < K; ++k) {
                                const Real g = R::sub(pr, pos[k]);
                                const bool t = (g > (Real)0) & (g < gap[k]);
                                gap[k] = t ? g : gap[k];
                                bi[k] = t ? (kk << 5) | j : bi[k];
                            }
                        }
                    }
                }
            }

            // ---- step resolution (race.py:267-274) ----
            bool fr[K], bl[K];
            bool any_blocked = false;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                fr[k] = racing[k] && gap[k] > theta[k];
                bl[k] = racing[k] && !fr[k];
                any_blocked |= bl[k];
            }
            Real pf[K];
#pragma unroll
            for (int k = 0; k < K; ++k) pf[k] = (Real)0;
            if (__any_sync(0xffffffffu, any_blocked)) {
                if constexpr (MODE == NATIVE) {
                    // lowest competitor index whose key is the front key (slot-major, then lane)
                    const uint32_t* row = my_rows + (tj & 1) * row_words;
#pragma unroll
                    for (int kk = K - 1; kk >= 0; --kk) {
                        const uint4* r4 = reinterpret_cast<const uint4*>(row + kk * S * a.WP + seg_off);
#pragma unroll
                        for (int c = CH - 1; c >= 0; --c) {
                            const uint4 v = r4[c];
#pragma unroll
                            for (int k = 0; k < K; ++k) {
                                bi[k] = (v.w == fkey[k]) ? (kk << 5) | (4 * c + 3) : bi[k];
                                bi[k] = (v.z == fkey[k]) ? (kk << 5) | (4 * c + 2) : bi[k];
                                bi[k] = (v.y == fkey[k]) ? (kk << 5) | (4 * c + 1) : bi[k];
                                bi[k] = (v.x == fkey[k]) ? (kk << 5) | (4 * c + 0) : bi[k];
                            }
                        }
                    }
                }
#pragma unroll
                for (int kk = 0; kk < K; ++kk) {
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const Real v = shfl(prev[kk], base + (bi[k] & 31));
                        pf[k] = ((bi[k] >> 5) == kk) ? v : pf[k];
                    }
                }
            }
            Real draw[K];
            if constexpr (MODE == INJECT) {
                // free slots consume the stream in competitor-index order (slot-major, then lane):
                // offset = free slots of lower index in this segment = popc of the ballot below me
                int seg_total = 0;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const unsigned fm = __ballot_sync(0xffffffffu, fr[k]) & segmask;
                    const int64_t at = cursor + seg_total + __popc(fm & lt_mask);
                    draw[k] = (fr[k] && at < cursor_end) ? (Real)__ldg(a.draws + at) : (Real)1;
                    seg_total += __popc(fm);
                }
                cursor += seg_total;
                if (cursor > cursor_end) {  // stream too short: stop this sim, report at finalize
                    bad = true;
#pragma unroll
                    for (int k = 0; k < K; ++k) { racing[k] = false; fr[k] = bl[k] = false; }
                }
            } else {
#pragma unroll
                for (int k = 0; k < K; ++k) draw[k] = rawd[k][tj];
            }

            // ---- synchronous update (race.py:299-320) ----
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const bool early_phase = pos[k] < bp[k];
                Real step;
                if (fr[k]) {
                    step = R::mul(early_phase ? rp_early[k] : rp_late[k], draw[k]);
                } else {
                    const Real m = (pf[k] < prev[k]) ? pf[k] : prev[k];  // Python min(prev_c, prev_front)
                    step = R::mul(early_phase ? early[k] : late[k], m);
                }
                if (racing[k]) {
                    Real p = R::add(pos[k], step);
                    if (p == pos[k]) p = R::next_up(p);
                    pos[k] = p;
                    prev[k] = step;
                    ct_sim += 1;
                    blk_sim += bl[k] ? 1 : 0;
                    if (p >= L) { fin[k] = start + rt + 1; racing[k] = false; }
                }
                if (MODE == INJECT) pv[k] = racing[k] ? pos[k] : NEG_INF;
            }
            if (seg_running && !diverged) rt += 1;
        }
    }

    // ---------------- flush: per-lane totals -> warp -> global; block histograms -> global ------
    unsigned long long v_ct = ct_tot, v_blk = blk_tot, v_div = n_div, v_bad = n_bad;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        v_ct += __shfl_xor_sync(0xffffffffu, v_ct, off);
        v_blk += __shfl_xor_sync(0xffffffffu, v_blk, off);
        v_div += __shfl_xor_sync(0xffffffffu, v_div, off);
        v_bad += __shfl_xor_sync(0xffffffffu, v_bad, off);
        first_div = min(first_div, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)first_div, off));
        first_bad = min(first_bad, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)first_bad, off));
    }
    const int ct_at = TL.ct();
    if (lane == 0) {
        if (v_ct) atomicAdd((unsigned long long*)&a.tally[ct_at + 0], v_ct);
        if (v_blk) atomicAdd((unsigned long long*)&a.tally[ct_at + 1], v_blk);
        if (v_div) atomicAdd((unsigned long long*)&a.tally[ct_at + 2], v_div);
        if (v_bad) atomicAdd((unsigned long long*)&a.tally[ct_at + 3], v_bad);
        // first_* stored as ~(index + 1) so that MAX picks the smallest index and 0 means none
        if (first_div != INT64_MAX)
            atomicMax((unsigned long long*)&a.tally[ct_at + 4], encode_first(first_div));
        if (first_bad != INT64_MAX)
            atomicMax((unsigned long long*)&a.tally[ct_at + 5], encode_first(first_bad));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < hist_len; i += blockDim.x) {
        const unsigned long long v = s_hist[i];
        if (v) atomicAdd((unsigned long long*)&a.tally[i], v);
    }
}

}  // namespace bbe
