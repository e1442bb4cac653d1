// native_kernel.cuh -- the throughput kernel: Philox draws, FP32 race state (BBE_MODE_NATIVE).
//
// Same model as exact_kernel.cuh (race.py:233-332 semantics, listed there); the arithmetic is FP32
// and the random stream is Philox4x32-10, so outcomes are statistically -- not bitwise -- equal to
// the reference's.  Everything else is the reference's rule set: synchronous ticks from
// start-of-tick positions, nearest still-racing rival strictly ahead with the lowest-index tie rule,
// gap > theta => free draw scaled by (resp * pref), else resp * min(prev_c, prev_front) with no draw,
// nextafter on a zero-progress step, finish at p >= L, order by (finish tick, L - pos, index).
//
// Front runner.  The host picks a frame (an offset of positions, L and breakpoints) in which every
// racing position is >= a floor `lo` > 0 and below L with bits(L) - bits(lo) < 2^(31-b), b = 5 index
// bits.  Non-negative floats order like their IEEE bits, so key = bits(pos) - bits(lo) + 1 is an
// order-preserving (31-b)-bit key.  Each lane publishes (key << b) | lane-in-segment (0 once finished)
// to a per-warp shared-memory row (double-buffered by tick parity, one __syncwarp per tick), reads its
// segment's row with 128- or 64-bit broadcast loads (VEC) and keeps one wrapped minimum (one VIADDMNMX
// per rival) that yields the nearest key strictly ahead together with the lowest index holding it.
//
// Sims: persistent grid; each segment starts on one sim and claims the next from a per-launch counter
// at a block boundary of NT ticks (common.cuh claim_next_sim).  Bookkeeping is kept off the per-tick path:
// rt (ticks advanced in the sim) is segment-uniform; racing <=> fin == kRacing (int32 finish tick
// relative to the state's tick); the tick-limit check runs at block boundaries; competitor-timesteps
// are summed from finish ticks at finalize; finish-order ranks come from one u64 key per competitor.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace bbe {

// Build-time variants for A/B measurement (tools/ab_build.sh); the defaults are the measured best
// (C2 on B200: 8, 9 or 10 blocks/SM were slower than 7 at every step of round 1).
#ifndef BBE_SPREAD_TAIL
#define BBE_SPREAD_TAIL 1
#endif
#ifndef BBE_NATIVE_MINBLOCKS_K2
#define BBE_NATIVE_MINBLOCKS_K2 5
#endif
#ifndef BBE_NATIVE_MINBLOCKS_K1
#define BBE_NATIVE_MINBLOCKS_K1 7  // 64 registers -> 8 resident blocks of 4 warps
#endif

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 1 + u, u in [0,1) with 23 random bits (exponent trick).
__device__ __forceinline__ float one_plus_u(uint32_t w) { return __uint_as_float(0x3f800000u | (w >> 9)); }

// Box-Muller pair -> two lognormal steps exp2(sg2*z + lmu2); uniform (a, b) -> (0,1] x [0,1).
__device__ __forceinline__ void lognormal_pair(uint32_t wa, uint32_t wb, float sg2, float lmu2, float& d0, float& d1) {
    const float u1 = 2.0f - one_plus_u(wa);  // (0, 1]
    const float r = sqrt_approx(-1.3862943611198906f * lg2_approx(u1));  // sqrt(-2 ln u1)
    float s, c;
    __sincosf(6.283185307179586f * (one_plus_u(wb) - 1.0f), &s, &c);
    const float a = sg2 * r;
    d0 = ex2_approx(fmaf(a, c, lmu2));
    d1 = ex2_approx(fmaf(a, s, lmu2));
}

// SCAN = false: every theta is 0, so nobody can be blocked (gap > 0 = theta) and the front-runner
// scan's result would never be used; the kernel then omits it.
// VEC: key-row load width in words (4: LDS.128, 2: LDS.64 -- fewer padding keys when W % 4 is 1 or 2).
// NT: ticks per block (a multiple of 4: one Philox call per slot per 4 ticks).  A block boundary --
// limit check, finish ballot, refill, the next draws -- costs about 1.5 ticks' work in C2, while a
// finished segment idles (NT-1)/2 ticks on average until the next boundary, so the host picks NT
// from the race's expected remaining length (bbe_sim.cu pick_ticks).
template <int K, int CH, bool SCAN, int VEC = 4, int NT = 4>
__global__ void __launch_bounds__(kBlockThreads, K == 1 ? BBE_NATIVE_MINBLOCKS_K1 : (K == 2 ? BBE_NATIVE_MINBLOCKS_K2 : 3))
native_kernel(const LaunchArgs a) {
    static_assert(VEC == 4 || VEC == 2, "key rows are read 4 or 2 words at a time");
    extern __shared__ __align__(16) unsigned long long s_dyn[];
    const TallyLayout TL{a.n, a.perms};
    const int hist_len = TL.hist_len();
    // 32-bit shared histograms (native ATOMS.ADD; a 64-bit shared add is a CAS loop).  A block's count
    // in one bin is at most the sims of its launch, which the host keeps below 2^32 (launch_one).
    uint32_t* s_hist = reinterpret_cast<uint32_t*>(s_dyn);
    for (int i = threadIdx.x; i < hist_len; i += blockDim.x) s_hist[i] = 0u;

    constexpr int WP = VEC * CH;
    constexpr int SLOT = native_slot_words(VEC, CH);  // words per slot row (segments, then a pad group)
    constexpr int PAR = K * SLOT;       // words per parity
    const int n = a.n, W = a.W, S = a.S;
    const int lane = threadIdx.x & (kWarp - 1);
    const int warp = threadIdx.x >> 5;
    const int seg = lane / W;
    const bool lane_on = seg < S;
    const int base = lane_on ? seg * W : 0;
    const int l = lane - seg * W;
    const unsigned segmask = lane_on ? ((W == 32 ? 0xffffffffu : ((1u << W) - 1u)) << base) : 0u;

    // key rows: [warp][parity][slot][SLOT]; lanes without a segment write the pad word of each row
    uint32_t* rows = reinterpret_cast<uint32_t*>(s_dyn + ((hist_len + 1) & ~1)) + warp * native_warp_words(K, VEC, CH);
    for (int i = lane; i < native_warp_words(K, VEC, CH); i += kWarp) rows[i] = 0u;
    uint32_t* const wr = rows + (lane_on ? seg * WP + l : SLOT - 1);
    const uint32_t* const rd = rows + (lane_on ? seg * WP : 0);
    __syncthreads();

    // ---- per-slot constants, FP32 ----
    int cidx[K];
    bool has[K], lognorm[K];
    float lms[K], span[K], sg2[K], lmu2[K], rpE[K], rpL[K], eE[K], eL[K], bp[K], th[K];
    const double* P = a.P;
    const float* Pf = a.Pf;
    bool any_lognorm = false;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int c = k * W + l;
        cidx[k] = c;
        has[k] = lane_on && c < n;
        const int cc = has[k] ? c : 0;
        lms[k] = Pf[NF_LO_MINUS_SPAN * n + cc];
        span[k] = Pf[NF_SPAN * n + cc];
        sg2[k] = Pf[NF_SG2 * n + cc];
        lmu2[k] = Pf[NF_LMU2 * n + cc];
        rpE[k] = Pf[NF_RP_EARLY * n + cc];
        rpL[k] = Pf[NF_RP_LATE * n + cc];
        eE[k] = Pf[NF_EARLY * n + cc];
        eL[k] = Pf[NF_LATE * n + cc];
        bp[k] = Pf[NF_BP * n + cc];
        th[k] = Pf[NF_THETA * n + cc];
        lognorm[k] = has[k] && P[F_FAMILY * n + cc] != 0.0;
        any_lognorm |= lognorm[k];
    }
    any_lognorm = __any_sync(0xffffffffu, any_lognorm);
    const float L = (float)a.L + a.shift;
    constexpr bool scan = SCAN;
    // front-runner values: key = bits(pos) - key_base in [1, 2^(31-b)) for a racing competitor (the
    // host picks the frame: bbe_sim.cu native_frame), b = a.key_bits index bits
    const int kbits = a.key_bits;
    const uint32_t mulb = a.key_mul, lowmask = mulb - 1u, nmulb = a.key_nmul;  // 2^b, -2^b: one IMAD each
    const uint32_t cl = (uint32_t)l - a.key_base * mulb;       // v = bits * 2^b + cl = (key << b) | l
    const uint32_t cn = a.key_base * mulb - lowmask - 1u;      // ~v' = bits * -2^b + cn, v' = v | lowmask

    // ---- segment bookkeeping ----
    const int64_t segs_total = (int64_t)gridDim.x * kWarpsPerBlock * S;
    // Segment slot -> first sim.  Slots are numbered block-fastest, so the sims of the last, partial
    // round land on one segment in each of many blocks (spread over every SM) instead of filling
    // the first few blocks and leaving most SMs idle at the tail.
    const int64_t slot = BBE_SPREAD_TAIL ? (int64_t)(warp * S + seg) * gridDim.x + blockIdx.x
                                         : ((int64_t)blockIdx.x * kWarpsPerBlock + warp) * S + seg;
    int64_t s = lane_on ? slot : a.n_sims;
    int32_t rt = 0;
    bool running = false;

    float pos[K], prev[K];
    int32_t fin[K];
    bool started[K];  // racing when the sim began (its competitor-timesteps = ticks until it stops)
    static_assert(NT % 4 == 0 && NT >= 4 && NT <= 16, "4, 8, 12 or 16 ticks per block");
    float rawd[K][NT];
    uint32_t blk_sim = 0;
    unsigned long long ct_tot = 0, blk_tot = 0, n_div = 0;
    int64_t first_div = INT64_MAX;

    auto load_sim = [&](bool do_it) {
        if (!do_it) return;
        running = lane_on && s < a.n_sims;
        rt = 0;
        blk_sim = 0;
        const uint64_t gs = (uint64_t)(a.sim_offset + s);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int cc = has[k] ? cidx[k] : 0;
            pos[k] = Pf[NF_POS0 * n + cc];
            prev[k] = Pf[NF_PREV0 * n + cc];
            const bool pre_finished = P[F_FIN0 * n + cc] >= 0.0;
            fin[k] = !(running && has[k]) ? kIdle : (pre_finished ? (int32_t)P[F_FINREL * n + cc] : kRacing);
            started[k] = fin[k] == kRacing;
            if (a.from_start && running && has[k]) {
                // race.py:233-241: one free draw per competitor, resp at position 0 (tick-block 0xFFFFFFFF)
                const U4 w = philox_rk(U4{0xFFFFFFFFu, (uint32_t)cidx[k], (uint32_t)gs, (uint32_t)(gs >> 32)}, a.rk);
                float d, d1;
                if (lognorm[k]) lognormal_pair(w.x, w.y, sg2[k], lmu2[k], d, d1);
                else d = fmaf(span[k], one_plus_u(w.x), lms[k]);
                prev[k] = __fmul_rn((a.shift < bp[k]) ? rpE[k] : rpL[k], d);
            }
        }
    };
    load_sim(true);

    while (true) {
        // ---------------- block boundary ----------------
        // Tick limit (race.py:381-386 / 402-404): the reference refuses the tick after `limit`.  Blocks
        // run whole, so a sim is diverged iff, once rt >= limit, a competitor racing at its start is
        // still racing or finished after tick `limit` -- exactly the sims the reference rejects.
        if (rt >= a.limit) {
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (started[k] && fin[k] > a.limit) fin[k] = kDiverged;
        }
        bool live = false, dv = false;
#pragma unroll
        for (int k = 0; k < K; ++k) { live |= fin[k] == kRacing; dv |= fin[k] == kDiverged; }
        const unsigned live_mask = __ballot_sync(0xffffffffu, live);
        const bool seg_done = running && ((live_mask & segmask) == 0u);
        if (__any_sync(0xffffffffu, seg_done)) {
            const bool diverged = (__ballot_sync(0xffffffffu, dv) & segmask) != 0u;
            // _finish_order (race.py:323-332): rank = #{i : (fin_i, L - pos_i, i) < (fin_c, L - pos_c, c)}.
            // (fin, L - pos) as one order-preserving u64 key (biased fin | float key of L - pos; slots
            // without a competitor sort last); the index tie-break folds into the compare:
            // i < c counts key_i <= key_c, i > c counts key_i < key_c.
            uint64_t key[K];
            int rank[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const uint32_t u = __float_as_uint(__fsub_rn(L, pos[k]));
                const uint32_t lo = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
                key[k] = has[k] ? ((uint64_t)((uint32_t)fin[k] ^ 0x80000000u) << 32) | lo : ~0ull;
                rank[k] = 0;
            }
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
                for (int j = 0; j < W; ++j) {
                    const uint64_t kr = shfl(key[kk], base + j);
                    const int i = kk * W + j;
#pragma unroll
                    for (int k = 0; k < K; ++k) rank[k] += (kr < key[k] + (i < cidx[k] ? 1u : 0u)) ? 1 : 0;
                }
            }
            uint32_t seg_blk = 0;  // per-sim blocked steps: only for the per-sim output
            if (a.blocked)
                for (int j = 0; j < W; ++j) seg_blk += shfl(blk_sim, base + j);
            int64_t lehmer = 0;
            if (a.perms) {
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
                if (diverged) {
                    if (l == 0) { n_div++; first_div = min(first_div, gs); }
                } else {
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        if (!has[k]) continue;
                        if (rank[k] == 0) atomicAdd(&s_hist[TL.wins() + cidx[k]], 1u);
                        atomicAdd(&s_hist[TL.ranks() + cidx[k] * n + rank[k]], 1u);
                        if (a.group_wins && rank[k] == 0)
                            atomicAdd(&a.group_wins[((a.group_base + s) / a.group_size) * n + cidx[k]], 1ull);
                    }
                    BBE_CHECK(!a.perms || (lehmer >= 0 && lehmer < a.perms));
                    if (a.perms && l == 0) atomicAdd(&s_hist[TL.perms() + lehmer], 1u);
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (!has[k]) continue;
                    // competitor-timesteps: a competitor racing at the start stepped every tick until
                    // it finished (fin = ticks) or the sim was cut at the limit (rt ticks)
                    if (started[k]) ct_tot += (fin[k] >= kDiverged) ? (uint32_t)min(rt, a.limit) : (uint32_t)fin[k];
                    const int64_t o = s * n + cidx[k];
                    if (a.winner && rank[k] == 0) a.winner[s] = diverged ? -1 : cidx[k];
                    if (a.order) a.order[s * n + rank[k]] = cidx[k];
                    if (a.finish_ticks) {
                        const double f0 = P[F_FIN0 * n + cidx[k]];
                        a.finish_ticks[o] = f0 >= 0.0 ? (int64_t)f0
                                                      : (fin[k] >= kDiverged ? -1 : a.tick0 + (int64_t)fin[k]);
                    }
                    if (a.final_pos) a.final_pos[o] = (double)pos[k] - (double)a.shift;
                }
                if (l == 0 && a.blocked) a.blocked[s] = seg_blk;
                blk_tot += blk_sim;
            }
            // next sim: claimed from a global counter (dynamic balance -- a segment that drew short
            // races takes more of them), one atomic per warp for all its finishing segments
            const int64_t next = claim_next_sim(seg_done, l == 0, base, segs_total, a.work);
            if (seg_done) s = next;
            load_sim(seg_done);
        }
        if (!__any_sync(0xffffffffu, running)) break;

        // ---------------- Philox: 4 draws per slot per call ----------------
        // counter word 0 = tick / 4, so the stream does not depend on the block length
        auto draw4 = [&](const int h) {
            const uint64_t gs = (uint64_t)(a.sim_offset + s);
            const uint32_t blk = ((uint32_t)rt >> 2) + h;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const U4 w = philox_rk(U4{blk, (uint32_t)cidx[k], (uint32_t)gs, (uint32_t)(gs >> 32)}, a.rk);
                float* const rd4 = &rawd[k][4 * h];
                rd4[0] = fmaf(span[k], one_plus_u(w.x), lms[k]);
                rd4[1] = fmaf(span[k], one_plus_u(w.y), lms[k]);
                rd4[2] = fmaf(span[k], one_plus_u(w.z), lms[k]);
                rd4[3] = fmaf(span[k], one_plus_u(w.w), lms[k]);
                if (any_lognorm) {  // warp-uniform: no divergent second copy of the Philox rounds
                    float l0, l1, l2, l3;
                    lognormal_pair(w.x, w.y, sg2[k], lmu2[k], l0, l1);
                    lognormal_pair(w.z, w.w, sg2[k], lmu2[k], l2, l3);
                    rd4[0] = lognorm[k] ? l0 : rd4[0];
                    rd4[1] = lognorm[k] ? l1 : rd4[1];
                    rd4[2] = lognorm[k] ? l2 : rd4[2];
                    rd4[3] = lognorm[k] ? l3 : rd4[3];
                }
            }
        };

        // ---------------- NT synchronous ticks ----------------
        auto tick = [&](const int tj) {
            bool racing[K];
#pragma unroll
            for (int k = 0; k < K; ++k) racing[k] = fin[k] == kRacing;

            // ---- front runner: nearest key strictly ahead, lowest index on ties (race.py:244-264) ----
            // Published value v = (key << b) | j; lane c keeps min over its segment of
            // v_r + ~(v_c | lowmask) = ((key_r - key_c) << b) + j_r - 2^b  (mod 2^32), one VIADDMNMX
            // per rival.  Rivals strictly ahead give ((dkey - 1) << b) + j < 2^31, ordered by (key, j);
            // equal keys, rivals behind and finished rivals (v = 0) wrap to >= 2^31.  So the minimum
            // holds the front's key AND its index -- no second pass.
            float gap[K];
            bool ahead[K];
            int fj[K], fk[K];
#pragma unroll
            for (int k = 0; k < K; ++k) { gap[k] = CUDART_INF_F; ahead[k] = false; fj[k] = 0; fk[k] = 0; }
            if constexpr (scan) {
                uint32_t kb[K], nk[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    kb[k] = __float_as_uint(pos[k]);
                    nk[k] = kb[k] * nmulb + cn;  // ~((key_c << b) | lowmask)
                    wr[(tj & 1) * PAR + k * SLOT] = racing[k] ? kb[k] * mulb + cl : 0u;
                }
                __syncwarp();
                uint32_t best[K];
#pragma unroll
                for (int kk = 0; kk < K; ++kk) {
                    uint32_t b0[K], b1[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) { b0[k] = 0xffffffffu; b1[k] = 0xffffffffu; }
                    if constexpr (VEC == 4) {
                        const uint4* r4 = reinterpret_cast<const uint4*>(rd + (tj & 1) * PAR + kk * SLOT);
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            const uint4 v = r4[c];
#pragma unroll
                            for (int k = 0; k < K; ++k) {
                                b0[k] = min(b0[k], v.x + nk[k]);
                                b1[k] = min(b1[k], v.y + nk[k]);
                                b0[k] = min(b0[k], v.z + nk[k]);
                                b1[k] = min(b1[k], v.w + nk[k]);
                            }
                        }
                    } else {
                        const uint2* r2 = reinterpret_cast<const uint2*>(rd + (tj & 1) * PAR + kk * SLOT);
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            const uint2 v = r2[c];
#pragma unroll
                            for (int k = 0; k < K; ++k) {
                                b0[k] = min(b0[k], v.x + nk[k]);
                                b1[k] = min(b1[k], v.y + nk[k]);
                            }
                        }
                    }
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const uint32_t d = min(b0[k], b1[k]);
                        // rows in slot order, strictly smaller key distance only: equal keys keep the
                        // lower slot, i.e. the lower competitor index
                        if (kk == 0 || (d >> kbits) < (best[k] >> kbits)) { best[k] = d; fk[k] = kk; }
                    }
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const uint32_t t = best[k] + mulb;  // (dkey << b) | j
                    fj[k] = (int)(t & lowmask);
                    ahead[k] = best[k] < 0x80000000u;
                    gap[k] = __fsub_rn(__uint_as_float(kb[k] + (t >> kbits)), pos[k]);  // used only if ahead
                }
            }

            // ---- step resolution (race.py:267-274) ----
            bool fr[K], bl[K], any_bl = false;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                fr[k] = !ahead[k] || gap[k] > th[k];
                bl[k] = racing[k] && !fr[k];
                any_bl |= bl[k];
            }
            float pf[K];
            if constexpr (K == 1) {
                pf[0] = shfl(prev[0], base + fj[0]);
            } else {
#pragma unroll
                for (int k = 0; k < K; ++k) pf[k] = 0.0f;
                if (__any_sync(0xffffffffu, any_bl)) {
#pragma unroll
                    for (int kk = 0; kk < K; ++kk) {
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            const float v = shfl(prev[kk], base + fj[k]);
                            pf[k] = (fk[k] == kk) ? v : pf[k];
                        }
                    }
                }
            }

            // ---- synchronous update (race.py:299-320) ----
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const bool early = pos[k] < bp[k];
                // Python min(prev_c, prev_front): steps are positive, so fminf returns the same value
                const float m = fminf(prev[k], pf[k]);
                const float step = __fmul_rn(fr[k] ? (early ? rpE[k] : rpL[k]) : (early ? eE[k] : eL[k]),
                                             fr[k] ? rawd[k][tj] : m);
                float p = __fadd_rn(pos[k], step);
                // positions are >= +0.0, so the next float up is the next bit pattern (race.py:310-313)
                p = (p == pos[k]) ? __uint_as_float(__float_as_uint(p) + 1u) : p;
                // branch-free: only racing competitors move
                const bool done = racing[k] && p >= L;
                pos[k] = racing[k] ? p : pos[k];
                // a finished competitor's previous step is never read again (finished rivals never
                // block, race.py:256-257), so it is written unconditionally
                prev[k] = step;
                blk_sim += bl[k] ? 1u : 0u;
                fin[k] = done ? rt + 1 : fin[k];
            }
            rt += 1;
        };
        __syncwarp();  // key rows: the previous block's reads precede this block's writes
#pragma unroll
        for (int h = 0; h < NT / 4; ++h) draw4(h);  // independent Philox chains, issued together
#pragma unroll
        for (int tj = 0; tj < NT; ++tj) tick(tj);
    }

    // ---------------- flush ----------------
    unsigned long long v_ct = ct_tot, v_blk = blk_tot, v_div = n_div;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        v_ct += __shfl_xor_sync(0xffffffffu, v_ct, off);
        v_blk += __shfl_xor_sync(0xffffffffu, v_blk, off);
        v_div += __shfl_xor_sync(0xffffffffu, v_div, off);
        first_div = min(first_div, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)first_div, off));
    }
    const int ct_at = TL.ct();
    if (lane == 0) {
        if (v_ct) atomicAdd((unsigned long long*)&a.tally[ct_at + 0], v_ct);
        if (v_blk) atomicAdd((unsigned long long*)&a.tally[ct_at + 1], v_blk);
        if (v_div) atomicAdd((unsigned long long*)&a.tally[ct_at + 2], v_div);
        if (first_div != INT64_MAX)
            atomicMax((unsigned long long*)&a.tally[ct_at + 4], encode_first(first_div));
    }
    __syncthreads();
    if (threadIdx.x == 0) release_work(a.work);
    for (int i = threadIdx.x; i < hist_len; i += blockDim.x) {
        const uint32_t v = s_hist[i];
        if (v) atomicAdd((unsigned long long*)&a.tally[i], (unsigned long long)v);
    }
}

}  // namespace bbe
