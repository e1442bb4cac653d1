// native64_kernel.cuh -- the throughput kernel at the reference's precision (BBE_MODE_NATIVE64):
// Philox4x32-10 draws, FP64 race state, the reference's FP64 operations in the reference's order.
//
// Semantics (all /root/reference/pkg/src/racemarket/race.py):
//   :46-47   uniform step  lo + (hi - lo) * random()            (random.py uniform, no FMA)
//   :68-69   lognormal     scale * exp(mu + z * sigma)          (random.py lognormvariate/normalvariate)
//   :93-96   responsiveness: early_mult if pos < breakpoint*L else late_mult
//   :233-241 initial_state: prev[c] = (resp(0)*pref)*draw         [from_start]
//   :244-264 _front_runner: nearest STILL-RACING rival STRICTLY ahead, gap = p_i - p_c, equal gaps ->
//            lowest index; finished rivals never block
//   :267-274 _resolve_step: free (no front, or gap > theta): (resp*pref)*draw; else resp*min(prev_c, prev_f)
//   :287-320 advance_race: synchronous; p = pos + step; p == pos -> nextafter(p, +inf); finish at p >= L
//   :323-332 _finish_order: sort by (finish_tick, L - pos, index)
// Every race operation is an explicit IEEE double operation (__dadd_rn/__dmul_rn/__dsub_rn: no FMA
// contraction), so given the same draws the kernel reproduces the reference's positions, finish ticks,
// order and blocked counts bit for bit (tests/test_gpu_native64.py against the C oracle's Philox
// draw source).  Only the word generator differs from the reference: Philox4x32-10 keyed by the
// request seed with counter (tick / 2, competitor, global sim index), instead of a per-sim MT19937.
//
// Draws.  One Philox call per competitor per two ticks gives words (x, y, z, w).  A uniform step takes
// lo + (hi - lo) * u with u = unit53(x, y) = (the top 53 bits of x:y) * 2^-53 for the even tick and
// unit53(z, w) for the odd one -- random()'s 53-bit grid, as the reference's.  A lognormal step
// takes a Box-Muller normal from u1 = 1 - unit53(x, y), u2 = unit53(z, w) (the cosine
// branch for the even tick, the sine branch for the odd one): the reference's Kinderman-Monahan loop
// needs a variable number of words, which a counter-based stream replaces by the same N(0, 1) law.
// Priming draws (run_race) use counter word 0 = 0xFFFFFFFF.
//
// Front runner.  A coarse 26-bit key per racing competitor: mantissa bits 51..26 of y = pos + C, where
// the host picks C (bbe_sim.cu native64_frame) so that every racing position maps into one binade
// [2^E, 2^(E+1)); the key is then a monotone (non-decreasing) function of the position.  Lanes publish
// v = (key << 5) | lane to a shared-memory row and keep one wrapped minimum of v_r + ~v_c per rival
// (one VIADDMNMX): the nearest rival in (key, index) order after c.  When all racing keys of a
// segment are distinct, that rival is exactly the reference's front (keys order like positions).  Two
// racing competitors sharing a key always show up: the lower of the two in (key, index) order finds
// the other as its nearest, with an equal key.  Such a tick -- or a blocked lane whose front could be
// a gap-rounding tie (p_f <= 2 gap, see exact_kernel.cuh) -- reruns the reference's own loop over
// the segment's FP64 positions for the whole warp (rare: the key cell is (L - min pos) / 2^26 wide).
//
// Draw staging.  At every NT-tick block boundary each lane computes its slots' NT step draws (Philox,
// the uniform/lognormal transform) in a rolled loop and parks them in a per-lane shared-memory column;
// the tick loop then reads one double per slot per tick.  The transcendental lognormal code and the
// Philox rounds thus appear once in the binary instead of once per unrolled tick (ncu round 2: with
// them inlined per tick the derby20 kernel spent 76 % of its stall samples on instruction fetch).
//
// Host flags (bbe_sim.cu native64_flags): kN64NoTie -- every racing start position exceeds twice the
// largest theta, so no blocked lane can face a gap-rounding tie and that test is skipped (C2: -0.5 %).
// kN64RespVar -- some competitor's early and late multipliers
// differ, so the responsiveness test `pos < breakpoint*L` (race.py:93-96) runs per tick; without it the
// early value is used (bit-identical, the two are equal).  kN64Guard -- the `p == pos -> nextafter`
// guard (race.py:310-313) can fire: off when every possible step exceeds 2^-52 of the largest
// |position|, where fl(pos + step) == pos is impossible.
//
// Layout, sims, tallies: as native_kernel.cuh (segments of W lanes, K competitors per lane, persistent
// grid with a claimed-sim counter, NT-tick blocks, shared-memory histograms flushed once per block).
#pragma once

#include "common.cuh"

namespace bbe {

template <bool B>
struct CBool {
    static constexpr bool value = B;
};

// BBE_N64_F32_PROBE builds (tools/f32_probe.py, never the product): every draw, step and position
// rounded to FP32 after each FP64 operation -- the FP32-state arithmetic on the very same Philox
// draws, to count the finish orders the state precision alone changes.
#ifndef BBE_N64_F32_PROBE
#define BBE_N64_F32_PROBE 0
#endif
#define BBE_P32(x) (BBE_N64_F32_PROBE ? (double)__double2float_rn(x) : (x))
#ifndef BBE_N64_LN_WORDS
#define BBE_N64_LN_WORDS 1  // lognormal items read their owner's parked Philox words (no second Philox)
#endif
#ifndef BBE_N64_TICK_ROLL
#define BBE_N64_TICK_ROLL 1
#endif
#ifndef BBE_N64_MINBLOCKS_K1
#define BBE_N64_MINBLOCKS_K1 5
#endif
#ifndef BBE_N64_MINBLOCKS_KN
#define BBE_N64_MINBLOCKS_KN 4
#endif
// Tick pairs per iteration of the draw-staging loop: 2 (two Philox chains per slot in flight) for the
// scan-free K <= 2 layouts and the narrow K = 1 scan layouts; 1 elsewhere, where the registers cost
// more than the ILP gains (A/B round 2, ms per launch, 1 -> 2: C3/C5 field 58.04 -> 54.91, C1 1.564 ->
// 1.484, C2 0.682 -> 0.665; derby20 (K = 2 with a scan) 33.22 -> 34.33).
#ifndef BBE_N64_DRAW_UNROLL
#define BBE_N64_DRAW_UNROLL 0  // 0 = the rule above; else forced (A/B builds)
#endif

// Box-Muller: two independent N(0, 1) from four words; u1 in (0, 1], u2 in [0, 1).
__device__ __forceinline__ void normal_pair64(const U4& w, double& n0, double& n1) {
    const double u1 = __dsub_rn(1.0, unit53(w.x, w.y));
    const double u2 = unit53(w.z, w.w);
    const double r = sqrt(__dmul_rn(-2.0, log(u1)));
    double s, c;
    sincospi(__dmul_rn(2.0, u2), &s, &c);
    n0 = __dmul_rn(r, c);
    n1 = __dmul_rn(r, s);
}

// The lognormal step draws of competitor c for ticks 2h and 2h + 1 of global sim gs (counter word 0 =
// h): scale * exp(mu + z * sigma) (random.py lognormvariate / normalvariate) with the Box-Muller pair
// of the same Philox words a uniform competitor would use.  Parameters are read from the parameter
// block (L1-resident), not held in registers.
static __device__ __noinline__ double2 ln_pair_w(const double* P, int n, int c, U4 x) {
    double z0, z1;
    normal_pair64(x, z0, z1);
    const double mu = P[F_MU * n + c], sigma = P[F_SIGMA * n + c], scale = P[F_SCALE * n + c];
    return make_double2(__dmul_rn(scale, exp(__dadd_rn(mu, __dmul_rn(z0, sigma)))),
                        __dmul_rn(scale, exp(__dadd_rn(mu, __dmul_rn(z1, sigma)))));
}

// the same from the counter: Philox words of (h, c, gs) first (the priming draws of run_race)
static __device__ __noinline__ double2 ln_pair(const double* P, int n, int c, uint32_t h, uint64_t gs, uint32_t k0, uint32_t k1) {
    U4 x{h, (uint32_t)c, (uint32_t)gs, (uint32_t)(gs >> 32)};
#pragma unroll
    for (int r = 0; r < 10; ++r) {  // philox_rk with the key schedule computed in place
        const uint32_t hi0 = __umulhi(0xD2511F53u, x.x), lo0 = 0xD2511F53u * x.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, x.z), lo1 = 0xCD9E8D57u * x.z;
        x = U4{hi1 ^ x.y ^ k0, lo1, hi0 ^ x.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return ln_pair_w(P, n, c, x);
}

// K: competitors per lane; CH: key-row chunks of 4 words (SCAN only); SCAN: some theta > 0 (else
// nobody can be blocked and the scan is omitted); LN: some lognormal competitor; NT: ticks per block.
template <int K, int CH, bool SCAN, bool LN, int NT>
__global__ void __launch_bounds__(kBlockThreads, K == 1 ? BBE_N64_MINBLOCKS_K1 : BBE_N64_MINBLOCKS_KN)
native64_kernel(const LaunchArgs a) {
    static_assert(NT % 2 == 0 && NT >= 2 && NT <= 16, "an even number of ticks per block");
    extern __shared__ __align__(16) unsigned long long s_dyn[];
    const TallyLayout TL{a.n, a.perms};
    const int hist_len = TL.hist_len();
    uint32_t* s_hist = reinterpret_cast<uint32_t*>(s_dyn);
    for (int i = threadIdx.x; i < hist_len; i += blockDim.x) s_hist[i] = 0u;
    // the lognormal competitors, in index order (their draws are computed lane-compacted, below)
    __shared__ uint8_t s_lnc[128];  // BBE_MAX_COMPETITORS
    __shared__ int s_nln;
    if (LN && threadIdx.x < kWarp) {
        int m = 0;
        for (int c0 = 0; c0 < a.n; c0 += kWarp) {
            const int c = c0 + (int)threadIdx.x;
            const bool is_ln = c < a.n && a.P[F_FAMILY * a.n + c] != 0.0;
            const unsigned b = __ballot_sync(0xffffffffu, is_ln);
            if (is_ln) s_lnc[m + __popc(b & ((1u << threadIdx.x) - 1u))] = (uint8_t)c;
            m += __popc(b);
        }
        if (threadIdx.x == 0) s_nln = m;
    }

    constexpr int WP = 4 * CH;
    constexpr int SLOT = native_slot_words(4, CH);
    constexpr int PAR = K * SLOT;
    const int n = a.n, W = a.W, S = a.S;
    const int lane = threadIdx.x & (kWarp - 1);
    const int warp = threadIdx.x >> 5;
    const int seg = lane / W;
    const bool lane_on = seg < S;
    const int base = lane_on ? seg * W : 0;
    const int l = lane - seg * W;
    const unsigned segmask = lane_on ? ((W == 32 ? 0xffffffffu : ((1u << W) - 1u)) << base) : 0u;

    // key rows (SCAN only: the scan-free kernels have none -- host smem_bytes with WP = 0)
    constexpr int ROWW = SCAN ? native_warp_words(K, 4, CH) : 0;
    uint32_t* rows = reinterpret_cast<uint32_t*>(s_dyn + ((hist_len + 1) & ~1)) + warp * ROWW;
    if (SCAN)
        for (int i = lane; i < ROWW; i += kWarp) rows[i] = 0u;
    uint32_t* const wr = rows + (lane_on ? seg * WP + l : SLOT - 1);
    const uint32_t* const rd = rows + (lane_on ? seg * WP : 0);
    // this lane's staged draws: [k][tick] doubles, lane-interleaved (conflict-free LDS.64/STS.64)
    double* const s_draw = reinterpret_cast<double*>(s_dyn + ((hist_len + 1) & ~1) + kWarpsPerBlock * ROWW / 2) +
                           warp * (K * NT * kWarp) + lane;
    __syncthreads();

    // ---- per-slot constants, FP64 (the host's double parameter block) ----
    int cidx[K];
    bool has[K], lognorm[K];
    double lo[K], span[K], rpE[K], rpL[K], eE[K], eL[K], bp[K], th[K];
    const double* P = a.P;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int c = k * W + l;
        cidx[k] = c;
        has[k] = lane_on && c < n;
        const int cc = has[k] ? c : 0;
        lo[k] = P[F_LO * n + cc];
        span[k] = P[F_SPAN * n + cc];
        rpE[k] = P[F_RP_EARLY * n + cc];
        rpL[k] = P[F_RP_LATE * n + cc];
        eE[k] = P[F_EARLY * n + cc];
        eL[k] = P[F_LATE * n + cc];
        bp[k] = P[F_BP * n + cc];
        th[k] = P[F_THETA * n + cc];
        lognorm[k] = LN && has[k] && P[F_FAMILY * n + cc] != 0.0;
    }
    const double L = a.L;
    const double C64 = a.key_c64;
    // the gap-rounding tie test (below) is needed only when some racing position can be <= 2 theta
    const bool tie_chk = !(a.n64_flags & kN64NoTie);
    const uint32_t cl = (uint32_t)l - a.key_sub64;  // v = funnel * 32 + cl = (key << 5) | l

    // ---- segment bookkeeping ----
    const int64_t segs_total = (int64_t)gridDim.x * kWarpsPerBlock * S;
    const int64_t slot = (int64_t)(warp * S + seg) * gridDim.x + blockIdx.x;  // block-fastest (spread tail)
    int64_t s = lane_on ? slot : a.n_sims;
    int32_t rt = 0;
    bool running = false;

    double pos[K], prev[K];
    int32_t fin[K];
    bool started[K];
    uint32_t blk_sim = 0;
    unsigned long long ct_tot = 0, blk_tot = 0, n_div = 0;
    int64_t first_div = INT64_MAX;

    // the uniform step draws of slot k for ticks 2h and 2h + 1 of the sim (counter word 0 = h)
    auto draw_pair = [&](int k, uint32_t h, uint64_t gs, double& d0, double& d1) {
        const U4 w = philox_rk(U4{h, (uint32_t)cidx[k], (uint32_t)gs, (uint32_t)(gs >> 32)}, a.rk);
        d0 = BBE_P32(__dadd_rn(lo[k], __dmul_rn(span[k], unit53(w.x, w.y))));
        d1 = BBE_P32(__dadd_rn(lo[k], __dmul_rn(span[k], unit53(w.z, w.w))));
    };

    auto load_sim = [&](bool do_it) {
        if (!do_it) return;
        running = lane_on && s < a.n_sims;
        rt = 0;
        blk_sim = 0;
        const uint64_t gs = (uint64_t)(a.sim_offset + s);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int cc = has[k] ? cidx[k] : 0;
            pos[k] = P[F_POS0 * n + cc];
            prev[k] = P[F_PREV0 * n + cc];
            const bool pre_finished = P[F_FIN0 * n + cc] >= 0.0;
            fin[k] = !(running && has[k]) ? kIdle : (pre_finished ? (int32_t)P[F_FINREL * n + cc] : kRacing);
            started[k] = fin[k] == kRacing;
            if (a.from_start && running && has[k]) {
                // race.py:233-241: one free draw per competitor, resp at position 0
                double d, d1;
                if (LN && lognorm[k]) d = ln_pair(P, n, cidx[k], 0xFFFFFFFFu, gs, a.rk[0], a.rk[1]).x;
                else draw_pair(k, 0xFFFFFFFFu, gs, d, d1);
                prev[k] = BBE_P32(__dmul_rn((0.0 < bp[k]) ? rpE[k] : rpL[k], d));
            }
        }
    };
    load_sim(true);

    while (true) {
        // ---------------- block boundary (as native_kernel.cuh) ----------------
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
            // _finish_order (race.py:323-332): rank = #{i : (fin_i, L - pos_i, i) < (fin_c, L - pos_c, c)}
            double lp[K];
            int rank[K];
#pragma unroll
            for (int k = 0; k < K; ++k) { lp[k] = __dsub_rn(L, pos[k]); rank[k] = 0; }
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
                for (int j = 0; j < W; ++j) {
                    const int32_t fr = shfl(fin[kk], base + j);
                    const double dr = shfl(lp[kk], base + j);
                    const int i = kk * W + j;
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const bool less = (fr < fin[k]) | ((fr == fin[k]) & ((dr < lp[k]) | ((dr == lp[k]) & (i < cidx[k]))));
                        rank[k] += (i < n && less) ? 1 : 0;
                    }
                }
            }
            uint32_t seg_blk = 0;
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
                        BBE_CHECK(cidx[k] < n && rank[k] >= 0 && rank[k] < n);
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
                    if (started[k]) ct_tot += (fin[k] >= kDiverged) ? (uint32_t)min(rt, a.limit) : (uint32_t)fin[k];
                    const int64_t o = s * n + cidx[k];
                    if (a.winner && rank[k] == 0) a.winner[s] = diverged ? -1 : cidx[k];
                    if (a.order) a.order[s * n + rank[k]] = cidx[k];
                    if (a.finish_ticks) {
                        const double f0 = P[F_FIN0 * n + cidx[k]];
                        a.finish_ticks[o] = f0 >= 0.0 ? (int64_t)f0
                                                      : (fin[k] >= kDiverged ? -1 : a.tick0 + (int64_t)fin[k]);
                    }
                    if (a.final_pos) a.final_pos[o] = pos[k];
                }
                if (l == 0 && a.blocked) a.blocked[s] = seg_blk;
                blk_tot += blk_sim;
            }
            const int64_t next = claim_next_sim(seg_done, l == 0, base, segs_total, a.work);
            if (seg_done) s = next;
            load_sim(seg_done);
        }
        if (!__any_sync(0xffffffffu, running)) break;

        // ---- the block's draws: NT per slot, into this lane's shared-memory column ----
        {
            const uint64_t gs = (uint64_t)(a.sim_offset + s);
            constexpr int DU = BBE_N64_DRAW_UNROLL ? BBE_N64_DRAW_UNROLL : (((!SCAN && K <= 2) || (K == 1 && CH <= 3)) ? 2 : 1);
#pragma unroll DU
            for (int h = 0; h < NT / 2; ++h) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    double d0, d1;
                    if constexpr (LN && BBE_N64_LN_WORDS) {
                        // a lognormal slot parks its raw words (x, y | z, w) in its two draw cells;
                        // the lane-compacted pass below turns them into the Box-Muller draws
                        const U4 w = philox_rk(U4{((uint32_t)rt >> 1) + (uint32_t)h, (uint32_t)cidx[k], (uint32_t)gs,
                                                  (uint32_t)(gs >> 32)}, a.rk);
                        const double u0 = __dadd_rn(lo[k], __dmul_rn(span[k], unit53(w.x, w.y)));
                        const double u1 = __dadd_rn(lo[k], __dmul_rn(span[k], unit53(w.z, w.w)));
                        d0 = lognorm[k] ? __hiloint2double((int)w.y, (int)w.x) : u0;
                        d1 = lognorm[k] ? __hiloint2double((int)w.w, (int)w.z) : u1;
                    } else {
                        draw_pair(k, ((uint32_t)rt >> 1) + (uint32_t)h, gs, d0, d1);
                    }
                    BBE_CHECK(in_dyn_smem(s_draw + (k * NT + 2 * h + 1) * kWarp, s_dyn));
                    s_draw[(k * NT + 2 * h) * kWarp] = d0;
                    s_draw[(k * NT + 2 * h + 1) * kWarp] = d1;
                }
            }
            if constexpr (LN) {
                // lognormal draws, lane-compacted: item j = (segment, lognormal competitor, tick pair)
                // runs on lane j % 32 and overwrites the owner lane's two staged draws (the owner's
                // own pass above wrote uniform values there).  C2 (2 lognormal of 10, 3 segments, 8
                // ticks): 24 items, one pass, instead of 4 pairs x (6 of 32 lanes active).
                const int m = s_nln;
                const int per_seg = m * (NT / 2);
                const int items = S * per_seg;
                __syncwarp();
                for (int j0 = 0; j0 < items; j0 += kWarp) {
                    const int j = j0 + lane;
                    const int sg = min(j, items - 1) / per_seg;
                    const int r = min(j, items - 1) - sg * per_seg;
                    const int i = r / (NT / 2), h = r - i * (NT / 2);
                    const int64_t s_item = shfl(s, sg * W);
                    const int32_t rt_item = shfl(rt, sg * W);
                    if (j < items && s_item < a.n_sims) {
                        const int c = s_lnc[i];
                        const int kk = c / W, owner = sg * W + (c - kk * W);
                        double* col = s_draw - lane + owner;
#if BBE_N64_LN_WORDS
                        const double q0 = col[(kk * NT + 2 * h) * kWarp], q1 = col[(kk * NT + 2 * h + 1) * kWarp];
                        const U4 wq{(uint32_t)__double2loint(q0), (uint32_t)__double2hiint(q0),
                                    (uint32_t)__double2loint(q1), (uint32_t)__double2hiint(q1)};
                        const double2 d = ln_pair_w(P, n, c, wq);
#else
                        const double2 d = ln_pair(P, n, c, ((uint32_t)rt_item >> 1) + (uint32_t)h,
                                                  (uint64_t)(a.sim_offset + s_item), a.rk[0], a.rk[1]);
#endif
                        BBE_CHECK(owner >= 0 && owner < kWarp && kk < K && h < NT / 2 &&
                                  in_dyn_smem(col + (kk * NT + 2 * h + 1) * kWarp, s_dyn));
                        col[(kk * NT + 2 * h) * kWarp] = d.x;
                        col[(kk * NT + 2 * h + 1) * kWarp] = d.y;
                    }
                }
                __syncwarp();
            }
        }

        auto tick = [&](const int tj, const int par, auto resp_var, auto guard) {
            bool racing[K];
#pragma unroll
            for (int k = 0; k < K; ++k) racing[k] = fin[k] == kRacing;

            // ---- front runner (race.py:244-264) ----
            double gap[K], pfpos[K];
            bool ahead[K];
            int fj[K], fk[K];
#pragma unroll
            for (int k = 0; k < K; ++k) { gap[k] = CUDART_INF; pfpos[k] = CUDART_INF; ahead[k] = false; fj[k] = 0; fk[k] = 0; }
            if constexpr (SCAN) {
                uint32_t v[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const double y = __dadd_rn(pos[k], C64);
                    const uint32_t key = __funnelshift_r((uint32_t)__double2loint(y), (uint32_t)__double2hiint(y), 26);
                    v[k] = key * 32u + cl;
                    BBE_CHECK(in_dyn_smem(wr + par * PAR + k * SLOT, s_dyn));
                    wr[par * PAR + k * SLOT] = racing[k] ? v[k] : 0u;
                }
                __syncwarp();
                // per (own slot k, row kk) offset: t = v_r + nk is < 2^31 iff rival r follows c in
                // (key, index) order -- rows below c's slot need a strictly larger key, c's own row a
                // larger (key, lane), rows above a key at least as large
                bool coll = false;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    uint32_t bestv = 0xffffffffu;
                    int bestkk = 0;
                    bool any = false;
#pragma unroll
                    for (int kk = 0; kk < K; ++kk) {
                        const uint32_t nk = kk < k ? ~(v[k] | 31u) : (kk == k ? ~v[k] : 0u - (v[k] & ~31u));
                        uint32_t b0 = 0xffffffffu, b1 = 0xffffffffu;
                        const uint4* r4 = reinterpret_cast<const uint4*>(rd + par * PAR + kk * SLOT);
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            const uint4 q = r4[c];
                            b0 = min(b0, q.x + nk);
                            b1 = min(b1, q.y + nk);
                            b0 = min(b0, q.z + nk);
                            b1 = min(b1, q.w + nk);
                        }
                        const uint32_t t = min(b0, b1);
                        const uint32_t vf = t - nk;  // the rival's own published value
                        // rows in slot order; a later row replaces only with a strictly smaller key
                        if (t < 0x80000000u && (!any || (vf >> 5) < (bestv >> 5))) { bestv = vf; bestkk = kk; any = true; }
                    }
                    ahead[k] = any;
                    fk[k] = bestkk;
                    fj[k] = (int)(bestv & 31u);
                    coll |= racing[k] && any && (bestv >> 5) == (v[k] >> 5);
                }
                // the front's FP64 position
#pragma unroll
                for (int kk = 0; kk < K; ++kk) {
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const double pr = shfl(pos[kk], base + fj[k]);
                        pfpos[k] = (K == 1 || fk[k] == kk) ? pr : pfpos[k];
                    }
                }
                bool need_exact = coll;
#pragma unroll
                for (int k = 0; k < K; ++k) gap[k] = ahead[k] ? __dsub_rn(pfpos[k], pos[k]) : CUDART_INF;
                if (tie_chk) {
#pragma unroll
                    for (int k = 0; k < K; ++k)  // a blocked lane whose front could be a gap-rounding tie
                        need_exact |= racing[k] && ahead[k] && !(gap[k] > th[k]) && !(pfpos[k] > __dmul_rn(2.0, gap[k]));
                }
                if (__any_sync(0xffffffffu, need_exact)) {
                    // the reference's loop (race.py:244-264) over the segment's start-of-tick positions
                    double bg[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) { bg[k] = CUDART_INF; ahead[k] = false; }
#pragma unroll
                    for (int kk = 0; kk < K; ++kk) {
                        for (int j = 0; j < W; ++j) {
                            const double pr = shfl(pos[kk], base + j);
                            const bool rr = shfl((int)racing[kk], base + j) != 0;
#pragma unroll
                            for (int k = 0; k < K; ++k) {
                                if (rr && pr > pos[k]) {
                                    const double g = __dsub_rn(pr, pos[k]);
                                    if (!ahead[k] || g < bg[k]) { bg[k] = g; ahead[k] = true; fk[k] = kk; fj[k] = j; }
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int k = 0; k < K; ++k) gap[k] = bg[k];
                }
            }

            // ---- step resolution (race.py:267-274) ----
            bool fr[K], bl[K], any_bl = false;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                fr[k] = !SCAN || !ahead[k] || gap[k] > th[k];
                bl[k] = racing[k] && !fr[k];
                any_bl |= bl[k];
            }
            double pf[K];
#pragma unroll
            for (int k = 0; k < K; ++k) pf[k] = 0.0;
            if constexpr (SCAN) {
                if (__any_sync(0xffffffffu, any_bl)) {
#pragma unroll
                    for (int kk = 0; kk < K; ++kk) {
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            const double pv = shfl(prev[kk], base + fj[k]);
                            pf[k] = (K == 1 || fk[k] == kk) ? pv : pf[k];
                        }
                    }
                }
            }

            // ---- synchronous update (race.py:299-320) ----
            bool eq_any = false;
            double pnew[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const bool early = decltype(resp_var)::value ? pos[k] < bp[k] : true;
                double step;
                const double dk = s_draw[(k * NT + tj) * kWarp];
                if (!SCAN || fr[k]) {
                    step = BBE_P32(__dmul_rn(early ? rpE[k] : rpL[k], dk));
                } else {
                    const double m = (pf[k] < prev[k]) ? pf[k] : prev[k];  // Python min(prev_c, prev_front)
                    step = BBE_P32(__dmul_rn(early ? eE[k] : eL[k], m));
                }
                pnew[k] = BBE_P32(__dadd_rn(pos[k], step));
                if constexpr (decltype(guard)::value) eq_any |= racing[k] && pnew[k] == pos[k];
                prev[k] = step;  // a finished competitor's previous step is never read again
            }
            if constexpr (decltype(guard)::value) {
                if (__any_sync(0xffffffffu, eq_any)) {
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        if (pnew[k] == pos[k]) pnew[k] = nextafter(pnew[k], CUDART_INF);
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const bool done = racing[k] && pnew[k] >= L;
                pos[k] = racing[k] ? pnew[k] : pos[k];
                blk_sim += bl[k] ? 1u : 0u;
                fin[k] = done ? rt + 1 : fin[k];
            }
            rt += 1;
        };

        // the block's NT ticks, in pairs (the key rows alternate by tick parity), under the host flags
        auto run_block = [&](auto resp_var, auto guard) {
            if constexpr (SCAN && K >= 2 && BBE_N64_TICK_ROLL) {
                // one tick body (the row parity a runtime value): the multi-slot scan layouts' tick is
                // large, and two unrolled copies overflow the instruction cache (derby20, K = 2: 27 %
                // no_instructions stalls; 33.4 -> 29.3 ms).  K = 1 keeps both: rolled it is 1.5-2 %
                // slower (C2, derby12/16/24/32).
#pragma unroll 1
                for (int t = 0; t < NT; ++t) tick(t, t & 1, resp_var, guard);
            } else {
#pragma unroll 1
                for (int tp = 0; tp < NT; tp += 2) {
                    tick(tp, 0, resp_var, guard);
                    tick(tp + 1, 1, resp_var, guard);
                }
            }
        };
        if (SCAN) __syncwarp();  // key rows: the previous block's reads precede this block's writes
        const int fl = a.n64_flags & (kN64RespVar | kN64Guard);
        if (fl == (kN64RespVar | kN64Guard)) run_block(CBool<true>{}, CBool<true>{});
        else if (fl == kN64RespVar) run_block(CBool<true>{}, CBool<false>{});
        else if (fl == kN64Guard) run_block(CBool<false>{}, CBool<true>{});
        else run_block(CBool<false>{}, CBool<false>{});
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
