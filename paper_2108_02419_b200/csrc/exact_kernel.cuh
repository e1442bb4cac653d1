// exact_kernel.cuh -- the bit-exact FP64 race kernel: BBE_MODE_INJECT and BBE_MODE_MT.
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
// Every operation is the reference's own IEEE double operation in the reference's order (explicit
// __dadd_rn/__dmul_rn/__dsub_rn/__ddiv_rn: no FMA contraction), so given the same draws the kernel
// reproduces positions, finish ticks, order and blocked counts bit for bit.
//
// Mapping: one sim per SEGMENT of W consecutive lanes, competitor c = k*W + l in lane l, slot k;
// S = 32/W sims per warp; persistent grid, a finished segment claims its next sim at a 4-tick block
// boundary.  Front runner: rounding is monotonic, so the reference's smallest gap
// min_i fl(p_i - p_c) equals fl(min_i p_i - p_c); each lane takes a positional min over its
// segment's start-of-tick positions (a shared-memory row per tick parity, 128-bit loads) and keeps
// the lowest index holding it.  That is the reference's front unless two distinct positions round
// to the same gap, which needs p* <= 2 gap; blocked lanes in that case rerun the reference's own gap
// arithmetic and lowest-index rule.
//
// Draw sources:
//   INJECT  recorded reference draws (CSR per sim); a free slot's offset in the tick = popc of free
//           slots of lower competitor index in its segment -- the reference's consumption order.
//   MT      per-sim CPython MT19937 (mt_stream.cuh) in shared memory.  Speculative rounds: every
//           pending competitor reads its words at the offset it would have if each pending lognormal
//           draw accepted its next Kinderman-Monahan trial (offsets from two ballots per slot);
//           draws before the first rejection are final.  Uniform-only fields (LN = false) need no
//           rounds: every draw is two words.  The whole warp twists a segment's block when its unread window runs low (the
//           unread words move to a side buffer just below the block first, so the window stays
//           contiguous and early twists leave the stream unchanged).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "mt_stream.cuh"

namespace bbe {

#ifndef BBE_MT_MINBLOCKS
#define BBE_MT_MINBLOCKS 5  // measured (C2, 100k sims, early round 1): 1 -> 3.82 ms, 5 -> 3.67 ms, 6 -> 4.41 ms
#endif

// LN = false (MT): the field has no lognormal competitor, so every draw takes exactly two words and a
// tick's offsets follow from one ballot per slot -- no speculative rounds.
// MT, K > 1 (fields of 33..128 competitors): 4 blocks/SM for K = 2 (126 registers, no spills; the C5
// field forced to K = 2: 90.8 -> 72.9 ms per 10^6 races, derby20: 116.8 -> 86.3 ms), 2 for K >= 3
// (4 is slower there: more spills)
#ifndef BBE_MT_LIMIT_PRED
#define BBE_MT_LIMIT_PRED 1  // the per-tick limit test without a branch (C2 MT 2.160 -> 2.131 ms)
#endif
#ifndef BBE_MT_LT_TABLE
#define BBE_MT_LT_TABLE 1  // log2 T from a per-launch 2-bit table (C2 MT 2.160 -> 2.125 ms; both: 2.090)
#endif
#ifndef BBE_MT_TWIST_SHFL
#define BBE_MT_TWIST_SHFL 1  // MT19937 twist with one warp sync per 32-word chunk (shuffled neighbours)
#endif
#ifndef BBE_MT_MINBLOCKS_K2
#define BBE_MT_MINBLOCKS_K2 4
#endif
// MT, K = 1 with at most 2 segments per warp (W >= 11): the block's MT states take little shared
// memory, so residency is set by registers -- LEAN kernels are built for more blocks per SM (A/B, C5
// field W = 20, 10^6 races: 5 -> 7 blocks/SM 33.3 -> 29.2 ms; with 4 segments per warp (W = 8, C1) the
// shared memory caps residency at 4 blocks and fewer registers only cost: 11.9 -> 12.4 ms)
#ifndef BBE_MT_MINBLOCKS_LEAN
#define BBE_MT_MINBLOCKS_LEAN 7
#endif
#ifndef BBE_MT_MINBLOCKS_LEAN_LN
#define BBE_MT_MINBLOCKS_LEAN_LN 5  // with lognormal competitors 6 or 7 spill and lose (derby20 24.9 -> 25.8 / 25.1 ms)
#endif
template <int K, int MODE, bool LN = true, bool LEAN = false>
__global__ void __launch_bounds__(kBlockThreads,
                                  MODE == MT ? (K == 1 ? (LEAN ? (LN ? BBE_MT_MINBLOCKS_LEAN_LN : BBE_MT_MINBLOCKS_LEAN)
                                                               : BBE_MT_MINBLOCKS)
                                                       : (K == 2 ? BBE_MT_MINBLOCKS_K2 : 2))
                                             : 1)
exact_kernel(const LaunchArgs a) {
    static_assert(MODE == INJECT || MODE == MT, "exact kernel modes");
    constexpr int kSeg = mt_seg_words(K);  // MT: words per segment (block + side buffer)
    extern __shared__ __align__(16) unsigned long long s_dyn[];
    const TallyLayout TL{a.n, a.perms};
    const int hist_len = TL.hist_len();
    const int n = a.n, W = a.W, S = a.S;
    const int lane = threadIdx.x & (kWarp - 1);
    const int warp = threadIdx.x >> 5;
    const int seg = lane / W;
    const bool lane_on = seg < S;
    const int base = lane_on ? seg * W : 0;
    const int l = lane - seg * W;
    const unsigned segmask = lane_on ? ((W == 32 ? 0xffffffffu : ((1u << W) - 1u)) << base) : 0u;
    const unsigned lt_mask = (1u << lane) - 1u;
    // MT: this segment's words: [side buffer: kSide][current block: 624]; the unread stream is the
    // contiguous window seg_mt[wp, kSeg)
    constexpr int kSide = mt_side_words(K);
    // dynamic shared memory: [MT segment words][position rows][lognormal offsets (MT)][histograms] --
    // the histograms last, so the per-word pointers do not depend on the field size
    uint32_t* const smem_w = reinterpret_cast<uint32_t*>(s_dyn);
    uint32_t* const seg_mt = smem_w + (warp * S + (lane_on ? seg : 0)) * kSeg;
    uint32_t* const mt = seg_mt + kSide;  // the 624-word MT19937 block
    // start-of-tick front-runner keys, per warp: [parity][slot] rows of kKRow words, segment at
    // seg * WPK (4-word chunks, padding words 0), idle lanes write the row's last word
    // segments of 8 <= W <= 12 lanes (at most 4 per warp) get 12-word rows (3 chunks, zero padding past
    // W), so their scan is a fixed 3-chunk loop; other widths use ceil(W / 4) chunks (INJECT runs W < 8,
    // up to 32 segments per warp, whose 12-word rows would overrun the key row)
    const bool kNarrow = W >= 8 && W <= 12;
    const int CHK = kNarrow ? 3 : (W + 3) >> 2, WPK = 4 * CHK;
    double* const xrows_all = reinterpret_cast<double*>(smem_w + (MODE == MT ? kWarpsPerBlock * S * kSeg : 0));
    uint32_t* const krows = reinterpret_cast<uint32_t*>(xrows_all + warp * 2 * K * kXSlot);
    constexpr int kKRow = 2 * kXSlot;  // words per key row (the double row's footprint; S * WPK <= 36)
    // MT, K = 1: the round's pending lognormal draws publish their speculative word offsets here, by
    // rank in their segment (lane base + rank), for the lanes that evaluate their trials
    int* const ln_off_all = reinterpret_cast<int*>(xrows_all + kWarpsPerBlock * 2 * K * kXSlot);
    int* const ln_off = ln_off_all + warp * kWarp;
    // 32-bit shared histograms (native ATOMS.ADD; a 64-bit shared add is a CAS loop).  A block's count
    // in one bin is at most the sims of its launch, which the host keeps below 2^32 (launch_one).
    uint32_t* const s_hist = reinterpret_cast<uint32_t*>(ln_off_all + (MODE == MT ? kWarpsPerBlock * kWarp : 0));
    for (int i = threadIdx.x; i < hist_len; i += blockDim.x) s_hist[i] = 0u;
    for (int i = lane; i < 2 * K * kKRow; i += kWarp) krows[i] = 0u;
    uint32_t* const kw = krows + (lane_on ? seg * WPK + l : kKRow - 1);
    const uint32_t* const kr = krows + (lane_on ? seg * WPK : 0);
    const double C64 = a.key_c64;
    const uint32_t cl = (uint32_t)l - a.key_sub64;  // v = funnel * 32 + cl = (key << 5) | l
#if BBE_MT_LT_TABLE
    // the K = 1 trial pass's log2 T for m pending lognormal draws (m < 32), two bits per m
    uint64_t lt_tab = 0;
    for (int mm = 1; mm < 32; ++mm) {
        const int v = (8 * mm <= W) ? 3 : (4 * mm <= W) ? 2 : (2 * mm <= W) ? 1 : 0;
        lt_tab |= (uint64_t)v << (2 * mm);
    }
#endif
    __syncthreads();

    // ---- per-slot constants (the lane->competitor map is fixed for the kernel) ----
    int cidx[K];
    bool has[K], lognorm[K];
    double lo[K], span[K], mu[K], sigma[K], scale[K], rpE[K], rpL[K], eE[K], eL[K], bp[K], th[K];
    double pos0[K], prev0[K];
    int64_t fin0[K];
    const double* P = a.P;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int c = k * W + l;
        cidx[k] = c;
        has[k] = lane_on && c < n;
        const int cc = has[k] ? c : 0;
        lo[k] = P[F_LO * n + cc];
        span[k] = P[F_SPAN * n + cc];
        mu[k] = P[F_MU * n + cc];
        sigma[k] = P[F_SIGMA * n + cc];
        scale[k] = P[F_SCALE * n + cc];
        rpE[k] = P[F_RP_EARLY * n + cc];
        rpL[k] = P[F_RP_LATE * n + cc];
        eE[k] = P[F_EARLY * n + cc];
        eL[k] = P[F_LATE * n + cc];
        bp[k] = P[F_BP * n + cc];
        th[k] = P[F_THETA * n + cc];
        pos0[k] = P[F_POS0 * n + cc];
        prev0[k] = P[F_PREV0 * n + cc];
        fin0[k] = has[k] ? (int64_t)P[F_FIN0 * n + cc] : INT64_MAX;
        lognorm[k] = has[k] && P[F_FAMILY * n + cc] != 0.0;
    }
    const double L = a.L;
    const double NEG_INF = -CUDART_INF;

    // ---- segment bookkeeping (replicated in every lane of the segment) ----
    const int64_t segs_total = (int64_t)gridDim.x * kWarpsPerBlock * S;
    int64_t s = lane_on ? ((int64_t)blockIdx.x * kWarpsPerBlock + warp) * S + seg : a.n_sims;
    const int64_t start = a.tick0;
    int32_t rt = 0;
    int64_t cursor = 0, cursor_end = 0;  // INJECT
    int wp = kSeg;                       // MT: start of the unread window seg_mt[wp, kSeg)
    bool running = false, diverged = false, bad = false;

    double pos[K], prev[K];
    int64_t fin[K];
    bool racing[K];
    uint32_t ct_sim = 0, blk_sim = 0;
    unsigned long long ct_tot = 0, blk_tot = 0, n_div = 0, n_bad = 0;
    int64_t first_div = INT64_MAX, first_bad = INT64_MAX;

    // ---- MT19937 stream helpers (warp-uniform calls) ----
    // Regenerate a segment's block in place (MT19937 twist): all 32 lanes of the warp twist one
    // needing segment at a time, 20 chunks of 32 words (32 < 227 keeps every "new" dependency in an
    // earlier chunk), so a segment's twist costs the same whether or not its warp-mates need one.
    uint32_t* const warp_mt = smem_w + warp * S * kSeg;
    auto mt_twist = [&](bool need) {
        unsigned todo = __ballot_sync(0xffffffffu, need && l == 0);  // one bit per needing segment
        __syncwarp();
        while (todo) {
            const int leader = __ffs(todo) - 1;
            todo &= todo - 1u;
            uint32_t* const t = warp_mt + (leader / W) * kSeg + kSide;
#if BBE_MT_TWIST_SHFL
            // one sync per chunk: y = the next word comes from lane + 1's x by shuffle (read before any
            // write of the chunk), lane 31 reads the next chunk's first word (old until the next chunk
            // writes it, after this chunk's sync); the last word wraps to the already-new t[0]
#pragma unroll
            for (int c0 = 0; c0 < kMtWords; c0 += kWarp) {
                const int i = c0 + lane;
                const bool act = i < kMtWords;
                const uint32_t x = act ? t[i] : 0u;
                const uint32_t nx = t[c0 + kWarp < kMtWords ? c0 + kWarp : 0];
                uint32_t y = __shfl_down_sync(0xffffffffu, x, 1);
                if (i + 1 == c0 + kWarp || i + 1 == kMtWords) y = nx;
                const uint32_t m = act ? t[i < kMtWords - kMtM ? i + kMtM : i + kMtM - kMtWords] : 0u;
                if (act) t[i] = mt_mix(x, y, m);
                __syncwarp();
            }
#else
            for (int c0 = 0; c0 < kMtWords; c0 += kWarp) {
                const int i = c0 + lane;
                const bool act = i < kMtWords;
                uint32_t x = 0, y = 0, m = 0;
                if (act) {
                    x = t[i];
                    y = t[i + 1 < kMtWords ? i + 1 : 0];
                    m = t[i < kMtWords - kMtM ? i + kMtM : i + kMtM - kMtWords];
                }
                __syncwarp();
                if (act) t[i] = mt_mix(x, y, m);
                __syncwarp();
            }
#endif
        }
    };
    // The segment's unread stream is the window seg_mt[wp, kSeg): words saved from earlier blocks
    // followed by the rest of the current block.  Before a round that may read up to 4WK words, a
    // shorter window is topped up: its words move to the end of the side buffer, just below the
    // block, and the block is twisted in place -- early, but the stream is the same, since the
    // twist reads the whole old block.
    // A round reads below offset fill_need: 4WK (every lane's 4 words), plus, for the K = 1 trial
    // pass, kMtMaxTrials - 1 further trials of one lognormal draw.
    const int fill_need = (K == 1 && LN) ? 4 * W + 4 * kMtMaxTrials : 4 * W * K;
    auto mt_window_fill = [&]() {
        const bool low = running && lane_on && kSeg - wp < fill_need;
        if (!__any_sync(0xffffffffu, low)) return;
        // keep < fill_need <= kSide words move down by exactly one block (624 > keep: the ranges are
        // disjoint), ending just below the block
        const int keep = kSeg - wp;
        if (low)
            for (int i = l; i < keep; i += W) seg_mt[kSide - keep + i] = seg_mt[wp + i];
        mt_twist(low);  // starts and ends with __syncwarp
        if (low) wp = kSide - keep;
    };
    // window offset k -> raw word.  No clamp: after mt_window_fill the window holds >= fill_need words
    // and a round reads below offset fill_need + 4, so an idle lane's read lands at most 3 words past
    // the segment, inside the block's dynamic shared memory (the next segment or the position rows).
    auto mt_word = [&](int k) -> uint32_t {
        BBE_CHECK(in_dyn_smem(seg_mt + wp + k, s_dyn));
        return seg_mt[wp + k];
    };
    auto mt_consume = [&](int c) { wp += c; };
    // One step draw per (slot, lane) with want[k], in competitor-index order within each segment
    // (slot-major, then lane): uniform(lo, hi) = lo + (hi - lo) * random(); scale *
    // lognormvariate(mu, sigma) via the Kinderman-Monahan loop of random.normalvariate
    // (Lib/random.py).  Warp-uniform call.
    auto mt_draws = [&](const bool (&want)[K], double (&d)[K]) {
        if constexpr (!LN) {
            // uniform(lo, hi) only: 2 words per draw in competitor-index order (slot-major, then lane)
            mt_window_fill();
            int slot_base = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const unsigned m = __ballot_sync(0xffffffffu, want[k]) & segmask;
                const int off = slot_base + 2 * __popc(m & lt_mask);
                slot_base += 2 * __popc(m);
                const uint32_t w0 = mt_temper(mt_word(off)), w1 = mt_temper(mt_word(off + 1));
                d[k] = want[k] ? __dadd_rn(lo[k], __dmul_rn(span[k], random53(w0, w1))) : 1.0;
            }
            if (lane_on && running) mt_consume(slot_base);
            return;
        }
        if constexpr (K == 1) {
            // ---- K = 1: one trial-evaluation pass per round ----
            // Offsets are speculative as below (each pending lognormal draw takes 4 words); then the
            // pending lognormal draw of rank i in its segment evaluates its trials j = 0..T-1 (words
            // off_i + 4j) on lanes i*T + j, T = the largest power of two <= kMtMaxTrials with m*T <= W
            // for m such draws.  In index
            // order, draw i starts `shift` trials into its grid (the extra trials of the draws before
            // it) and accepts at the first accepting trial from there; the lanes after it move by its
            // extra trials.  A draw with no accepting trial left in its grid ends the round: it and
            // every later draw stay pending, its grid's words are consumed.
            bool pend = want[0], got_ln = false;
            double u1a = 0.0, u2a = 1.0;
            d[0] = 1.0;
            while (__any_sync(0xffffffffu, pend)) {
                mt_window_fill();
                const unsigned pm = __ballot_sync(0xffffffffu, pend) & segmask;
                const unsigned lm = __ballot_sync(0xffffffffu, pend && lognorm[0]) & segmask;
                const int off = 2 * (__popc(pm & lt_mask) + __popc(lm & lt_mask));
                const int used_all = 2 * (__popc(pm) + __popc(lm));
                const int m = __popc(lm);
                // T: the largest power of two <= kMtMaxTrials with m*T <= W (shifts, no division)
#if BBE_MT_LT_TABLE
                const int lt = (int)((lt_tab >> (2 * m)) & 3ull);  // lt_tab: the expression below per m
#else
                const int lt = (8 * m <= W) ? 3 : (4 * m <= W) ? 2 : (2 * m <= W) ? 1 : 0;
#endif
                const int T = 1 << lt;
                const int ti = l >> lt, tj = l & (T - 1);
                if (pend && lognorm[0]) ln_off[base + __popc(lm & lt_mask)] = off;
                __syncwarp();
                bool acc = false;
                if (lane_on && running && ti < m) {
                    const int at = ln_off[base + ti] + 4 * tj;
                    acc = km_accept(mt_temper(mt_word(at)), mt_word(at + 1), mt_temper(mt_word(at + 2)),
                                    mt_temper(mt_word(at + 3)), a.nv_magic);
                }
                const unsigned am = __ballot_sync(0xffffffffu, acc) & segmask;
                int shift = 0, my_shift = 0, my_grid = 0, fail_lane = kWarp, fail_used = 0;
                unsigned rem = lm;
                for (int i = 0; i < m; ++i) {
                    const int li = __ffs(rem) - 1;
                    rem &= rem - 1u;
                    const unsigned avail = ((am >> (base + i * T)) & ((1u << T) - 1u)) >> shift;
                    if (!avail) {
                        fail_lane = li;
                        fail_used = ln_off[base + i] + 4 * T;
                        break;
                    }
                    const int t = __ffs(avail) - 1;  // extra trials of draw i
                    if (lane == li) my_grid = shift + t;
                    shift += t;
                    if (lane > li) my_shift = shift;
                }
                __syncwarp();  // ln_off reads precede the next round's writes
                if (pend && lane < fail_lane) {
                    const int at = off + 4 * (lognorm[0] ? my_grid : my_shift);
                    const double r = random53(mt_temper(mt_word(at)), mt_temper(mt_word(at + 1)));
                    if (lognorm[0]) {
                        got_ln = true;
                        u1a = r;
                        u2a = __dsub_rn(1.0, random53(mt_temper(mt_word(at + 2)), mt_temper(mt_word(at + 3))));
                    } else {
                        d[0] = __dadd_rn(lo[0], __dmul_rn(span[0], r));
                    }
                    pend = false;
                }
                if (lane_on && running) mt_consume(fail_lane < kWarp ? fail_used : used_all + 4 * shift);
            }
            if (got_ln) {
                const double z = __ddiv_rn(__dmul_rn(a.nv_magic, __dsub_rn(u1a, 0.5)), u2a);
                d[0] = __dmul_rn(scale[0], libm_exp(__dadd_rn(mu[0], __dmul_rn(z, sigma[0]))));
            }
            return;
        }
        double ln_u1[K], ln_u2[K];  // the accepted Kinderman-Monahan pair of a lognormal competitor
        bool ln_draw[K], pend[K];
        bool any_pend = false;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            d[k] = 1.0;
            ln_u1[k] = 0.0;
            ln_u2[k] = 1.0;
            ln_draw[k] = false;
            pend[k] = want[k];
            any_pend |= want[k];
        }
        // Speculative rounds: every pending competitor takes its words at the offset it would have if
        // each pending lognormal draw accepted its next Kinderman-Monahan trial (2 words per uniform
        // draw, 4 per trial).  Draws up to the first rejected trial in index order are then final;
        // the rejected one consumed its 4 words and retries first in the next round.
        while (__any_sync(0xffffffffu, any_pend)) {
            mt_window_fill();
            // offsets: a pending competitor takes 2 words, +2 more if lognormal -- two ballots per
            // slot give every lane its segment-local prefix
            int off[K];
            int slot_base = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const unsigned pm = __ballot_sync(0xffffffffu, pend[k]) & segmask;
                const unsigned lm = __ballot_sync(0xffffffffu, pend[k] && lognorm[k]) & segmask;
                off[k] = slot_base + 2 * (__popc(pm & lt_mask) + __popc(lm & lt_mask));
                slot_base += 2 * (__popc(pm) + __popc(lm));
            }
            const int used_all = slot_base;  // the whole round's words
            double r01[K];  // random() from the first two words: a uniform draw, or a trial's u1
            bool ok[K];
            uint32_t w23[K][2];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                r01[k] = random53(mt_temper(mt_word(off[k])), mt_temper(mt_word(off[k] + 1)));
                w23[k][0] = mt_temper(mt_word(off[k] + 2));
                w23[k][1] = mt_temper(mt_word(off[k] + 3));
                ok[k] = true;
                if (pend[k] && lognorm[k]) {
                    const double u1 = r01[k];
                    const double u2 = __dsub_rn(1.0, random53(w23[k][0], w23[k][1]));
                    // accept iff z*z/4 <= -log(u2) (Lib/random.py normalvariate).  Decide in FP32 when
                    // the two sides are far apart (relative 1e-4, absolute 1e-5: >25x the FP32 error of
                    // either side), else in FP64 exactly as CPython does -- the same decision either way.
                    const float z32 = __fdividef((float)a.nv_magic * ((float)u1 - 0.5f), (float)u2);
                    const float zz32 = 0.25f * z32 * z32;
                    const float l32 = -__logf((float)u2);
                    const float gap32 = zz32 - l32;
                    bool acc;
                    if (fabsf(gap32) > 1e-4f * fmaxf(fabsf(zz32), fabsf(l32)) + 1e-5f) {
                        acc = gap32 < 0.0f;
                    } else {
                        const double zx = __ddiv_rn(__dmul_rn(a.nv_magic, __dsub_rn(u1, 0.5)), u2);
                        acc = __dmul_rn(__dmul_rn(zx, zx), 0.25) <= -log(u2);  // z*z/4.0 (exact scaling)
                    }
                    ok[k] = acc;
                    ln_u1[k] = u1;
                    ln_u2[k] = u2;
                }
            }
            // first rejected trial in index order: lowest slot with a rejection, lowest lane in it
            int kb = K;
            unsigned first_bad = 0u;
#pragma unroll
            for (int k = K - 1; k >= 0; --k) {
                const unsigned bad_k = __ballot_sync(0xffffffffu, pend[k] && !ok[k]) & segmask;
                if (bad_k) { kb = k; first_bad = bad_k & (0u - bad_k); }
            }
            int off_kb = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) off_kb = (k == kb) ? off[k] : off_kb;
            const int used_bad = __shfl_sync(0xffffffffu, off_kb, first_bad ? __ffs(first_bad) - 1 : lane) + 4;
            any_pend = false;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const bool done = pend[k] & ((k < kb) | ((k == kb) & ((1u << lane) < first_bad)));
                if (done) {
                    if (lognorm[k]) ln_draw[k] = true;
                    else d[k] = __dadd_rn(lo[k], __dmul_rn(span[k], r01[k]));
                    pend[k] = false;
                }
                any_pend |= pend[k];
            }
            if (lane_on && running) mt_consume(first_bad ? used_bad : used_all);
        }
        // lognormvariate's value for every accepted pair at once (the stream order is already fixed):
        // z = NV*(u1-0.5)/u2, scale * exp(mu + z*sigma) with the host libm's exp
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (ln_draw[k]) {
                const double z = __ddiv_rn(__dmul_rn(a.nv_magic, __dsub_rn(ln_u1[k], 0.5)), ln_u2[k]);
                d[k] = __dmul_rn(scale[k], libm_exp(__dadd_rn(mu[k], __dmul_rn(z, sigma[k]))));
            }
        }
    };

    // trajectory snapshot after tick t of the current sim (t = 0: the state the sim starts from)
    auto record = [&](int32_t t) {
        const int64_t row = (s * ((int64_t)a.traj_cap + 1) + t) * n;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (!has[k]) continue;
            a.traj_pos[row + cidx[k]] = pos[k];
            a.traj_prev[row + cidx[k]] = prev[k];
        }
    };

    // refill the segment with its next sim; warp-uniform (every lane calls it)
    auto load_sim = [&](bool do_it) {
        if (do_it) {
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
            if (MODE == MT && running) {
                // 624 words = 156 16-byte chunks; the block and each sim's state are 16-byte aligned
                const uint4* src = reinterpret_cast<const uint4*>(a.mt_states + s * kMtWords);
                for (int i = l; i < kMtWords / 4; i += W) reinterpret_cast<uint4*>(mt)[i] = __ldg(src + i);
                wp = kSeg;  // random.Random(seed): the first draw twists
            }
        }
        if (MODE == MT) __syncwarp();
        if (a.from_start) {
            // race.py:233-241: one free draw per competitor, in index order, resp at position 0
            double d[K];
            if constexpr (MODE == MT) {
                bool want[K];
#pragma unroll
                for (int k = 0; k < K; ++k) want[k] = do_it && running && has[k];
                mt_draws(want, d);
            } else {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int64_t at = cursor + cidx[k];
                    d[k] = at < cursor_end ? a.draws[at] : 1.0;
                }
            }
            if (do_it && running) {
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (has[k]) prev[k] = __dmul_rn((0.0 < bp[k]) ? rpE[k] : rpL[k], d[k]);
                if (MODE == INJECT) {
                    if (cursor + n > cursor_end) bad = true;  // stream shorter than the priming draws
                    cursor += n;
                }
            }
        }
        if (do_it && a.traj_pos && running) record(0);
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
            double lp[K];
            int rank[K];
#pragma unroll
            for (int k = 0; k < K; ++k) { lp[k] = __dsub_rn(L, pos[k]); rank[k] = 0; }
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
                for (int j = 0; j < W; ++j) {
                    const int64_t fr = shfl(fin[kk], base + j);
                    const double dr = shfl(lp[kk], base + j);
                    const int i = kk * W + j;
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        // non-short-circuit operators: predicated compares instead of branches
                        const bool less = (fr < fin[k]) | ((fr == fin[k]) & ((dr < lp[k]) | ((dr == lp[k]) & (i < cidx[k]))));
                        rank[k] += (i < n && less) ? 1 : 0;
                    }
                }
            }
            uint32_t seg_blk = 0;  // per-sim blocked steps: only for the per-sim output
            if (a.blocked)
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
                    for (int qq = 2; qq <= n - 1 - rank[k]; ++qq) f *= qq;
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
                    const int64_t o = s * n + cidx[k];
                    if (a.winner && rank[k] == 0) a.winner[s] = diverged ? -1 : cidx[k];
                    if (a.order) a.order[s * n + rank[k]] = cidx[k];
                    if (a.finish_ticks) a.finish_ticks[o] = fin[k] == INT64_MAX ? -1 : fin[k];
                    if (a.final_pos) a.final_pos[o] = pos[k];
                }
                if (l == 0) {
                    if (a.blocked) a.blocked[s] = seg_blk;
                    if (MODE == INJECT && a.draws_used) a.draws_used[s] = cursor - a.draw_offsets[s];
                }
                ct_tot += ct_sim;
                blk_tot += blk_sim;
            }
            const int64_t next = claim_next_sim(seg_done, l == 0, base, segs_total, a.work);
            if (seg_done) s = next;
            load_sim(seg_done);
        }
        if (!__any_sync(0xffffffffu, running)) break;

        // ---------------- kTicksPerBlock synchronous ticks ---------------------------------------
        __syncwarp();  // key rows: the previous block's reads precede this block's writes
        for (int tj = 0; tj < kTicksPerBlock; ++tj) {
            bool any_racing = false;
#pragma unroll
            for (int k = 0; k < K; ++k) any_racing |= racing[k];
            const unsigned rmask = __ballot_sync(0xffffffffu, any_racing);
            const bool seg_running = (rmask & segmask) != 0u;
            if (rmask == 0u) break;  // every segment finished inside this block

            // tick-limit check before the advance (race.py:381-386, 402-404)
#if BBE_MT_LIMIT_PRED
            {  // predicated, no branch
                const bool lim = seg_running && rt >= a.limit;
                diverged |= lim;
#pragma unroll
                for (int k = 0; k < K; ++k) racing[k] = racing[k] && !lim;
            }
#else
            if (seg_running && rt >= a.limit) {
                diverged = true;
#pragma unroll
                for (int k = 0; k < K; ++k) racing[k] = false;
            }
#endif

            // ---- front runner (race.py:244-264) ----
            // Coarse keys, as native64_kernel.cuh: key = mantissa bits 51..26 of pos + C64 (the host's
            // native64_frame puts every racing position of the race in one binade, so the key is a
            // monotone function of the position).  Each lane publishes v = (key << 5) | lane and keeps
            // one wrapped minimum of v_r + nk per rival (VIADDMNMX): the nearest rival after c in
            // (key, index) order.  With all racing keys of the segment distinct that is exactly the
            // reference's front (the smallest position strictly ahead, by its lowest index) and
            // gap = fl(p_front - p_c) is the reference's smallest gap (rounding is monotonic).  Two
            // racing competitors sharing a key always show up (the lower in (key, index) order finds
            // the other with an equal key), and so does a blocked lane whose front could be a
            // gap-rounding tie (distinct positions whose gaps round equal need p_front <= 2 gap); then
            // the whole warp reruns the reference's own loop over the segment's FP64 positions.
            double gap[K], pfp[K];
            bool ahead[K];
            int fk[K], fj[K];
#pragma unroll
            for (int k = 0; k < K; ++k) { gap[k] = CUDART_INF; pfp[k] = CUDART_INF; ahead[k] = false; fk[k] = 0; fj[k] = 0; }
            const int par = (tj & 1) * K * kKRow;
            if (a.scan) {
                uint32_t v[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const double y = __dadd_rn(pos[k], C64);
                    const uint32_t key = __funnelshift_r((uint32_t)__double2loint(y), (uint32_t)__double2hiint(y), 26);
                    v[k] = key * 32u + cl;
                    BBE_CHECK(in_dyn_smem(kw + par + k * kKRow, s_dyn) && (!lane_on || seg * WPK + l < kKRow - 1));
                    kw[par + k * kKRow] = racing[k] ? v[k] : 0u;
                }
                __syncwarp();
                bool coll = false;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    uint32_t bestv = 0xffffffffu;
                    int bestkk = 0;
                    bool any = false;
#pragma unroll
                    for (int kk = 0; kk < K; ++kk) {
                        // t = v_r + nk is < 2^31 iff rival r follows c in (key, index) order: rows below
                        // c's slot need a strictly larger key, c's own row a larger (key, lane), rows
                        // above a key at least as large; finished lanes and padding publish 0
                        const uint32_t nk = kk < k ? ~(v[k] | 31u) : (kk == k ? ~v[k] : 0u - (v[k] & ~31u));
                        uint32_t b0 = 0xffffffffu, b1 = 0xffffffffu;
                        const uint4* r4 = reinterpret_cast<const uint4*>(kr + par + kk * kKRow);
                        BBE_CHECK(in_dyn_smem(r4 + CHK - 1, s_dyn));
                        auto chunk = [&](const uint4 q) {
                            b0 = min(b0, q.x + nk);
                            b1 = min(b1, q.y + nk);
                            b0 = min(b0, q.z + nk);
                            b1 = min(b1, q.w + nk);
                        };
                        if (kNarrow) {
#pragma unroll
                            for (int c = 0; c < 3; ++c) chunk(r4[c]);
                        } else {
#pragma unroll 2
                            for (int c = 0; c < CHK; ++c) chunk(r4[c]);
                        }
                        const uint32_t t = min(b0, b1);
                        const uint32_t vf = t - nk;
                        if (t < 0x80000000u && (!any || (vf >> 5) < (bestv >> 5))) { bestv = vf; bestkk = kk; any = true; }
                    }
                    ahead[k] = any;
                    fk[k] = bestkk;
                    fj[k] = (int)(bestv & 31u);
                    coll |= racing[k] && any && (bestv >> 5) == (v[k] >> 5);
                }
#pragma unroll
                for (int kk = 0; kk < K; ++kk) {
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const double pr = shfl(pos[kk], base + fj[k]);
                        pfp[k] = (K == 1 || fk[k] == kk) ? pr : pfp[k];
                    }
                }
                bool need_exact = coll;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    gap[k] = ahead[k] ? __dsub_rn(pfp[k], pos[k]) : CUDART_INF;
                    need_exact |= racing[k] && ahead[k] && !(gap[k] > th[k]) && !(pfp[k] > __dmul_rn(2.0, gap[k]));
                }
                if (__any_sync(0xffffffffu, need_exact)) {
                    // race.py:244-264 verbatim over the segment's start-of-tick positions, in index order
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
            bool fr[K], bl[K];
            bool any_blocked = false;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                // race.py:271: free when nobody is strictly ahead (front is None) -- tested explicitly, as
                // gap = inf > theta fails for theta = inf or NaN -- or when gap > theta
                fr[k] = racing[k] && (!ahead[k] || gap[k] > th[k]);
                bl[k] = racing[k] && !fr[k];
                any_blocked |= bl[k];
            }
            double pf[K];
#pragma unroll
            for (int k = 0; k < K; ++k) pf[k] = 0.0;
            if (__any_sync(0xffffffffu, any_blocked)) {
#pragma unroll
                for (int kk = 0; kk < K; ++kk) {
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const double v = shfl(prev[kk], base + fj[k]);
                        pf[k] = (K == 1 || fk[k] == kk) ? v : pf[k];
                    }
                }
            }
            double draw[K];
            if constexpr (MODE == INJECT) {
                // free slots consume the stream in competitor-index order (slot-major, then lane)
                int seg_total = 0;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const unsigned fm = __ballot_sync(0xffffffffu, fr[k]) & segmask;
                    const int64_t at = cursor + seg_total + __popc(fm & lt_mask);
                    draw[k] = (fr[k] && at < cursor_end) ? __ldg(a.draws + at) : 1.0;
                    seg_total += __popc(fm);
                }
                cursor += seg_total;
                if (cursor > cursor_end) {  // stream too short: stop this sim, report at finalize
                    bad = true;
#pragma unroll
                    for (int k = 0; k < K; ++k) { racing[k] = false; fr[k] = bl[k] = false; }
                }
            } else {
                mt_draws(fr, draw);
            }

            // ---- synchronous update (race.py:299-320) ----
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const bool early = pos[k] < bp[k];
                double step;
                if (fr[k]) {
                    step = __dmul_rn(early ? rpE[k] : rpL[k], draw[k]);
                } else {
                    const double m = (pf[k] < prev[k]) ? pf[k] : prev[k];  // Python min(prev_c, prev_front)
                    step = __dmul_rn(early ? eE[k] : eL[k], m);
                }
                if (racing[k]) {
                    double p = __dadd_rn(pos[k], step);
                    if (p == pos[k]) p = nextafter(p, CUDART_INF);
                    pos[k] = p;
                    prev[k] = step;
                    ct_sim += 1;
                    blk_sim += bl[k] ? 1 : 0;
                    if (p >= L) { fin[k] = start + rt + 1; racing[k] = false; }
                }
            }
            if (seg_running && !diverged) {
                rt += 1;
                if (a.traj_pos && rt <= a.traj_cap) record(rt);
            }
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
        if (first_div != INT64_MAX) atomicMax((unsigned long long*)&a.tally[ct_at + 4], encode_first(first_div));
        if (first_bad != INT64_MAX) atomicMax((unsigned long long*)&a.tally[ct_at + 5], encode_first(first_bad));
    }
    __syncthreads();
    if (threadIdx.x == 0) release_work(a.work);
    for (int i = threadIdx.x; i < hist_len; i += blockDim.x) {
        const uint32_t v = s_hist[i];
        if (v) atomicAdd((unsigned long long*)&a.tally[i], (unsigned long long)v);
    }
}

}  // namespace bbe
