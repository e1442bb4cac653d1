// bbe_sim.cu -- C-ABI (include/bbe_sim.h) over the sm_100a race kernels.
//
// Host responsibilities: validate (race.py:175-189 errors), pack the race into a small SoA parameter
// block (one H2D copy), size a persistent grid to residency on this GPU, launch, and bring tallies
// (and optional per-sim records) back.  Each call leases a context (cached device buffers, pinned
// staging, a private stream) from a per-device pool, so concurrent host threads never share one.
// No CPU fallback exists: every entry point that needs a GPU returns BBE_ENODEV / BBE_ECUDA when
// there is none.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is dlopen'ed (nccl_api)
#ifdef BBE_TIMING
#include <chrono>
#endif
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: named ranges for nsys / ncu timelines

#include "../../include/bbe_sim.h"
#include "kernels.h"

using namespace bbe;

namespace {

thread_local std::string g_err;

#ifdef BBE_TIMING  // host-side timing probes of the call path (A/B builds only)
struct Probe {
    const char* name[16] = {};
    double sum[16] = {};
    long cnt[16] = {}, seen[16] = {};
    ~Probe() {
        for (int i = 0; i < 16; ++i)
            if (cnt[i]) std::fprintf(stderr, "probe %-28s %8.2f us\n", name[i], sum[i] / cnt[i]);
    }
} g_probe;
inline double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define PROBE_T0 double t_probe = now_us();
#define PROBE(i, nm)                                         \
    do {                                                     \
        const double t1_ = now_us();                         \
        g_probe.name[i] = nm;                                \
        if (++g_probe.seen[i] > 50) {                        \
            g_probe.sum[i] += t1_ - t_probe;                 \
            g_probe.cnt[i] += 1;                             \
        }                                                    \
        t_probe = t1_;                                       \
    } while (0)
#else
#define PROBE_T0
#define PROBE(i, nm)
#endif

struct NvtxRange {  // one named range per C-ABI call (free when no profiler is attached)
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define BBE_CK(x)                                                                                \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) return fail(BBE_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max(bytes, (size_t)4096);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
};

struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max(bytes, (size_t)4096);
        cudaError_t e = cudaMallocHost(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
};

struct DevCtx {
    bool busy = false;  // leased to one call (bbe_simulate_begin .. _end, or one async launch)
    int dev = -1;
    bool ready = false;
    int sm_count = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    HostBuf h_params, h_tally, h_seeds;  // h_seeds: bbe_rp_predict's MT dry-run seeds
    DevBuf d_params, d_draws, d_offsets, d_winner, d_order, d_fin, d_fpos, d_blocked, d_dused;
    DevBuf d_seeds, d_mt_states;  // MT mode
    DevBuf d_traj;                               // trajectories (positions, previous steps)
    DevBuf d_work;                               // work counters, a ring of kWorkSlots pairs
    std::map<std::pair<const void*, size_t>, int> occupancy;  // blocks per SM by (kernel, smem)
    int work_slot = 0;
    // bbe_rp_predict NATIVE: parameter H2D + kernel + tally D2H as one CUDA graph (one launch call
    // instead of three), re-instantiated when the kernel, grid or buffers change
    struct RpGraph {
        cudaGraph_t graph = nullptr;  // kept: its kernel node addresses the exec's node
        cudaGraphExec_t exec = nullptr;
        cudaGraphNode_t knode = nullptr;
        const void* fn = nullptr;
        int grid = 0;
        size_t smem = 0, bytes = 0, tbytes = 0;
        const void *hp = nullptr, *dp = nullptr, *ht = nullptr;
    } rp_graph;
    bool mt_table = false;                       // c_mt_init uploaded on this device
    // the call in flight between bbe_simulate_begin and bbe_simulate_end
    bool pending = false;
    bbe_result* pend_out = nullptr;
    int pend_n = 0, pend_nperm = 0, pend_K = 0;
    int64_t pend_ns = 0, pend_limit = 0;
    struct Copy { void* dst; const void* src; size_t bytes; };
    std::vector<Copy> pend_copies;  // pinned staging -> caller buffers, done in _end
    HostBuf h_out;                  // pinned staging of per-sim outputs
};

// Contexts (stream, events, staging buffers) are pooled per device and leased to one call at a
// time, so host threads can call concurrently: each call takes an idle context or creates one.
std::mutex g_ctx_mu;
std::vector<std::vector<DevCtx*>> g_pool;  // per device
thread_local DevCtx* tl_last = nullptr;    // the context of this thread's most recent launch
std::map<std::pair<int, const void*>, size_t> g_smem_limit;  // dynamic-smem limit set per (device, kernel)

void release_ctx(DevCtx* c) {
    std::lock_guard<std::mutex> g(g_ctx_mu);
    c->busy = false;
}

struct Lease {  // releases the context unless the call keeps it (a call left in flight)
    DevCtx* c = nullptr;
    bool keep = false;
    ~Lease() {
        if (c && !keep) release_ctx(c);
    }
};

int acquire_ctx(Lease& lease) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(BBE_ENODEV, "no CUDA device visible (the simulator has no CPU fallback)");
    }
    int dev = 0;
    BBE_CK(cudaGetDevice(&dev));
    DevCtx* c = nullptr;
    {
        std::lock_guard<std::mutex> g(g_ctx_mu);
        if ((int)g_pool.size() < ndev) g_pool.resize(ndev);
        for (DevCtx* p : g_pool[dev])
            if (!p->busy) {
                c = p;
                break;
            }
        if (!c) {
            c = new DevCtx();
            g_pool[dev].push_back(c);
        }
        c->busy = true;
    }
    lease.c = c;
    if (!c->ready) {
        c->dev = dev;
        BBE_CK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, dev));
        BBE_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        BBE_CK(cudaEventCreate(&c->ev0));
        BBE_CK(cudaEventCreate(&c->ev1));
        c->ready = true;
    }
    tl_last = c;
    return BBE_OK;
}

int64_t factorial(int n) {
    int64_t f = 1;
    for (int i = 2; i <= n; ++i) f *= i;
    return f;
}

int nperm_for(int n) { return n <= BBE_MAX_PERM_COMPETITORS ? (int)factorial(n) : 0; }

// race.py:175-189 / :42-44 / :62-66 / :87-91 / :108-116 (ids are checked by the Python host)
int validate(const bbe_race* race, const bbe_competitor* comps, const bbe_state* st, const bbe_request* rq) {
    if (!race || !comps || !st || !rq) return fail(BBE_EINVAL, "null argument");
    const int n = race->n;
    if (n < 1 || n > BBE_MAX_COMPETITORS)
        return fail(BBE_EINVAL, "n must be in [1, " + std::to_string(BBE_MAX_COMPETITORS) + "], got " + std::to_string(n));
    if (!(race->track_length > 0.0)) return fail(BBE_EINVAL, "track_length must be > 0");
    if (race->tick_limit < 1) return fail(BBE_EINVAL, "tick_limit must be >= 1");
    for (int c = 0; c < n; ++c) {
        const bbe_competitor& p = comps[c];
        if (p.family == BBE_FAMILY_UNIFORM) {
            if (!(0.0 < p.lo && p.lo <= p.hi)) return fail(BBE_EINVAL, "uniform steps need 0 < lo <= hi");
        } else if (p.family == BBE_FAMILY_LOGNORMAL) {
            if (p.sigma < 0.0) return fail(BBE_EINVAL, "lognormal sigma must be >= 0");
            if (!(p.scale > 0.0)) return fail(BBE_EINVAL, "lognormal scale must be > 0");
        } else {
            return fail(BBE_EINVAL, "unknown step family");
        }
        if (p.theta < 0.0) return fail(BBE_EINVAL, "theta must be >= 0");
        if (!(p.early_mult > 0.0) || !(p.late_mult > 0.0)) return fail(BBE_EINVAL, "responsiveness multipliers must be > 0");
        if (!(p.pref_factor > 0.0)) return fail(BBE_EINVAL, "pref_factor must be > 0");
    }
    if (!st->from_start && (!st->positions || !st->prev_steps || !st->finish_ticks))
        return fail(BBE_EINVAL, "continuation state needs positions, prev_steps and finish_ticks");
    if (rq->mode == BBE_MODE_NATIVE || rq->mode == BBE_MODE_NATIVE64) {
        // the front-runner frames (native_frame) need finite positions and track length
        if (!std::isfinite(race->track_length)) return fail(BBE_EINVAL, "mode native needs a finite track_length");
        for (int c = 0; !st->from_start && c < n; ++c)
            if (!std::isfinite(st->positions[c])) return fail(BBE_EINVAL, "mode native needs finite positions");
    }
    if (rq->n_sims < 0 || rq->sim_offset < 0) return fail(BBE_EINVAL, "n_sims and sim_offset must be >= 0");
    if (rq->group_size < 0) return fail(BBE_EINVAL, "group_size must be >= 0");
    if (rq->mode == BBE_MODE_INJECT) {
        if (!rq->draws || !rq->draw_offsets) return fail(BBE_EINVAL, "inject mode needs draws and draw_offsets");
    } else if (rq->mode != BBE_MODE_MT && rq->mode != BBE_MODE_NATIVE && rq->mode != BBE_MODE_NATIVE64) {
        return fail(BBE_EINVAL, "unknown mode");
    }
    return BBE_OK;
}

// Competitors per lane K for the NATIVE kernel (profiles/r1_k_sweep.md: every K timed for n = 6..128,
// with and without blocking competitors, after the 8/16-tick blocks).  util(K) = occupied slots /
// (32 K) with S = 32 / ceil(n/K) races per warp.  n > 32: without a scan K = 3 when it fits and fills
// >= 20 % more slots than K = 2, else (and with a scan: profiles/r1_sweep.md, n = 40) the smallest K
// that fits.  With a front-runner scan (some theta > 0): K = 1,
// or K = 2 when that fills >= 40 % more slots (K = 1 runs 16-tick blocks, K = 2 with a scan 4).
// Without: K = 2 (more independent work per lane), K = 1 when it fills > 10 % more slots, K = 3 when
// that fills > 15 % more than K = 2.
double slot_util(int n, int k) {
    const int w = (n + k - 1) / k;
    if (w > kWarp) return 0.0;
    return (double)n * (kWarp / w) / (kWarp * k);
}

int choose_k(int n, bool scan, int hint) {
    if (hint > 0 && hint <= 4 && (n + hint - 1) / hint <= kWarp) return hint;
    if (n > kWarp) {
        const double w2 = slot_util(n, 2), w3 = slot_util(n, 3);
        if (!scan && w2 > 0.0 && w3 > 0.0) return w3 >= 1.2 * w2 ? 3 : 2;
        for (int k = 2; k <= 4; ++k)
            if ((n + k - 1) / k <= kWarp) return k;
        return -1;
    }
    const double u1 = slot_util(n, 1), u2 = slot_util(n, 2), u3 = slot_util(n, 3);
    if (scan) return u2 >= 1.4 * u1 ? 2 : 1;
    if (u1 > 1.1 * u2) return 1;
    return u3 > 1.15 * u2 ? 3 : 2;
}

void pack_params(const bbe_race* race, const bbe_competitor* comps, const bbe_state* st, double* P) {
    const int n = race->n;
    for (int c = 0; c < n; ++c) {
        const bbe_competitor& p = comps[c];
        P[F_LO * n + c] = p.lo;
        P[F_SPAN * n + c] = p.hi - p.lo;  // uniform(a, b) = a + (b - a) * random()
        P[F_LMU * n + c] = p.mu + std::log(p.family == BBE_FAMILY_LOGNORMAL ? p.scale : 1.0);
        P[F_SIGMA * n + c] = p.sigma;
        P[F_SCALE * n + c] = p.scale;
        P[F_MU * n + c] = p.mu;
        P[F_RP_EARLY * n + c] = p.early_mult * p.pref_factor;  // (resp * pref), race.py:273
        P[F_RP_LATE * n + c] = p.late_mult * p.pref_factor;
        P[F_EARLY * n + c] = p.early_mult;
        P[F_LATE * n + c] = p.late_mult;
        P[F_BP * n + c] = p.bp_abs;
        P[F_THETA * n + c] = p.theta;
        if (st->from_start) {
            P[F_POS0 * n + c] = 0.0;
            P[F_PREV0 * n + c] = 0.0;
            P[F_FIN0 * n + c] = -1.0;
        } else {
            P[F_POS0 * n + c] = st->positions[c];
            P[F_PREV0 * n + c] = st->prev_steps[c];
            P[F_FIN0 * n + c] = (double)(st->finish_ticks[c] < 0 ? -1 : st->finish_ticks[c]);
        }
        P[F_FAMILY * n + c] = (double)p.family;
    }
    // Pre-finished competitors: their finish ticks only ever compare with each other and with later
    // (new) finishes, so an order-preserving compression to -m..-1 keeps _finish_order exact while
    // letting the kernel hold ticks as int32 relative to the state's tick.
    // (A finish tick after the state's own tick -- an inconsistent state -- keeps its plain offset.)
    for (int c = 0; c < n; ++c) {
        double rel = 0.0;
        if (!st->from_start && st->finish_ticks[c] > st->tick) {
            rel = (double)std::min<int64_t>(st->finish_ticks[c] - st->tick, INT32_MAX - 8);  // below the
                                                                                          // kernels' sentinels
        } else if (!st->from_start && st->finish_ticks[c] >= 0) {
            int greater_distinct = 0;
            for (int d = 0; d < n; ++d) {
                if (st->finish_ticks[d] < 0 || st->finish_ticks[d] > st->tick ||
                    st->finish_ticks[d] <= st->finish_ticks[c])
                    continue;
                bool seen = false;
                for (int e = 0; e < d; ++e)
                    if (st->finish_ticks[e] == st->finish_ticks[d]) seen = true;
                if (!seen) ++greater_distinct;
            }
            rel = -1.0 - greater_distinct;
        }
        P[F_FINREL * n + c] = rel;
    }
}

size_t param_bytes(int n) { return (size_t)F_COUNT * n * sizeof(double) + (size_t)NF_COUNT * n * sizeof(float); }

// NATIVE front-runner frame (native_kernel.cuh): an offset of positions, L and breakpoints, and the
// key base, such that every racing position p satisfies 1 <= bits(p) - key_base < 2^(31 - key_bits)
// for the whole race (racing positions only grow and stay below L, or start at their initial value).
// The offset is 0 whenever the state already fits (C2: positions ~900..2000).
struct NativeFrame {
    float shift;
    uint32_t key_base;
    int key_bits;
    double c64;      // NATIVE64: key of pos = mantissa bits 51..26 of pos + c64 (native64_frame)
    uint32_t sub64;  // NATIVE64: the exponent bit the key window drags in, << 31
    int flags64;     // NATIVE64: kN64RespVar | kN64Guard (native64_flags)
};

// NATIVE64 host flags (native64_kernel.cuh).  kN64RespVar: some competitor has early != late
// multiplier (so the per-tick breakpoint test matters).  kN64Guard: unless every step the race can
// take provably exceeds 2^-52 * B, B = the largest |position| a racing competitor can start a tick
// at (max(L, |initial positions|)), fl(pos + step) == pos is possible and the nextafter guard
// (race.py:310-313) stays.  Step lower bounds: free steps (resp * pref) * draw with draw >= lo
// (uniform: lo + span * r, r >= 0) or >= scale * exp(mu - 8.58 sigma) (Box-Muller |z| <= 8.572 for
// u1 >= 2^-53), halved for rounding; blocked steps resp * min(prev_c, prev_front) can shrink without
// bound when a multiplier is < 1, else stay >= the smallest free step and initial previous step.
int native64_flags(const bbe_race* race, const bbe_competitor* comps, const bbe_state* st) {
    const int n = race->n;
    int fl = 0;
    bool scan = false, small_mult = false;
    double min_free = INFINITY, min_prev = INFINITY, B = std::fabs(race->track_length);
    for (int c = 0; c < n; ++c) {
        const bbe_competitor& p = comps[c];
        const double rpE = p.early_mult * p.pref_factor, rpL = p.late_mult * p.pref_factor;
        if (!(rpE == rpL) || !(p.early_mult == p.late_mult)) fl |= kN64RespVar;
        const bool racing = st->from_start || st->finish_ticks[c] < 0;
        if (!racing) continue;
        scan = scan || !(p.theta <= 0.0);
        small_mult = small_mult || !(p.early_mult >= 1.0) || !(p.late_mult >= 1.0);
        const double dmin = p.family == BBE_FAMILY_LOGNORMAL ? p.scale * std::exp(p.mu - 8.58 * p.sigma) : p.lo;
        min_free = std::min(min_free, 0.5 * std::min(rpE, rpL) * dmin);
        if (!st->from_start) {
            min_prev = std::min(min_prev, st->prev_steps[c]);
            B = std::max(B, std::fabs(st->positions[c]));
        }
    }
    double step_min = min_free;
    if (scan) step_min = small_mult ? 0.0 : std::min(min_free, min_prev);
    if (!(step_min > std::ldexp(B, -52))) fl |= kN64Guard;
    // kN64NoTie: a blocked lane has gap <= theta_max and its front ahead at a position >= the smallest
    // racing start position (positions never decrease); when that exceeds 2 theta_max, p_front > 2 gap
    // always holds, so distinct positions can never round to the same gap (native64_kernel.cuh)
#ifndef BBE_N64_TIE_FLAG
#define BBE_N64_TIE_FLAG 1
#endif
    if (BBE_N64_TIE_FLAG && !st->from_start) {
        double theta_max = 0.0, min_pos = INFINITY;
        bool finite = true;
        for (int c = 0; c < n; ++c) {
            finite = finite && std::isfinite(comps[c].theta);
            theta_max = std::max(theta_max, comps[c].theta);
            if (st->finish_ticks[c] < 0) min_pos = std::min(min_pos, st->positions[c]);
        }
        if (finite && min_pos > 2.0 * theta_max) fl |= kN64NoTie;
    }
    return fl;
}

// NATIVE64 coarse front-runner key (native64_kernel.cuh): every racing position p -- from the
// smallest racing start position `base` up to hi = max(L, largest racing start position) -- maps to
// y = fl(p + c64) inside one binade (2^E, 2^(E+1)), so the 26 mantissa bits below the top are a
// monotone key of p with cells 2^(E-26) wide.  c64 = 2^E + 2^(E-20) - base: the 2^(E-20) margin keeps
// y above 2^E (and every racing key >= 2^6 > 0, the value of a finished lane) despite the rounding of
// c64 itself; 2^E >= (1 + 2^-10) (hi - base) keeps y below 2^(E+1).
void native64_frame(const bbe_race* race, const bbe_state* st, NativeFrame* fr) {
    const int n = race->n;
    double lo = INFINITY, hi = race->track_length;
    for (int c = 0; c < n; ++c) {
        if (!st->from_start && st->finish_ticks[c] >= 0) continue;
        const double p = st->from_start ? 0.0 : st->positions[c];
        lo = std::min(lo, p);
        hi = std::max(hi, p);
    }
    if (!(lo < INFINITY)) lo = 0.0;  // nobody racing: the scan never runs on a live key
    const double R = std::max(hi - lo, 1e-300) * (1.0 + 1.0 / 1024.0);
    int e = 0;
    std::frexp(R, &e);  // R < 2^e
    const double two_e = std::ldexp(1.0, e);
    fr->c64 = two_e + std::ldexp(1.0, e - 20) - lo;
    const int biased = e + 1023;  // exponent field of y
    fr->sub64 = (uint32_t)(biased & 1) << 31;
}

uint32_t f32_bits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, sizeof u);
    return u;
}

NativeFrame native_frame(const bbe_race* race, const bbe_state* st, int W) {
    // 5 index bits for every layout (W <= 32): the frame, and so every FP32 operation of a sim, is
    // then the same whatever competitors-per-lane layout runs it
    (void)W;
    NativeFrame fr{0.0f, f32_bits(1.0f) - 1u, 5};
    const uint64_t R = 1ull << (31 - fr.key_bits);
    const int n = race->n;
    auto racing = [&](int c) { return st->from_start || st->finish_ticks[c] < 0; };
    auto pos_of = [&](int c) { return st->from_start ? 0.0 : st->positions[c]; };
    double min_pos = INFINITY;
    for (int c = 0; c < n; ++c)
        if (racing(c)) min_pos = std::min(min_pos, pos_of(c));
    if (!(min_pos < INFINITY)) return fr;  // nobody racing: the scan never runs on a live key
    // whether `shift` is a valid frame; sets key_base
    auto fits = [&](float shift) {
        float lo = INFINITY, hi = (float)race->track_length + shift;  // the kernel's L
        for (int c = 0; c < n; ++c) {
            if (!racing(c)) continue;
            const float p = (float)(pos_of(c) + (double)shift);  // as packed below
            lo = std::min(lo, p);
            hi = std::max(hi, p);
        }
        if (!(lo > 0.0f) || !(hi < INFINITY)) return false;
        fr.key_base = f32_bits(lo) - 1u;
        return (uint64_t)(f32_bits(hi) - fr.key_base) < R;
    };
    if (min_pos > 0.0 && fits(0.0f)) return fr;
    for (int e = 0; e < 128; ++e) {
        const double target = std::ldexp(1.0, e);
        if (target <= min_pos) continue;
        for (float shift : {(float)(target - min_pos), std::nextafter((float)(target - min_pos), INFINITY)}) {
            if (fits(shift)) {
                fr.shift = shift;
                return fr;
            }
        }
    }
    fr.shift = NAN;  // unreachable for finite inputs (validate() rejects non-finite ones)
    return fr;
}

NativeFrame native_frames(const bbe_race* race, const bbe_competitor* comps, const bbe_state* st, int W) {
    NativeFrame fr = native_frame(race, st, W);
    native64_frame(race, st, &fr);
    fr.flags64 = native64_flags(race, comps, st);
    return fr;
}

// NATIVE FP32 block, appended after the double block, in the frame `fr`.
void pack_params_f32(const bbe_race* race, const bbe_competitor* comps, const bbe_state* st, double* P,
                     const NativeFrame& fr) {
    const int n = race->n;
    float* F = reinterpret_cast<float*>(P + (size_t)F_COUNT * n);
    const double shift = fr.shift;
    const double log2e = 1.4426950408889634;
    for (int c = 0; c < n; ++c) {
        const bbe_competitor& p = comps[c];
        const double span = p.hi - p.lo;
        F[NF_LO_MINUS_SPAN * n + c] = (float)(p.lo - span);
        F[NF_SPAN * n + c] = (float)span;
        F[NF_SG2 * n + c] = (float)(p.sigma * log2e);
        F[NF_LMU2 * n + c] = (float)((p.mu + std::log(p.family == BBE_FAMILY_LOGNORMAL ? p.scale : 1.0)) * log2e);
        F[NF_RP_EARLY * n + c] = (float)(p.early_mult * p.pref_factor);
        F[NF_RP_LATE * n + c] = (float)(p.late_mult * p.pref_factor);
        F[NF_EARLY * n + c] = (float)p.early_mult;
        F[NF_LATE * n + c] = (float)p.late_mult;
        F[NF_BP * n + c] = (float)(p.bp_abs + shift);
        F[NF_THETA * n + c] = (float)p.theta;
        F[NF_POS0 * n + c] = (float)((st->from_start ? 0.0 : st->positions[c]) + shift);
        F[NF_PREV0 * n + c] = st->from_start ? 0.0f : (float)st->prev_steps[c];
    }
}

void philox_round_keys(uint64_t seed, uint32_t* rk) {
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        rk[2 * r] = k0;
        rk[2 * r + 1] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

#ifndef BBE_NATIVE_VEC2
#define BBE_NATIVE_VEC2 1
#endif

struct Plan {
    int mode, n, K, W, S, CH, WP, nperm, tally_len, NT;
    size_t smem;
    KernelFn fn;
    int grid;
};

// Expected ticks until the last racing competitor finishes, ignoring blocking: max over racing c of
// (L - pos_c) / (mean step of c), the mean step at the smaller responsiveness multiplier.
double expected_ticks(const bbe_race* race, const bbe_competitor* comps, const bbe_state* st) {
    double t = 0.0;
    for (int c = 0; c < race->n; ++c) {
        if (!st->from_start && st->finish_ticks[c] >= 0) continue;
        const bbe_competitor& p = comps[c];
        const double draw = p.family == BBE_FAMILY_LOGNORMAL ? p.scale * std::exp(p.mu + 0.5 * p.sigma * p.sigma)
                                                             : 0.5 * (p.lo + p.hi);
        const double step = p.pref_factor * std::min(p.early_mult, p.late_mult) * draw;
        const double rem = race->track_length - (st->from_start ? 0.0 : st->positions[c]);
        if (step > 0.0) t = std::max(t, rem / step);
    }
    return t;
}

// NATIVE ticks per block (native_kernel.cuh NT) from the expected race length T.  A boundary costs
// about 1.5 ticks' work at C2 (more in scan-free fields) and a finished segment idles (NT-1)/2 ticks
// on average; the thresholds are read off a sweep of NT over race lengths (profiles/r1_ticks_sweep.md):
// K = 1: 16 from ~43 ticks, else 8; K = 2 without a scan: 16 from ~21 ticks, else 4; other layouts 4
// (longer blocks spill there).  BBE_TICKS overrides (tuning).
int pick_ticks(int K, bool scan, double T) {
    static const int env = [] {
        const char* e = std::getenv("BBE_TICKS");
        return e ? std::atoi(e) : 0;
    }();
    if (env == 4 || env == 8 || env == 16) return K == 1 ? (env == 16 ? 16 : 8) : env;
    if (K == 1) return T >= 43.0 ? 16 : 8;
    if (K == 2 && !scan) return T >= 21.0 ? 16 : 4;
    return 4;
}

// NATIVE64 ticks per block: scan-free fields 16 from ~43 expected ticks (the FP32 K = 1 threshold),
// else 8; with a scan 8 (the only build).
int pick_ticks64(bool scan, double T) {
    static const int env = [] {
        const char* e = std::getenv("BBE_TICKS64");
        return e ? std::atoi(e) : 0;
    }();
    if (scan) return BBE_N64_SCAN_NT;
    if (env == 8 || env == 16) return env;
    return T >= 43.0 ? 16 : 8;
}

KernelFn pick_native64_scan(int k, int ch, bool ln) {
    if (k == 1) return ln ? pick_native64_scan_k1_ln1(k, ch) : pick_native64_scan_k1_ln0(k, ch);
    return ln ? pick_native64_scan_kn_ln1(k, ch) : pick_native64_scan_kn_ln0(k, ch);
}

KernelFn pick_native(int k, int ch, bool scan, int vec, int nt) {
    if (k == 1) return nt == 16 ? pick_native_k1_nt16(ch, scan, vec) : pick_native_k1_nt8(ch, scan, vec);
    if (vec != 4) return nullptr;
    return nt == 16 ? pick_native_kn_nt16(k, ch, scan) : pick_native_kn_nt4(k, ch, scan);
}

int make_plan(DevCtx* ctx, const bbe_race* race, const bbe_competitor* comps, const bbe_state* st,
              const bbe_request* rq, int want_perms, Plan* pl) {
    bool scan = false;  // any theta > 0 (or NaN: `gap > NaN` is false, race.py:271): the scan is needed
    bool ln = false;    // any lognormal competitor (MT: speculative draw rounds)
    for (int c = 0; c < race->n; ++c) {
        scan = scan || !(comps[c].theta <= 0.0);
        ln = ln || comps[c].family == BBE_FAMILY_LOGNORMAL;
    }
    const int n = race->n;
    pl->mode = rq->mode;
    pl->n = n;
    // exact modes: the fewest slots that fit a warp (an MT slot adds a speculative word window per
    // lane); NATIVE: the measured layout rule
    const int k_min = (n + kWarp - 1) / kWarp;
    const bool native = rq->mode == BBE_MODE_NATIVE || rq->mode == BBE_MODE_NATIVE64;
    if (native) pl->K = choose_k(n, scan, rq->lanes_per_slot_hint);
    else pl->K = (rq->lanes_per_slot_hint >= k_min && rq->lanes_per_slot_hint <= 4) ? rq->lanes_per_slot_hint : k_min;
    if (pl->K > 4) pl->K = -1;
    if (pl->K < 0) return fail(BBE_EINVAL, "field too large for one warp");
    pl->W = (n + pl->K - 1) / pl->K;
    if (rq->mode == BBE_MODE_MT) pl->W = std::max(pl->W, 8);  // <= 4 MT states (2.5 KB each) per warp
    pl->S = kWarp / pl->W;
    // NATIVE K = 1 with a scan: 2-word key loads when that avoids padding keys (W % 4 in {1, 2})
    const bool vec2 = BBE_NATIVE_VEC2 && rq->mode == BBE_MODE_NATIVE && pl->K == 1 && scan &&
                      ((pl->W + 1) & ~1) < ((pl->W + 3) & ~3);
    pl->CH = vec2 ? (pl->W + 1) / 2 : (pl->W + 3) / 4;  // NATIVE64: always 4-word chunks
    pl->WP = (vec2 ? 2 : 4) * pl->CH;
    pl->nperm = want_perms ? nperm_for(n) : 0;
    TallyLayout TL{n, pl->nperm};
    pl->tally_len = TL.len();
    const int kmode = rq->mode == BBE_MODE_NATIVE ? NATIVE
                      : rq->mode == BBE_MODE_NATIVE64 ? NATIVE64 : (rq->mode == BBE_MODE_MT ? MT : INJECT);
    pl->smem = smem_bytes(kmode, (TL.hist_len() + 1) & ~1, pl->K, pl->S, pl->WP);
    if (rq->mode == BBE_MODE_NATIVE64) {
        pl->NT = pick_ticks64(scan, expected_ticks(race, comps, st));
        pl->smem = smem_bytes(kmode, (TL.hist_len() + 1) & ~1, pl->K, pl->S, scan ? pl->WP : 0, pl->NT);
        pl->fn = scan ? pick_native64_scan(pl->K, pl->CH, ln) : pick_native64_free(pl->K, ln, pl->NT);
    } else {
        pl->NT = rq->mode == BBE_MODE_NATIVE ? pick_ticks(pl->K, scan, expected_ticks(race, comps, st)) : 4;
        pl->fn = rq->mode == BBE_MODE_NATIVE ? pick_native(pl->K, pl->CH, scan, vec2 ? 2 : 4, pl->NT)
                                             : pick_exact(rq->mode == BBE_MODE_MT ? MT : INJECT, pl->K, ln, pl->S <= 2);
    }
    if (!pl->fn && rq->mode == BBE_MODE_NATIVE && pl->NT != 4) {
        pl->NT = 4;  // that block length is not built for this layout
        pl->fn = pick_native(pl->K, pl->CH, scan, vec2 ? 2 : 4, 4);
    }
    if (!pl->fn) return fail(BBE_EINVAL, "no kernel for this configuration");
    // the kernel's dynamic-smem limit only ever grows (a smaller later request keeps the larger
    // limit valid); residency per (kernel, dynamic smem) is queried once per device
    if (pl->smem > 48 * 1024) {
        // the limit is a device-wide attribute of the kernel: tracked per (device, kernel) for all
        // contexts, and only ever raised
        std::lock_guard<std::mutex> g(g_ctx_mu);
        size_t& limit = g_smem_limit[std::make_pair(ctx->dev, (const void*)pl->fn)];
        if (pl->smem > limit) {
            BBE_CK(cudaFuncSetAttribute((const void*)pl->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl->smem));
            limit = pl->smem;
        }
    }
    int per_sm = 0;
    const auto key = std::make_pair((const void*)pl->fn, pl->smem);
    auto it = ctx->occupancy.find(key);
    if (it != ctx->occupancy.end()) {
        per_sm = it->second;
    } else {
        BBE_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl->fn, kBlockThreads, pl->smem));
        ctx->occupancy[key] = per_sm;
    }
    if (per_sm < 1) per_sm = 1;
    const int64_t sims_per_block = (int64_t)(kBlockThreads / kWarp) * pl->S;
    const int64_t need = (rq->n_sims + sims_per_block - 1) / sims_per_block;
    const int64_t cap = (int64_t)per_sm * ctx->sm_count;
    pl->grid = (int)std::max<int64_t>(1, std::min(need, cap));
    return BBE_OK;
}

}  // namespace

extern "C" {

uint32_t bbe_host_mt_getrandbits64(uint32_t* mt, uint32_t idx, int64_t count, uint64_t* out, int64_t out_len);

int bbe_version(void) { return BBE_ABI_VERSION; }

float bbe_last_kernel_ms(void) {
    DevCtx* ctx = tl_last;
    if (!ctx) return -1.f;
    if (cudaEventSynchronize(ctx->ev1) != cudaSuccess) return -1.f;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1) != cudaSuccess) {
        cudaGetLastError();
        return -1.f;
    }
    return ms;
}

const char* bbe_last_error(void) { return g_err.c_str(); }

int bbe_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int bbe_device_info(int device, char* name64, int32_t* sm_count, int32_t* clock_khz) {
    cudaDeviceProp p;
    BBE_CK(cudaGetDeviceProperties(&p, device));
    if (name64) {
        std::strncpy(name64, p.name, 63);
        name64[63] = 0;
    }
    if (sm_count) *sm_count = p.multiProcessorCount;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
    if (clock_khz) *clock_khz = clk;
    return BBE_OK;
}

int bbe_mt_getrandbits64(uint32_t* st, int64_t count, uint64_t* out) {
    if (!st || count < 0) return fail(BBE_EINVAL, "bad arguments");
    if (st[624] > 624) return fail(BBE_EINVAL, "MT19937 position out of range");
    st[624] = bbe_host_mt_getrandbits64(st, st[624], count, out, count);  // host_mt.cpp
    return BBE_OK;
}

int bbe_mt_advance64(uint32_t* state624, int32_t* pos, int64_t count, uint64_t* out, int64_t out_len) {
    if (!state624 || !pos || count < 0 || *pos < 0 || *pos > 624) return fail(BBE_EINVAL, "bad arguments");
    *pos = (int32_t)bbe_host_mt_getrandbits64(state624, (uint32_t)*pos, count, out, out ? out_len : 0);
    return BBE_OK;
}

int bbe_mt_advance64_many(int64_t n_gen, uint32_t* const* states, int32_t* const* pos, const int64_t* counts,
                          uint64_t* const* outs, const int64_t* out_lens, int32_t threads) {
    NvtxRange nvtx_range("bbe_mt_advance64_many");
    if (n_gen < 0 || (n_gen && (!states || !pos || !counts))) return fail(BBE_EINVAL, "bad arguments");
    for (int64_t g = 0; g < n_gen; ++g)
        if (!states[g] || !pos[g] || counts[g] < 0 || *pos[g] < 0 || *pos[g] > 624)
            return fail(BBE_EINVAL, "bad generator " + std::to_string(g));
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    int64_t words = 0;
    for (int64_t g = 0; g < n_gen; ++g) words += counts[g];
    // below ~64k draws the thread start-up costs more than it saves
    threads = (int)std::min<int64_t>(threads, std::max<int64_t>(1, std::min<int64_t>(n_gen, words / 65536 + 1)));
    // a generator listed more than once is advanced by one thread, in list order (its owner: the
    // thread of its first occurrence), so no two threads ever write the same state
    std::vector<int> owner(n_gen);
    {
        std::map<const uint32_t*, int> first;
        for (int64_t g = 0; g < n_gen; ++g) {
            auto it = first.find(states[g]);
            owner[g] = it == first.end() ? (int)(g % threads) : it->second;
            if (it == first.end()) first.emplace(states[g], owner[g]);
        }
    }
    auto work = [&](int t) {
        for (int64_t g = 0; g < n_gen; ++g) {
            if (owner[g] != t) continue;
            uint64_t* o = outs ? outs[g] : nullptr;
            const int64_t ol = (o && out_lens) ? out_lens[g] : 0;
            *pos[g] = (int32_t)bbe_host_mt_getrandbits64(states[g], (uint32_t)*pos[g], counts[g], o, o ? ol : 0);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    return BBE_OK;
}

int64_t bbe_param_bytes(int32_t n) {
    if (n < 1 || n > BBE_MAX_COMPETITORS) return -1;
    return (int64_t)param_bytes(n);
}

int64_t bbe_tally_len(int32_t n) {
    if (n < 1 || n > BBE_MAX_COMPETITORS) return -1;
    return TallyLayout{n, nperm_for(n)}.len();
}

int64_t bbe_tally_offset(int32_t n, int32_t field) {
    if (n < 1 || n > BBE_MAX_COMPETITORS) return -1;
    TallyLayout T{n, nperm_for(n)};
    switch (field) {
        case 0: return T.wins();
        case 1: return T.ranks();
        case 2: return T.perms();
        case 3: return T.ct();
        case 4: return T.blocked();
        case 5: return T.n_div();
        case 6: return T.n_bad();
        case 7: return T.first_div();
        case 8: return T.first_bad();
    }
    return -1;
}

// seeding.py:24-59, the per-run seeds of batch.py:117-119
static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
static uint64_t fnv1a(const unsigned char* b, int len) {
    uint64_t h = 0xCBF29CE484222325ull;
    for (int i = 0; i < len; ++i) h = (h ^ b[i]) * 0x100000001B3ull;
    return h;
}

int bbe_derive_seeds(uint64_t master, int64_t first, int64_t count, uint64_t* out) {
    if (!out || count < 0) return fail(BBE_EINVAL, "bad arguments");
    const unsigned char run[5] = {'s', ':', 'r', 'u', 'n'};
    const uint64_t h0 = splitmix64(splitmix64(master) ^ fnv1a(run, 5));
    for (int64_t j = 0; j < count; ++j) {
        const uint64_t i = (uint64_t)(first + j);
        unsigned char b[10] = {'i', ':'};
        for (int k = 0; k < 8; ++k) b[2 + k] = (unsigned char)(i >> (56 - 8 * k));
        out[j] = splitmix64(h0 ^ fnv1a(b, 10));
    }
    return BBE_OK;
}

constexpr int64_t kRpSplitMin = 16384;  // bbe_rp_predict MT: one part per this many dry runs
#ifndef BBE_RP_FIRST
#define BBE_RP_FIRST 15  // percent of an MT bbe_rp_predict call in its first part (C2: 50 -> 2.53 ms, 25 -> 2.50, 15 -> 2.49)
#endif
#ifndef BBE_RP_PARTS
#define BBE_RP_PARTS 2  // at most this many parts (streams) per MT bbe_rp_predict call (C2: 3 or 4 parts were 1.5 % slower)
#endif
constexpr int kWorkSlots = 64;  // concurrent native launches per device with their own work counters
constexpr size_t kMaxStagedBytes = 256ull << 20;  // per-sim outputs staged through pinned memory up to this

// The kernels' shared-memory histograms are 32-bit: a launch never runs 2^32 or more sims.
constexpr int64_t kMaxLaunchSims = 1ll << 31;

// The launch arguments of sims [c0, c0 + cn) of `a`: per-sim streams and outputs are indexed by the
// launch-local sim index, so every per-sim pointer moves by c0.
static LaunchArgs sub_launch(const LaunchArgs& a, int64_t c0, int64_t cn) {
    LaunchArgs b = a;
    const int64_t n = a.n;
    b.n_sims = cn;
    b.sim_offset = a.sim_offset + c0;
    b.group_base = a.group_base + c0;
    if (b.draw_offsets) b.draw_offsets += c0;
    if (b.draws_used) b.draws_used += c0;
    if (b.mt_states) b.mt_states += c0 * kMtWords;
    if (b.winner) b.winner += c0;
    if (b.order) b.order += c0 * n;
    if (b.finish_ticks) b.finish_ticks += c0 * n;
    if (b.final_pos) b.final_pos += c0 * n;
    if (b.blocked) b.blocked += c0;
    if (b.traj_pos) {
        b.traj_pos += c0 * ((int64_t)b.traj_cap + 1) * n;
        b.traj_prev += c0 * ((int64_t)b.traj_cap + 1) * n;
    }
    return b;
}

// The launch's work-counter pair (the kernel leaves it zeroed; consecutive launches rotate through
// the ring) and its persistent grid (never more blocks than the launch's sims need).
static int prepare_launch(DevCtx* ctx, const Plan& pl, cudaStream_t stream, LaunchArgs* a, int* grid) {
    if (!ctx->d_work.p) {
        BBE_CK(ctx->d_work.ensure(kWorkSlots * 2 * sizeof(unsigned long long)));
        BBE_CK(cudaMemsetAsync(ctx->d_work.p, 0, kWorkSlots * 2 * sizeof(unsigned long long), stream));
        BBE_CK(cudaStreamSynchronize(stream));
    }
    a->work = (unsigned long long*)ctx->d_work.p + 2 * ctx->work_slot;
    ctx->work_slot = (ctx->work_slot + 1) % kWorkSlots;
    const int64_t sims_per_block = (int64_t)kWarpsPerBlock * pl.S;
    *grid = (int)std::max<int64_t>(1, std::min<int64_t>(pl.grid, (a->n_sims + sims_per_block - 1) / sims_per_block));
    return BBE_OK;
}

static int launch_one(DevCtx* ctx, const Plan& pl, const LaunchArgs& a0, cudaStream_t stream) {
    if (a0.n_sims == 0) return BBE_OK;
    if (a0.n_sims > kMaxLaunchSims) {
        for (int64_t c0 = 0; c0 < a0.n_sims; c0 += kMaxLaunchSims) {
            const int rc = launch_one(ctx, pl, sub_launch(a0, c0, std::min(kMaxLaunchSims, a0.n_sims - c0)), stream);
            if (rc) return rc;
        }
        return BBE_OK;
    }
    LaunchArgs a = a0;
    int grid = 0;
    int rc = prepare_launch(ctx, pl, stream, &a, &grid);
    if (rc) return rc;
    pl.fn<<<grid, kBlockThreads, pl.smem, stream>>>(a);
    BBE_CK(cudaGetLastError());
    return BBE_OK;
}

constexpr int64_t kMtChunk = 131072;  // sims seeded per MT chunk: 320 MB of seeded states

// init_genrand(19650218) (CPython _randommodule.c), the start of every init_by_array
static void mt_init_table(uint32_t* t) {
    t[0] = 19650218u;
    for (int i = 1; i < kMtWords; ++i) t[i] = 1812433253u * (t[i - 1] ^ (t[i - 1] >> 30)) + (uint32_t)i;
}

// ---- the host libm's exp table (see mt_stream.cuh: libm_exp) ----
struct LibmExp {
    bool ok = false;
    double c[8];
    uint64_t tab[256];
};

static double host_libm_exp(const LibmExp& E, double x) {  // the kernel's evaluation order, on the host
    double kd = std::fma(E.c[0], x, E.c[1]);
    uint64_t ki;
    std::memcpy(&ki, &kd, 8);
    kd = kd - E.c[1];
    const double r = std::fma(kd, E.c[3], std::fma(kd, E.c[2], x));
    const int idx = 2 * (int)(ki % 128u);
    const uint64_t sbits = E.tab[idx + 1] + (ki << 45);
    double tail, scale;
    std::memcpy(&tail, &E.tab[idx], 8);
    std::memcpy(&scale, &sbits, 8);
    const double r2 = r * r;
    const double tmp = std::fma(r2 * r2, std::fma(r, E.c[7], E.c[6]), std::fma(r2, std::fma(r, E.c[5], E.c[4]), tail + r));
    return std::fma(scale, tmp, scale);
}

// Locate glibc's __exp_data (N/ln2, 0x1.8p52, -ln2hi/N, -ln2lo/N, C2..C5, ..., table of 2^(i/128))
// in the libm file the process loaded, then check the evaluation against exp() itself.
static const LibmExp& libm_exp_table() {
    static LibmExp E;
    static std::once_flag once;
    std::call_once(once, [] {
        Dl_info info;
        if (!dladdr((void*)static_cast<double (*)(double)>(&::exp), &info) || !info.dli_fname) return;
        FILE* f = std::fopen(info.dli_fname, "rb");
        if (!f) return;
        std::vector<unsigned char> b;
        unsigned char chunk[65536];
        size_t got;
        while ((got = std::fread(chunk, 1, sizeof(chunk), f)) > 0) b.insert(b.end(), chunk, chunk + got);
        std::fclose(f);
        const uint64_t inv = 0x40671547652b82feull, shift = 0x4338000000000000ull, one = 0x3ff0000000000000ull;
        for (size_t i = 0; i + 8 * 300 <= b.size(); i += 8) {
            uint64_t q0;
            std::memcpy(&q0, &b[i], 8);
            if (q0 != inv) continue;
            uint64_t q[300];
            std::memcpy(q, &b[i], sizeof(q));
            if (q[1] != shift) continue;
            for (int t = 8; t < 40; ++t) {
                if (q[t] != 0 || q[t + 1] != one) continue;
                for (int k = 0; k < 8; ++k) std::memcpy(&E.c[k], &q[k], 8);
                std::memcpy(E.tab, &q[t], sizeof(E.tab));
                uint64_t s = 88172645463325252ull;
                bool good = true;
                for (int n = 0; n < 20000 && good; ++n) {
                    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
                    const double x = ((double)(s >> 11) / 9007199254740992.0) * 40.0 - 20.0;
                    const double a = host_libm_exp(E, x), ref = std::exp(x);
                    good = std::memcmp(&a, &ref, 8) == 0;
                }
                E.ok = good;
                return;
            }
        }
    });
    return E;
}

static uint64_t h_run_of(uint64_t master) {  // splitmix64(splitmix64(master) ^ fnv1a("s:run"))
    uint64_t h = 0xCBF29CE484222325ull;
    for (char ch : std::string("s:run")) h = (h ^ (unsigned char)ch) * 0x100000001B3ull;
    return splitmix64_host(splitmix64_host(master) ^ h);
}

// Launch the race kernel for the whole request (MT: chunked seeding + race per chunk).  `d_seeds`
// (MT, device, per-sim) may be NULL -> derive_seed(seed_master, "run", global index).
static int launch_all(DevCtx* ctx, const Plan& pl, LaunchArgs a, const bbe_competitor* comps, const uint64_t* d_seeds,
                      uint64_t seed_master, cudaStream_t stream) {
    a.scan = 0;
    for (int c = 0; c < a.n; ++c)
        if (!(comps[c].theta <= 0.0)) a.scan = 1;  // theta > 0 or NaN (see make_plan)
    if (pl.mode != BBE_MODE_MT) return launch_one(ctx, pl, a, stream);

    if (!ctx->mt_table) {
        uint32_t t[kMtWords];
        mt_init_table(t);
        const LibmExp& E = libm_exp_table();
        BBE_CK(upload_mt_tables(t, E.ok ? 1 : 0, E.tab, E.c));
        ctx->mt_table = true;
    }
    a.nv_magic = 4 * std::exp(-0.5) / std::sqrt(2.0);  // random.NV_MAGICCONST, host libm
    const int64_t total = a.n_sims;
    const int64_t chunk = std::min<int64_t>(total, kMtChunk);
    const int64_t pad = (chunk + 31) & ~31;
    BBE_CK(ctx->d_mt_states.ensure((size_t)pad * kMtWords * 4));
    const uint64_t h_run = h_run_of(seed_master);
    const int64_t off0 = a.sim_offset;
    for (int64_t c0 = 0; c0 < total; c0 += chunk) {
        const int64_t cn = std::min(chunk, total - c0);
        BBE_CK(launch_mt_seed(stream, d_seeds ? d_seeds + c0 : nullptr, h_run, off0 + c0, cn,
                              (uint32_t*)ctx->d_mt_states.p));
        LaunchArgs b = sub_launch(a, c0, cn);
        b.mt_states = (const uint32_t*)ctx->d_mt_states.p;  // the chunk's seeded states
        int rc = launch_one(ctx, pl, b, stream);
        if (rc) return rc;
    }
    return BBE_OK;
}

static int build_args(const Plan& pl, const bbe_race* race, const bbe_state* st, const bbe_request* rq,
                      const double* d_params, const double* d_draws, const int64_t* d_offsets, uint64_t* d_tally,
                      const bbe_result* dev_out, const NativeFrame& fr, LaunchArgs* out) {
    LaunchArgs& a = *out;
    a = LaunchArgs{};
    a.P = d_params;
    a.Pf = reinterpret_cast<const float*>(d_params + (size_t)F_COUNT * race->n);
    a.shift = fr.shift;
    a.key_base = fr.key_base;
    a.key_bits = fr.key_bits;
    a.key_mul = 1u << fr.key_bits;
    a.key_nmul = 0u - a.key_mul;
    a.key_c64 = fr.c64;
    a.key_sub64 = fr.sub64;
    a.n64_flags = fr.flags64;
    philox_round_keys(rq->seed, a.rk);
    a.n = race->n;
    a.W = pl.W;
    a.S = pl.S;
    a.WP = pl.WP;
    a.from_start = st->from_start ? 1 : 0;
    a.perms = pl.nperm;
    a.L = race->track_length;
    a.tick0 = st->from_start ? 0 : st->tick;
    a.limit = (int32_t)std::min<int64_t>(race->tick_limit, INT32_MAX);
    a.n_sims = rq->n_sims;
    a.sim_offset = rq->sim_offset;
    a.seed = rq->seed;
    a.draws = d_draws;
    a.draw_offsets = d_offsets;
    a.tally = d_tally;
    if (dev_out) {
        a.winner = dev_out->winner;
        a.order = dev_out->order;
        a.finish_ticks = dev_out->finish_ticks;
        a.final_pos = dev_out->final_positions;
        a.blocked = dev_out->blocked;
        a.draws_used = dev_out->draws_used;
        if (rq->group_size > 0 && dev_out->group_wins) {
            a.group_wins = (unsigned long long*)dev_out->group_wins;
            a.group_size = rq->group_size;
        }
        a.traj_pos = dev_out->traj_cap > 0 ? dev_out->traj_positions : nullptr;
        a.traj_prev = dev_out->traj_cap > 0 ? dev_out->traj_prev_steps : nullptr;
        a.traj_cap = dev_out->traj_cap;
    }
    return BBE_OK;
}

int bbe_simulate_begin(const bbe_race* race, const bbe_competitor* comps, const bbe_state* st, const bbe_request* rq,
                       bbe_result* out) {
    NvtxRange nvtx_range("bbe_simulate_begin");
    PROBE_T0
    int rc = validate(race, comps, st, rq);
    if (rc) return rc;
    if (!out || !out->wins) return fail(BBE_EINVAL, "result needs a wins buffer");
    Lease lease;
    if ((rc = acquire_ctx(lease))) return rc;
    DevCtx* const ctx = lease.c;
    const int n = race->n;
    const int64_t ns = rq->n_sims;
    PROBE(0, "begin: validate+acquire");
    Plan pl;
    if ((rc = make_plan(ctx, race, comps, st, rq, out->perms != nullptr, &pl))) return rc;
    cudaStream_t s = ctx->stream;
    PROBE(1, "begin: plan");

    // parameters and the zeroed tally: one pinned staging block, one H2D copy
    const size_t pbytes = (param_bytes(n) + 63) & ~(size_t)63;
    const size_t tbytes = (size_t)pl.tally_len * sizeof(uint64_t);
    // per-group winner counts (zeroed with the tally)
    const bool groups = rq->group_size > 0 && out->group_wins && ns > 0;
    const size_t gbytes = groups ? (size_t)((ns + rq->group_size - 1) / rq->group_size) * n * sizeof(uint64_t) : 0;
    BBE_CK(cudaEventSynchronize(ctx->ev1));  // a previous async launch on this ctx has read its params
    BBE_CK(ctx->h_params.ensure(pbytes + tbytes + gbytes));
    BBE_CK(ctx->d_params.ensure(pbytes + tbytes + gbytes));
    BBE_CK(ctx->h_tally.ensure(tbytes));
    pack_params(race, comps, st, (double*)ctx->h_params.p);
    const NativeFrame fr = native_frames(race, comps, st, pl.W);
    pack_params_f32(race, comps, st, (double*)ctx->h_params.p, fr);
    std::memset((char*)ctx->h_params.p + pbytes, 0, tbytes + gbytes);
    uint64_t* const d_tally = (uint64_t*)((char*)ctx->d_params.p + pbytes);
    uint64_t* const d_groups = groups ? d_tally + pl.tally_len : nullptr;
    PROBE(2, "begin: pack");
    BBE_CK(cudaMemcpyAsync(ctx->d_params.p, ctx->h_params.p, pbytes + tbytes + gbytes, cudaMemcpyHostToDevice, s));
    PROBE(3, "begin: H2D api");

    const double* d_draws = nullptr;
    const int64_t* d_offsets = nullptr;
    if (rq->mode == BBE_MODE_INJECT) {
        const int64_t nd = rq->draw_offsets[ns];
        if (rq->draw_offsets[0] != 0 || nd < 0) return fail(BBE_EINVAL, "draw_offsets must start at 0 and be non-decreasing");
        BBE_CK(ctx->d_draws.ensure((size_t)std::max<int64_t>(nd, 1) * sizeof(double)));
        BBE_CK(ctx->d_offsets.ensure((size_t)(ns + 1) * sizeof(int64_t)));
        if (nd) BBE_CK(cudaMemcpyAsync(ctx->d_draws.p, rq->draws, (size_t)nd * sizeof(double), cudaMemcpyHostToDevice, s));
        BBE_CK(cudaMemcpyAsync(ctx->d_offsets.p, rq->draw_offsets, (size_t)(ns + 1) * sizeof(int64_t),
                               cudaMemcpyHostToDevice, s));
        d_draws = (const double*)ctx->d_draws.p;
        d_offsets = (const int64_t*)ctx->d_offsets.p;
    }
    const uint64_t* d_seeds = nullptr;
    if (rq->mode == BBE_MODE_MT && rq->seeds && ns) {
        BBE_CK(ctx->d_seeds.ensure((size_t)ns * sizeof(uint64_t)));
        BBE_CK(cudaMemcpyAsync(ctx->d_seeds.p, rq->seeds, (size_t)ns * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
        d_seeds = (const uint64_t*)ctx->d_seeds.p;
    }


    bbe_result dev{};
    const size_t nsn = (size_t)ns * n;
    if (out->winner) { BBE_CK(ctx->d_winner.ensure(ns * sizeof(int32_t))); dev.winner = (int32_t*)ctx->d_winner.p; }
    if (out->order) { BBE_CK(ctx->d_order.ensure(nsn * sizeof(int32_t))); dev.order = (int32_t*)ctx->d_order.p; }
    if (out->finish_ticks) { BBE_CK(ctx->d_fin.ensure(nsn * sizeof(int64_t))); dev.finish_ticks = (int64_t*)ctx->d_fin.p; }
    if (out->final_positions) { BBE_CK(ctx->d_fpos.ensure(nsn * sizeof(double))); dev.final_positions = (double*)ctx->d_fpos.p; }
    if (out->blocked) { BBE_CK(ctx->d_blocked.ensure(ns * sizeof(int64_t))); dev.blocked = (int64_t*)ctx->d_blocked.p; }
    if (out->draws_used && rq->mode == BBE_MODE_INJECT) {
        BBE_CK(ctx->d_dused.ensure(ns * sizeof(int64_t)));
        dev.draws_used = (int64_t*)ctx->d_dused.p;
    }
    size_t traj_elems = 0;
    if (out->traj_cap > 0 && out->traj_positions && out->traj_prev_steps) {
        if (rq->mode == BBE_MODE_NATIVE || rq->mode == BBE_MODE_NATIVE64)
            return fail(BBE_EINVAL, "trajectories are recorded by the exact modes (mt, inject)");
        traj_elems = (size_t)ns * ((size_t)out->traj_cap + 1) * n;
        BBE_CK(ctx->d_traj.ensure(2 * traj_elems * sizeof(double)));
        dev.traj_positions = (double*)ctx->d_traj.p;
        dev.traj_prev_steps = (double*)ctx->d_traj.p + traj_elems;
        dev.traj_cap = out->traj_cap;
    }

    dev.group_wins = d_groups;
    LaunchArgs a;
    build_args(pl, race, st, rq, (const double*)ctx->d_params.p, d_draws, d_offsets, d_tally, &dev, fr, &a);
    PROBE(4, "begin: outputs+args");
    BBE_CK(cudaEventRecord(ctx->ev0, s));
    PROBE(5, "begin: record ev0");
    if ((rc = launch_all(ctx, pl, a, comps, d_seeds, rq->seed_master, s))) return rc;
    PROBE(6, "begin: launch");
    BBE_CK(cudaEventRecord(ctx->ev1, s));
    PROBE(7, "begin: record ev1");

    BBE_CK(cudaMemcpyAsync(ctx->h_tally.p, d_tally, tbytes, cudaMemcpyDeviceToHost, s));
    PROBE(8, "begin: D2H api");
    // Per-sim outputs go device -> pinned staging asynchronously (a copy into pageable memory would
    // block this call until the kernel ends); _end copies them into the caller's buffers.  Very
    // large outputs (trajectories) are copied directly.
    struct Out { void* dst; const void* src; size_t bytes; };
    std::vector<Out> outs;
    if (ns) {
        if (out->winner) outs.push_back({out->winner, dev.winner, ns * sizeof(int32_t)});
        if (out->order) outs.push_back({out->order, dev.order, nsn * sizeof(int32_t)});
        if (out->finish_ticks) outs.push_back({out->finish_ticks, dev.finish_ticks, nsn * sizeof(int64_t)});
        if (out->final_positions) outs.push_back({out->final_positions, dev.final_positions, nsn * sizeof(double)});
        if (out->blocked) outs.push_back({out->blocked, dev.blocked, ns * sizeof(int64_t)});
        if (dev.draws_used) outs.push_back({out->draws_used, dev.draws_used, ns * sizeof(int64_t)});
        if (groups) outs.push_back({out->group_wins, d_groups, gbytes});
        if (traj_elems) {
            outs.push_back({out->traj_positions, dev.traj_positions, traj_elems * sizeof(double)});
            outs.push_back({out->traj_prev_steps, dev.traj_prev_steps, traj_elems * sizeof(double)});
        }
    }
    size_t staged = 0;
    for (const Out& o : outs) staged += (o.bytes + 255) & ~(size_t)255;
    ctx->pend_copies.clear();
    if (staged && staged <= kMaxStagedBytes) {
        BBE_CK(ctx->h_out.ensure(staged));
        size_t at = 0;
        for (const Out& o : outs) {
            char* h = (char*)ctx->h_out.p + at;
            BBE_CK(cudaMemcpyAsync(h, o.src, o.bytes, cudaMemcpyDeviceToHost, s));
            ctx->pend_copies.push_back({o.dst, h, o.bytes});
            at += (o.bytes + 255) & ~(size_t)255;
        }
    } else {
        for (const Out& o : outs) BBE_CK(cudaMemcpyAsync(o.dst, o.src, o.bytes, cudaMemcpyDeviceToHost, s));
    }
    ctx->pending = true;
    ctx->pend_out = out;
    ctx->pend_n = n;
    ctx->pend_nperm = pl.nperm;
    ctx->pend_K = pl.K;
    ctx->pend_ns = ns;
    ctx->pend_limit = race->tick_limit;
    lease.keep = true;  // in flight until bbe_simulate_end(out)
    return BBE_OK;
}

int bbe_simulate_end(bbe_result* out) {
    NvtxRange nvtx_range("bbe_simulate_end");
    Lease lease;
    {
        std::lock_guard<std::mutex> g(g_ctx_mu);
        for (auto& dev_pool : g_pool)
            for (DevCtx* p : dev_pool)
                if (p->busy && p->pending && p->pend_out == out) lease.c = p;
    }
    if (!lease.c) return fail(BBE_EINVAL, "no call in flight for this result");
    DevCtx* const ctx = lease.c;
    ctx->pending = false;
    PROBE_T0
    BBE_CK(cudaStreamSynchronize(ctx->stream));
    PROBE(9, "end: sync");
    for (const auto& c : ctx->pend_copies) std::memcpy(c.dst, c.src, c.bytes);
    ctx->pend_copies.clear();
    const int n = ctx->pend_n;
    const int64_t ns = ctx->pend_ns;
    struct { int nperm, K; } pl{ctx->pend_nperm, ctx->pend_K};
    const uint64_t* T = (const uint64_t*)ctx->h_tally.p;
    TallyLayout TL{n, pl.nperm};
    std::memcpy(out->wins, T + TL.wins(), n * sizeof(uint64_t));
    if (out->ranks) std::memcpy(out->ranks, T + TL.ranks(), (size_t)n * n * sizeof(uint64_t));
    if (out->perms && pl.nperm) std::memcpy(out->perms, T + TL.perms(), (size_t)pl.nperm * sizeof(uint64_t));
    out->competitor_steps = T[TL.ct()];
    out->blocked_steps = T[TL.blocked()];
    out->first_diverged = decode_first(T[TL.first_div()]);
    out->first_bad_draws = decode_first(T[TL.first_bad()]);
    float ms = 0.f;
    if (ns) cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    out->kernel_ms = ms;
    out->lanes_per_slot = pl.K;
    PROBE(10, "end: copy-out+elapsed");
    if (T[TL.n_div()]) return fail(BBE_EDIVERGED, "race exceeded tick_limit=" + std::to_string(ctx->pend_limit) +
                                                      " in sim " + std::to_string(out->first_diverged));
    if (T[TL.n_bad()]) return fail(BBE_EDRAWS, "injected draw stream under/over-consumed in sim " +
                                                   std::to_string(out->first_bad_draws));
    return BBE_OK;
}

}  // extern "C"

// bbe_rp_predict NATIVE: the staged parameters' H2D, the kernel and the tally D2H as one graph
// launch.  The graph is captured once per (kernel, grid, buffers) and its kernel node's arguments
// are replaced every call (seed, work slot, frame); the copies read and write the same staging.
static int launch_graph(DevCtx* ctx, const Plan& pl, LaunchArgs a, size_t bytes, size_t tbytes, uint64_t* d_tally) {
    cudaStream_t s = ctx->stream;
    int grid = 0;
    int rc = prepare_launch(ctx, pl, s, &a, &grid);
    if (rc) return rc;
    DevCtx::RpGraph& g = ctx->rp_graph;
    const bool same = g.exec && g.fn == (const void*)pl.fn && g.grid == grid && g.smem == pl.smem && g.bytes == bytes &&
                      g.tbytes == tbytes && g.hp == ctx->h_params.p && g.dp == ctx->d_params.p && g.ht == ctx->h_tally.p;
    if (!same) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
        g = DevCtx::RpGraph{};
        cudaGraph_t graph = nullptr;
        BBE_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        cudaMemcpyAsync(ctx->d_params.p, ctx->h_params.p, bytes, cudaMemcpyHostToDevice, s);
        pl.fn<<<grid, kBlockThreads, pl.smem, s>>>(a);
        cudaMemcpyAsync(ctx->h_tally.p, d_tally, tbytes, cudaMemcpyDeviceToHost, s);
        BBE_CK(cudaStreamEndCapture(s, &graph));
        size_t nn = 0;
        BBE_CK(cudaGraphGetNodes(graph, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        BBE_CK(cudaGraphGetNodes(graph, nodes.data(), &nn));
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType t;
            BBE_CK(cudaGraphNodeGetType(nd, &t));
            if (t == cudaGraphNodeTypeKernel) g.knode = nd;
        }
        g.graph = graph;
        BBE_CK(cudaGraphInstantiate(&g.exec, graph, 0));
        if (!g.knode) return fail(BBE_ECUDA, "captured graph has no kernel node");
        g.fn = (const void*)pl.fn;
        g.grid = grid;
        g.smem = pl.smem;
        g.bytes = bytes;
        g.tbytes = tbytes;
        g.hp = ctx->h_params.p;
        g.dp = ctx->d_params.p;
        g.ht = ctx->h_tally.p;
    } else {
        cudaKernelNodeParams kp{};
        void* args[] = {&a};
        kp.func = (void*)pl.fn;
        kp.gridDim = dim3(grid);
        kp.blockDim = dim3(kBlockThreads);
        kp.sharedMemBytes = (unsigned)pl.smem;
        kp.kernelParams = args;
        BBE_CK(cudaGraphExecKernelNodeSetParams(g.exec, g.knode, &kp));
    }
    BBE_CK(cudaGraphLaunch(g.exec, s));
    return BBE_OK;
}

// bbe_rp_predict: one winner-tally launch of rq on ctx's stream -- parameters + zeroed tally H2D,
// the kernel(s), the tally D2H into ctx->h_tally.  d_seeds (MT) must already be on ctx's stream.
static int enqueue_tally(DevCtx* ctx, const bbe_race* race, const bbe_competitor* comps, const bbe_state* st,
                         const bbe_request& rq, const uint64_t* d_seeds, const Plan& pl) {
    cudaStream_t s = ctx->stream;
    const size_t pbytes = (param_bytes(race->n) + 63) & ~(size_t)63;
    const size_t tbytes = (size_t)pl.tally_len * sizeof(uint64_t);
    BBE_CK(cudaEventSynchronize(ctx->ev1));  // a previous async launch on this ctx has read its params
    BBE_CK(ctx->h_params.ensure(pbytes + tbytes));
    BBE_CK(ctx->d_params.ensure(pbytes + tbytes));
    BBE_CK(ctx->h_tally.ensure(tbytes));
    pack_params(race, comps, st, (double*)ctx->h_params.p);
    const NativeFrame fr = native_frames(race, comps, st, pl.W);
    pack_params_f32(race, comps, st, (double*)ctx->h_params.p, fr);
    std::memset((char*)ctx->h_params.p + pbytes, 0, tbytes);
    uint64_t* const d_tally = (uint64_t*)((char*)ctx->d_params.p + pbytes);
    LaunchArgs a;
    build_args(pl, race, st, &rq, (const double*)ctx->d_params.p, nullptr, nullptr, d_tally, nullptr, fr, &a);
    // the graph is kept per context and re-captured when its grid changes, so it is used only for
    // calls that fill the persistent grid (their grid is the same from call to call)
    const int64_t sims_per_block = (int64_t)kWarpsPerBlock * pl.S;
    if ((pl.mode == BBE_MODE_NATIVE || pl.mode == BBE_MODE_NATIVE64) && rq.n_sims <= kMaxLaunchSims &&
        (rq.n_sims + sims_per_block - 1) / sims_per_block >= pl.grid)
        return launch_graph(ctx, pl, a, pbytes + tbytes, tbytes, d_tally);
    BBE_CK(cudaMemcpyAsync(ctx->d_params.p, ctx->h_params.p, pbytes + tbytes, cudaMemcpyHostToDevice, s));
    int rc = launch_all(ctx, pl, a, comps, d_seeds, 0, s);
    if (rc) return rc;
    BBE_CK(cudaMemcpyAsync(ctx->h_tally.p, d_tally, tbytes, cudaMemcpyDeviceToHost, s));
    return BBE_OK;
}

// bbe_rp_predict, MT: draw `count` dry-run seeds from the bettor's stream straight into ctx's pinned
// staging, copy them up and enqueue the seeding + race kernels for sims [off, off + count).
static int enqueue_mt_part(DevCtx* ctx, const bbe_race* race, const bbe_competitor* comps, const bbe_state* st,
                           int64_t off, int64_t count, uint32_t* state624, int32_t* pos, Plan* pl) {
    bbe_request rq{};
    rq.n_sims = count;
    rq.sim_offset = off;
    rq.mode = BBE_MODE_MT;
    int rc = make_plan(ctx, race, comps, st, &rq, 0, pl);
    if (rc) return rc;
    BBE_CK(ctx->h_seeds.ensure((size_t)count * sizeof(uint64_t)));
    BBE_CK(ctx->d_seeds.ensure((size_t)count * sizeof(uint64_t)));
    BBE_CK(cudaEventSynchronize(ctx->ev1));  // the staging's previous contents have been copied
    *pos = (int32_t)bbe_host_mt_getrandbits64(state624, (uint32_t)*pos, count, (uint64_t*)ctx->h_seeds.p, count);
    BBE_CK(cudaMemcpyAsync(ctx->d_seeds.p, ctx->h_seeds.p, (size_t)count * sizeof(uint64_t), cudaMemcpyHostToDevice,
                           ctx->stream));
    return enqueue_tally(ctx, race, comps, st, rq, (const uint64_t*)ctx->d_seeds.p, *pl);
}

// Wait for a bbe_rp_predict launch and add its winner counts into wins[n]; divergence -> error.
static int finish_tally(DevCtx* ctx, const Plan& pl, int n, int64_t limit, uint64_t* wins, int64_t* first_div) {
    BBE_CK(cudaStreamSynchronize(ctx->stream));
    const uint64_t* T = (const uint64_t*)ctx->h_tally.p;
    const TallyLayout TL{n, pl.nperm};
    for (int c = 0; c < n; ++c) wins[c] += T[TL.wins() + c];
    if (T[TL.n_div()]) {
        const int64_t fd = decode_first(T[TL.first_div()]);
        if (first_div && (*first_div < 0 || fd < *first_div)) *first_div = fd;
        return fail(BBE_EDIVERGED, "race exceeded tick_limit=" + std::to_string(limit) + " in sim " + std::to_string(fd));
    }
    return BBE_OK;
}

// The entry points that write a CPython random.Random in place (bbe_rp_predict, bbe_mt_advance64*)
// are bound through ctypes.PyDLL, so they run with the GIL held and no other Python thread can touch
// the generator mid-write.  bbe_rp_predict then drops the GIL for its GPU wait, once every write to
// the generator is done (and takes it back before returning).  The CPython symbols are looked up in
// the running process; in a process without Python, or a caller without the GIL, nothing happens.
class GilRelease {
  public:
    void release() {
        const Fns& f = fns();
        if (!ts_ && f.check && f.save && f.restore && f.check()) ts_ = f.save();
    }
    void reacquire() {
        if (ts_) fns().restore(ts_);
        ts_ = nullptr;
    }
    ~GilRelease() { reacquire(); }

  private:
    struct Fns {
        int (*check)() = nullptr;
        void* (*save)() = nullptr;
        void (*restore)(void*) = nullptr;
    };
    static const Fns& fns() {
        static const Fns f = [] {
            Fns g;
            g.check = (int (*)())dlsym(RTLD_DEFAULT, "PyGILState_Check");
            g.save = (void* (*)())dlsym(RTLD_DEFAULT, "PyEval_SaveThread");
            g.restore = (void (*)(void*))dlsym(RTLD_DEFAULT, "PyEval_RestoreThread");
            return g;
        }();
        return f;
    }
    void* ts_ = nullptr;
};

// On a diverged dry run the reference has drawn only the seeds up to and including the failing one
// (agents.py:164 raises inside that simulate_from): put the bettor's stream back there.
static void rewind_stream(const uint32_t* saved624, int32_t saved_pos, int64_t first_div, uint32_t* state624,
                          int32_t* pos) {
    if (first_div < 0) return;
    std::memcpy(state624, saved624, 624 * sizeof(uint32_t));
    *pos = (int32_t)bbe_host_mt_getrandbits64(state624, (uint32_t)saved_pos, first_div + 1, nullptr, 0);
}

// ---- NCCL (single process, every visible GPU): the tally all-reduce of bbe_simulate_multi ----
// NCCL is dlopen'ed (RTLD_NOLOAD first: a process running torch already holds its libnccl, and one
// process must not load two).  Types come from nccl.h; nothing links against libnccl.
struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclCommInitAll) init = nullptr;
    decltype(&ncclAllReduce) allreduce = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error = nullptr;
};

static const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return a;
        }
        a.init = (decltype(a.init))dlsym(h, "ncclCommInitAll");
        a.allreduce = (decltype(a.allreduce))dlsym(h, "ncclAllReduce");
        a.group_start = (decltype(a.group_start))dlsym(h, "ncclGroupStart");
        a.group_end = (decltype(a.group_end))dlsym(h, "ncclGroupEnd");
        a.error = (decltype(a.error))dlsym(h, "ncclGetErrorString");
        a.ok = a.init && a.allreduce && a.group_start && a.group_end && a.error;
        if (!a.ok) a.why = "libnccl.so.2 lacks the collective entry points";
        return a;
    }();
    return api;
}

// One communicator clique per device count (devices 0..k-1), created once and kept for the process
// (not destroyed at exit: ncclCommDestroy from a static destructor would race the CUDA runtime's own
// teardown; the driver reclaims the resources with the process).
static std::mutex g_nccl_mu;
static std::map<int, std::vector<ncclComm_t>> g_nccl_comms;

static int nccl_comms(int k, std::vector<ncclComm_t>** out) {
    const NcclApi& api = nccl_api();
    if (!api.ok) return fail(BBE_ENCCL, api.why);
    std::lock_guard<std::mutex> g(g_nccl_mu);
    auto it = g_nccl_comms.find(k);
    if (it == g_nccl_comms.end()) {
        std::vector<ncclComm_t> comms(k);
        std::vector<int> devs(k);
        for (int i = 0; i < k; ++i) devs[i] = i;
        const ncclResult_t r = api.init(comms.data(), k, devs.data());
        if (r != ncclSuccess) return fail(BBE_ENCCL, std::string("ncclCommInitAll: ") + api.error(r));
        it = g_nccl_comms.emplace(k, std::move(comms)).first;
    }
    *out = &it->second;
    return BBE_OK;
}

// Per-device state of a tally-only multi-GPU call: the device tally every part on that device adds
// into, its stream, and events around the device's work.
struct MultiDev {
    cudaStream_t s = nullptr;
    uint64_t* d_tally = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int rc = BBE_OK;
    std::string err;
};

extern "C" {

int bbe_rp_predict(const bbe_race* race, const bbe_competitor* comps, const bbe_state* st, int64_t d, int32_t mode,
                   uint32_t* state624, int32_t* pos, uint64_t* wins, int64_t* first_diverged) {
    NvtxRange nvtx_range("bbe_rp_predict");
    if (!state624 || !pos || !wins || *pos < 0 || *pos > 624 || d < 0) return fail(BBE_EINVAL, "bad arguments");
    if (mode != BBE_MODE_NATIVE && mode != BBE_MODE_NATIVE64 && mode != BBE_MODE_MT)
        return fail(BBE_EINVAL, "rp_predict modes: native, native64, mt");
    bbe_request rq{};
    rq.n_sims = d;
    rq.mode = mode;
    int rc = validate(race, comps, st, &rq);
    if (rc) return rc;
    const int n = race->n;
    std::fill(wins, wins + n, 0ull);
    if (first_diverged) *first_diverged = -1;
    if (d == 0) return BBE_OK;
    Lease lease;
    if ((rc = acquire_ctx(lease))) return rc;
    DevCtx* const ctx = lease.c;
    uint32_t saved[624];
    std::memcpy(saved, state624, sizeof(saved));
    const int32_t saved_pos = *pos;
    int64_t fd_local = -1;
    int64_t* const fd = first_diverged ? first_diverged : &fd_local;
    GilRelease gil;
    if (mode == BBE_MODE_NATIVE || mode == BBE_MODE_NATIVE64) {
        // the first dry-run seed keys the Philox stream; the other d-1 draws advance the bettor's
        // stream on the host while the kernel runs
        uint64_t key = 0;
        *pos = (int32_t)bbe_host_mt_getrandbits64(state624, (uint32_t)*pos, 1, &key, 1);
        rq.seed = key;
        Plan pl;
        if ((rc = make_plan(ctx, race, comps, st, &rq, 0, &pl))) return rc;
        if ((rc = enqueue_tally(ctx, race, comps, st, rq, nullptr, pl))) return rc;
        *pos = (int32_t)bbe_host_mt_getrandbits64(state624, (uint32_t)*pos, d - 1, nullptr, 0);
        gil.release();
        rc = finish_tally(ctx, pl, n, race->tick_limit, wins, fd);
        gil.reacquire();
        if (rc == BBE_EDIVERGED) rewind_stream(saved, saved_pos, *fd, state624, pos);
        return rc;
    }
    // MT: every dry run replays random.Random(getrandbits(64)).  Large calls run as P parts on P
    // streams (P = d / kRpSplitMin, at most BBE_RP_PARTS): the host draws part p+1's seeds while the
    // GPU runs part p, and each launch fills the previous one's tail.
    const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(BBE_RP_PARTS, d / kRpSplitMin));
    Lease extra[BBE_RP_PARTS];
    DevCtx* cx[BBE_RP_PARTS];
    Plan pp[BBE_RP_PARTS];
    int rcs[BBE_RP_PARTS];
    cx[0] = ctx;
    int enq = 0;  // parts enqueued
    for (int p = 0; p < parts; ++p) {
        if (p > 0 && (rc = acquire_ctx(extra[p]))) break;
        if (p > 0) cx[p] = extra[p].c;
        // part boundaries: the first part is BBE_RP_FIRST % of d (its seeds are the only ones drawn
        // before the GPU starts), the rest is split evenly
        auto cut = [&](int q) -> int64_t {
            if (q == 0) return 0;
            if (q == parts) return d;
            const int64_t first = d * BBE_RP_FIRST / 100;
            return parts == 1 ? d : first + (d - first) * (q - 1) / (parts - 1);
        };
        const int64_t a0 = cut(p), a1 = cut(p + 1);
        if ((rc = enqueue_mt_part(cx[p], race, comps, st, a0, a1 - a0, state624, pos, &pp[p]))) break;
        enq = p + 1;
    }
    gil.release();  // every seed has been drawn
    int first_rc = BBE_OK;
    for (int p = 0; p < enq; ++p) {
        rcs[p] = finish_tally(cx[p], pp[p], n, race->tick_limit, wins, fd);
        if (rcs[p] && !first_rc) first_rc = rcs[p];
    }
    gil.reacquire();
    if (!rc && first_rc == BBE_EDIVERGED) rewind_stream(saved, saved_pos, *fd, state624, pos);
    return rc ? rc : first_rc;
}

int bbe_simulate(const bbe_race* race, const bbe_competitor* comps, const bbe_state* st, const bbe_request* rq,
                 bbe_result* out) {
    const int rc = bbe_simulate_begin(race, comps, st, rq, out);
    return rc ? rc : bbe_simulate_end(out);
}

int bbe_simulate_multi(int32_t n_parts, const bbe_race* race, const bbe_competitor* comps, const bbe_state* st,
                       const bbe_request* rq, bbe_result* out) {
    NvtxRange nvtx_range("bbe_simulate_multi");
    int rc = validate(race, comps, st, rq);
    if (rc) return rc;
    if (!out || !out->wins) return fail(BBE_EINVAL, "result needs a wins buffer");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(BBE_ENODEV, "no CUDA device");
    }
    if (n_parts <= 0) n_parts = ndev;
    const int n = race->n;
    const int64_t N = rq->n_sims;
    const int nperm = out->perms ? nperm_for(n) : 0;
    if (rq->mode == BBE_MODE_INJECT && (!rq->draw_offsets || rq->draw_offsets[0] != 0))
        return fail(BBE_EINVAL, "draw_offsets must start at 0 and be non-decreasing");
    struct Part {
        bbe_request rq;
        bbe_result res;
        std::vector<uint64_t> wins, ranks, perms;
        std::vector<int64_t> offsets;  // INJECT: rebased CSR offsets of the shard
        int rc = BBE_OK;
        std::string err;
    };
    std::vector<Part> parts(n_parts);
    const int traj_stride = out->traj_cap > 0 ? (out->traj_cap + 1) * n : 0;
    for (int p = 0; p < n_parts; ++p) {
        Part& P = parts[p];
        // shard_range (parallel.py); with per-group winners, shard edges fall on group edges
        const int64_t g = (rq->group_size > 0 && out->group_wins) ? rq->group_size : 1;
        const int64_t ng = (N + g - 1) / g;
        const int64_t a = std::min(N, ng * p / n_parts * g), b = std::min(N, ng * (p + 1) / n_parts * g);
        P.rq = *rq;
        P.rq.n_sims = b - a;
        P.rq.sim_offset = rq->sim_offset + a;
        if (rq->seeds) P.rq.seeds = rq->seeds + a;
        if (rq->mode == BBE_MODE_INJECT) {
            const int64_t base = rq->draw_offsets[a];
            P.offsets.resize(b - a + 1);
            for (int64_t i = 0; i <= b - a; ++i) P.offsets[i] = rq->draw_offsets[a + i] - base;
            P.rq.draws = rq->draws + base;
            P.rq.draw_offsets = P.offsets.data();
        }
        P.wins.assign(n, 0);
        if (out->ranks) P.ranks.assign((size_t)n * n, 0);
        if (nperm) P.perms.assign(nperm, 0);
        P.res = *out;
        P.res.wins = P.wins.data();
        P.res.ranks = out->ranks ? P.ranks.data() : nullptr;
        P.res.perms = nperm ? P.perms.data() : nullptr;
        if (out->group_wins && rq->group_size > 0) P.res.group_wins = out->group_wins + (a / g) * n;
        if (out->winner) P.res.winner = out->winner + a;
        if (out->order) P.res.order = out->order + a * n;
        if (out->finish_ticks) P.res.finish_ticks = out->finish_ticks + a * n;
        if (out->final_positions) P.res.final_positions = out->final_positions + a * n;
        if (out->blocked) P.res.blocked = out->blocked + a;
        if (out->draws_used) P.res.draws_used = out->draws_used + a;
        if (traj_stride) {
            P.res.traj_positions = out->traj_positions + a * traj_stride;
            P.res.traj_prev_steps = out->traj_prev_steps + a * traj_stride;
        }
    }
    // Tally-only requests (no per-sim outputs; NATIVE, NATIVE64, or MT with device-derived run seeds):
    // every device adds its parts
    // into one device tally on its own stream, then ONE grouped NCCL all-reduce (SUM over the counters,
    // MAX over the two complement-encoded "first failing sim" fields, fused by ncclGroupStart/End)
    // combines them over NVLink; device 0's tally is the only D2H copy.
    const bool tally_only = !out->winner && !out->order && !out->finish_ticks && !out->final_positions &&
                            !out->blocked && !out->draws_used && !out->traj_positions && !out->group_wins &&
                            rq->mode != BBE_MODE_INJECT && !(rq->mode == BBE_MODE_MT && rq->seeds);
    if (tally_only) {
        const int used = std::min(ndev, n_parts);
        const TallyLayout T{n, nperm_for(n)};
        const int64_t tl = T.len();
        std::vector<MultiDev> md(used);
        auto run_dev = [&](int d) {
            MultiDev& M = md[d];
            auto ok = [&](cudaError_t e, const char* what) {
                if (e != cudaSuccess && M.rc == BBE_OK) {
                    M.rc = BBE_ECUDA;
                    M.err = std::string(what) + ": " + cudaGetErrorString(e);
                }
                return e == cudaSuccess;
            };
            if (!ok(cudaSetDevice(d), "cudaSetDevice") ||
                !ok(cudaStreamCreateWithFlags(&M.s, cudaStreamNonBlocking), "cudaStreamCreate") ||
                !ok(cudaEventCreate(&M.e0), "cudaEventCreate") || !ok(cudaEventCreate(&M.e1), "cudaEventCreate") ||
                !ok(cudaMallocAsync((void**)&M.d_tally, tl * sizeof(uint64_t), M.s), "cudaMallocAsync") ||
                !ok(cudaMemsetAsync(M.d_tally, 0, tl * sizeof(uint64_t), M.s), "cudaMemsetAsync") ||
                !ok(cudaEventRecord(M.e0, M.s), "cudaEventRecord"))
                return;
            for (int p = d; p < n_parts; p += ndev) {
                if (parts[p].rq.n_sims == 0) continue;
                const int r = bbe_simulate_async(race, comps, st, &parts[p].rq, nullptr, M.d_tally, M.s);
                if (r != BBE_OK) {
                    M.rc = r;
                    M.err = bbe_last_error();
                    return;
                }
            }
            ok(cudaEventRecord(M.e1, M.s), "cudaEventRecord");
        };
        int caller = 0;
        cudaGetDevice(&caller);
        {
            std::vector<std::thread> th;
            for (int d = 1; d < used; ++d) th.emplace_back(run_dev, d);
            run_dev(0);
            for (auto& t : th) t.join();
        }
        int rc2 = BBE_OK;
        std::string err2;
        for (const MultiDev& M : md)
            if (M.rc != BBE_OK && rc2 == BBE_OK) { rc2 = M.rc; err2 = M.err; }
        if (rc2 == BBE_OK && used > 1) {
            std::vector<ncclComm_t>* comms = nullptr;
            if ((rc2 = nccl_comms(used, &comms)) != BBE_OK) {
                err2 = g_err;
            } else {
                const NcclApi& api = nccl_api();
                const int64_t nsum = T.ct() + 4;  // wins, ranks, perms, ct, blocked, n_div, n_bad
                api.group_start();
                for (int d = 0; d < used; ++d) {
                    api.allreduce(md[d].d_tally, md[d].d_tally, nsum, ncclUint64, ncclSum, (*comms)[d], md[d].s);
                    api.allreduce(md[d].d_tally + nsum, md[d].d_tally + nsum, 2, ncclUint64, ncclMax, (*comms)[d], md[d].s);
                }
                const ncclResult_t r = api.group_end();
                if (r != ncclSuccess) { rc2 = BBE_ENCCL; err2 = std::string("ncclAllReduce: ") + api.error(r); }
            }
        }
        std::vector<uint64_t> h(tl, 0);
        float kms = 0.f;
        if (rc2 == BBE_OK) {
            cudaSetDevice(0);
            cudaError_t e = cudaMemcpyAsync(h.data(), md[0].d_tally, tl * sizeof(uint64_t), cudaMemcpyDeviceToHost, md[0].s);
            for (int d = 0; d < used && e == cudaSuccess; ++d) {
                cudaSetDevice(d);
                e = cudaStreamSynchronize(md[d].s);
                float ms = 0.f;
                if (e == cudaSuccess && cudaEventElapsedTime(&ms, md[d].e0, md[d].e1) == cudaSuccess) kms = std::max(kms, ms);
            }
            if (e != cudaSuccess) { rc2 = BBE_ECUDA; err2 = std::string("multi-GPU tally: ") + cudaGetErrorString(e); }
        }
        for (int d = 0; d < used; ++d) {  // release (after a failure too)
            cudaSetDevice(d);
            if (md[d].s) cudaStreamSynchronize(md[d].s);
            if (md[d].d_tally) cudaFree(md[d].d_tally);
            if (md[d].s) cudaStreamDestroy(md[d].s);
            if (md[d].e0) cudaEventDestroy(md[d].e0);
            if (md[d].e1) cudaEventDestroy(md[d].e1);
        }
        cudaGetLastError();
        cudaSetDevice(caller);
        if (rc2 != BBE_OK) return fail(rc2, err2);
        std::copy(h.begin(), h.begin() + n, out->wins);
        if (out->ranks) std::copy(h.begin() + T.ranks(), h.begin() + T.ranks() + (size_t)n * n, out->ranks);
        if (nperm) std::copy(h.begin() + T.perms(), h.begin() + T.perms() + nperm, out->perms);
        out->competitor_steps = h[T.ct()];
        out->blocked_steps = h[T.ct() + 1];
        auto first = [](uint64_t v) -> int64_t { return v == 0 ? -1 : (int64_t)(0x7fffffffffffffffull - v); };
        out->first_diverged = first(h[T.ct() + 4]);
        out->first_bad_draws = first(h[T.ct() + 5]);
        out->kernel_ms = kms;
        out->lanes_per_slot = 0;
        if (h[T.ct() + 2])
            return fail(BBE_EDIVERGED, "race exceeded tick_limit=" + std::to_string(race->tick_limit) + " in sim " +
                                           std::to_string(out->first_diverged));
        if (h[T.ct() + 3])
            return fail(BBE_EDRAWS, "draw stream under/over-consumed in sim " + std::to_string(out->first_bad_draws));
        return BBE_OK;
    }
    // per-sim outputs (or host-memory draws / seeds): one host thread per device; a
    // device's parts run in order on that thread, each with its own host outputs, merged below
    auto run_device = [&](int d) {
        if (cudaSetDevice(d) != cudaSuccess) {
            cudaGetLastError();
            for (int p = d; p < n_parts; p += ndev) { parts[p].rc = BBE_ECUDA; parts[p].err = "cudaSetDevice failed"; }
            return;
        }
        for (int p = d; p < n_parts; p += ndev) {
            parts[p].rc = bbe_simulate(race, comps, st, &parts[p].rq, &parts[p].res);
            if (parts[p].rc != BBE_OK) parts[p].err = bbe_last_error();
        }
    };
    int caller_dev = 0;
    cudaGetDevice(&caller_dev);
    std::vector<std::thread> threads;
    for (int d = 1; d < std::min(ndev, n_parts); ++d) threads.emplace_back(run_device, d);
    run_device(0);
    for (auto& t : threads) t.join();
    cudaSetDevice(caller_dev);
    // merge (parallel.py reduce_tally on the host)
    std::fill(out->wins, out->wins + n, 0ull);
    if (out->ranks) std::fill(out->ranks, out->ranks + (size_t)n * n, 0ull);
    if (nperm) std::fill(out->perms, out->perms + nperm, 0ull);
    out->competitor_steps = out->blocked_steps = 0;
    out->first_diverged = out->first_bad_draws = -1;
    out->kernel_ms = 0.f;
    int worst = BBE_OK;
    std::string worst_err;
    for (const Part& P : parts) {
        if (P.rc != BBE_OK && P.rc != BBE_EDIVERGED && P.rc != BBE_EDRAWS) {
            if (worst == BBE_OK || worst == BBE_EDIVERGED || worst == BBE_EDRAWS) { worst = P.rc; worst_err = P.err; }
            continue;
        }
        for (int c = 0; c < n; ++c) out->wins[c] += P.wins[c];
        if (out->ranks) for (size_t i = 0; i < (size_t)n * n; ++i) out->ranks[i] += P.ranks[i];
        if (nperm) for (int i = 0; i < nperm; ++i) out->perms[i] += P.perms[i];
        out->competitor_steps += P.res.competitor_steps;
        out->blocked_steps += P.res.blocked_steps;
        auto keep_min = [](int64_t& acc, int64_t v) { if (v >= 0 && (acc < 0 || v < acc)) acc = v; };
        keep_min(out->first_diverged, P.res.first_diverged);
        keep_min(out->first_bad_draws, P.res.first_bad_draws);
        out->kernel_ms = std::max(out->kernel_ms, P.res.kernel_ms);
        out->lanes_per_slot = P.res.lanes_per_slot;
    }
    if (worst != BBE_OK) return fail(worst, worst_err);
    if (out->first_diverged >= 0)
        return fail(BBE_EDIVERGED, "race exceeded tick_limit=" + std::to_string(race->tick_limit) + " in sim " +
                                       std::to_string(out->first_diverged));
    if (out->first_bad_draws >= 0)
        return fail(BBE_EDRAWS, "injected draw stream under/over-consumed in sim " + std::to_string(out->first_bad_draws));
    return BBE_OK;
}

int bbe_simulate_async(const bbe_race* race, const bbe_competitor* comps, const bbe_state* st, const bbe_request* rq,
                       const bbe_result* dev_out, uint64_t* d_tally, void* stream) {
    NvtxRange nvtx_range("bbe_simulate_async");
    int rc = validate(race, comps, st, rq);
    if (rc) return rc;
    if (!d_tally) return fail(BBE_EINVAL, "d_tally is required");
    Lease lease;
    if ((rc = acquire_ctx(lease))) return rc;
    DevCtx* const ctx = lease.c;
    Plan pl;
    const bool perms = nperm_for(race->n) > 0;
    if ((rc = make_plan(ctx, race, comps, st, rq, perms, &pl))) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // NULL = legacy default stream (torch's default)
    // parameters: staged through pinned memory; the copy is ordered on `s` before the kernel, and
    // the staging block is not reused until that copy has been consumed (sync on an event).
    const size_t pbytes = param_bytes(race->n);
    BBE_CK(ctx->h_params.ensure(pbytes));
    BBE_CK(ctx->d_params.ensure(pbytes));
    BBE_CK(cudaEventSynchronize(ctx->ev1));  // previous async launch on this ctx has read its params
    pack_params(race, comps, st, (double*)ctx->h_params.p);
    const NativeFrame fr = native_frames(race, comps, st, pl.W);
    pack_params_f32(race, comps, st, (double*)ctx->h_params.p, fr);
    BBE_CK(cudaMemcpyAsync(ctx->d_params.p, ctx->h_params.p, pbytes, cudaMemcpyHostToDevice, s));
    LaunchArgs a;
    build_args(pl, race, st, rq, (const double*)ctx->d_params.p, rq->draws, rq->draw_offsets, d_tally, dev_out, fr,
               &a);
    BBE_CK(cudaEventRecord(ctx->ev0, s));
    if ((rc = launch_all(ctx, pl, a, comps, rq->seeds, rq->seed_master, s))) return rc;
    BBE_CK(cudaEventRecord(ctx->ev1, s));
    return BBE_OK;
}

// ---- prepared races (device-resident parameters) ----
}  // extern "C"

struct bbe_prepared {
    int dev = -1;
    Plan pl{};
    bbe_race race{};
    int64_t tick = 0;
    int32_t from_start = 0;
    NativeFrame fr{};
    double* d_params = nullptr;
    unsigned long long* d_work = nullptr;
    int work_slot = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool timed = false;
};

static void free_prepared(bbe_prepared* p) {
    if (!p) return;
    if (p->d_params) cudaFree(p->d_params);
    if (p->d_work) cudaFree(p->d_work);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    delete p;
}

extern "C" {

int bbe_prepare(const bbe_race* race, const bbe_competitor* comps, const bbe_state* st, int32_t mode,
                int32_t lanes_per_slot_hint, bbe_prepared** out) {
    NvtxRange nvtx_range("bbe_prepare");
    if (!out) return fail(BBE_EINVAL, "out is NULL");
    *out = nullptr;
    bbe_request rq{};
    rq.n_sims = INT64_MAX / 2;  // plan for a full persistent grid; each launch trims it
    if (mode != BBE_MODE_NATIVE && mode != BBE_MODE_NATIVE64) return fail(BBE_EINVAL, "prepared races: native, native64");
    rq.mode = mode;
    rq.lanes_per_slot_hint = lanes_per_slot_hint;
    int rc = validate(race, comps, st, &rq);
    if (rc) return rc;
    Lease lease;
    if ((rc = acquire_ctx(lease))) return rc;
    bbe_prepared* p = new bbe_prepared();
    p->dev = lease.c->dev;
    // the device tally has bbe_tally_len(n) entries: full-order bins for n <= 6 (as bbe_simulate_async)
    if ((rc = make_plan(lease.c, race, comps, st, &rq, nperm_for(race->n) > 0, &p->pl))) {
        free_prepared(p);
        return rc;
    }
    p->race = *race;
    p->tick = st->from_start ? 0 : st->tick;
    p->from_start = st->from_start;
    p->fr = native_frames(race, comps, st, p->pl.W);
    const size_t pbytes = param_bytes(race->n);
    std::vector<double> h(pbytes / sizeof(double) + 1);
    pack_params(race, comps, st, h.data());
    pack_params_f32(race, comps, st, h.data(), p->fr);
    cudaError_t e = cudaMalloc(&p->d_params, pbytes);
    if (e == cudaSuccess) e = cudaMemcpy(p->d_params, h.data(), pbytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_work, kWorkSlots * 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(p->d_work, 0, kWorkSlots * 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaEventCreate(&p->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&p->ev1);
    if (e != cudaSuccess) {
        free_prepared(p);
        return fail(BBE_ECUDA, std::string("bbe_prepare: ") + cudaGetErrorString(e));
    }
    *out = p;
    return BBE_OK;
}

int bbe_launch_prepared(bbe_prepared* p, int64_t n_sims, int64_t sim_offset, uint64_t seed, uint64_t* d_tally,
                        void* stream) {
    if (!p || !d_tally || n_sims < 0 || sim_offset < 0) return fail(BBE_EINVAL, "bad arguments");
    int dev = -1;
    BBE_CK(cudaGetDevice(&dev));
    if (dev != p->dev) return fail(BBE_EINVAL, "prepared on device " + std::to_string(p->dev) + ", current device " +
                                                std::to_string(dev));
    cudaStream_t s = (cudaStream_t)stream;
    bbe_request rq{};
    rq.n_sims = n_sims;
    rq.sim_offset = sim_offset;
    rq.seed = seed;
    rq.mode = p->pl.mode;
    bbe_state st{};
    st.tick = p->tick;
    st.from_start = p->from_start;
    LaunchArgs a0;
    build_args(p->pl, &p->race, &st, &rq, p->d_params, nullptr, nullptr, d_tally, nullptr, p->fr, &a0);
    BBE_CK(cudaEventRecord(p->ev0, s));
    for (int64_t c0 = 0; c0 < n_sims; c0 += kMaxLaunchSims) {
        LaunchArgs a = sub_launch(a0, c0, std::min(kMaxLaunchSims, n_sims - c0));
        a.work = p->d_work + 2 * p->work_slot;
        p->work_slot = (p->work_slot + 1) % kWorkSlots;
        const int64_t spb = (int64_t)kWarpsPerBlock * p->pl.S;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(p->pl.grid, (a.n_sims + spb - 1) / spb));
        p->pl.fn<<<grid, kBlockThreads, p->pl.smem, s>>>(a);
        BBE_CK(cudaGetLastError());
    }
    BBE_CK(cudaEventRecord(p->ev1, s));
    p->timed = n_sims > 0;
    return BBE_OK;
}

float bbe_prepared_kernel_ms(bbe_prepared* p) {
    if (!p || !p->timed || cudaEventSynchronize(p->ev1) != cudaSuccess) return -1.f;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p->ev0, p->ev1) != cudaSuccess) {
        cudaGetLastError();
        return -1.f;
    }
    return ms;
}

void bbe_release_prepared(bbe_prepared* p) { free_prepared(p); }

int bbe_mt_exp_exact(void) { return libm_exp_table().ok ? 1 : 0; }

}  // extern "C"
