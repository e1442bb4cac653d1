/*
 * bbe_sim.h -- C-ABI of the B200-native batched Monte Carlo race simulator.
 *
 * This is the drop-in boundary for the Bristol Betting Exchange dry-run hot path.  The reference
 * (racemarket, pure Python) has no FFI layer; each entry point below replaces a group of reference
 * functions, cited as /root/reference/pkg/src/racemarket/<file>:<line>:
 *
 *   bbe_simulate          race.py:393-406  simulate_from(state, config, seed)      (batched over sims)
 *                         race.py:373-390  run_race(config, seed, record=False)    (from_start = 1)
 *                         agents.py:153-166 rp_predict(state, config, d, rng)      (wins -> (w+1)/(d+n))
 *                         batch.py:110-124 run_batch(BatchConfig)                  (per-sim outputs)
 *                         batch.py:149-170 estimate_pmf / pmf_from_results         (perms tally, n <= 6)
 *   bbe_simulate_multi    the same over several GPUs (one host thread per device; tally-only requests
 *                         combined by one grouped NCCL all-reduce, per-sim outputs host-merged):
 *                         run_batch(BatchConfig(workers=N)), batch.py:120-124.
 *   bbe_simulate_async    the same, device-resident: tallies accumulate into a device buffer on a
 *                         caller stream (used by the multi-GPU path before one NCCL all-reduce).
 *   bbe_rp_predict        agents.py:153-166 rp_predict(state, config, d, rng) in one call: the d
 *                         getrandbits(64) dry-run seeds drawn from the bettor's own MT19937 state
 *                         (advanced in place), the d continuations, the winner counts.
 *   bbe_prepare / bbe_launch_prepared   bbe_simulate_async for one race state launched many times
 *                         (parameters uploaded once).
 *   bbe_derive_seeds      seeding.py:50-59 derive_seed(master, "run", i) for a range of i.
 *   bbe_last_error        -- (error text for the Python exceptions of race.py:27-32, batch.py:30-38)
 *
 * All types are plain C; no torch or CUDA types appear.  Host pointers are caller-owned and only
 * touched during the call.  Calls are thread-safe: concurrent calls on one device each lease their
 * own context (stream + staging buffers) from a per-device pool.  The caller must not let another
 * thread use the same generator state (bbe_rp_predict, bbe_mt_advance64*) during a call; from
 * Python, bind those through ctypes.PyDLL (the GIL then excludes every other thread).
 *
 * Return codes: BBE_OK, BBE_EINVAL (-> RaceConfigError), BBE_EDIVERGED (-> RaceDivergedError /
 * BatchRunError(first_diverged)), BBE_EDRAWS (inject stream under/over-consumed), BBE_ECUDA,
 * BBE_ENODEV, BBE_ENCCL (the multi-GPU tally all-reduce failed, or libnccl is not loadable).
 */
#ifndef BBE_SIM_H
#define BBE_SIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BBE_ABI_VERSION 5 /* 3: bbe_rp_predict; 4: prepared races; 5: BBE_MODE_NATIVE64, bbe_prepare(mode) */
#define BBE_MAX_COMPETITORS 128
#define BBE_MAX_PERM_COMPETITORS 6 /* batch.py:27 MAX_FULL_OUTCOME_COMPETITORS */

enum {
    BBE_OK = 0,
    BBE_EINVAL = 1,
    BBE_EDIVERGED = 2,
    BBE_EDRAWS = 3,
    BBE_ECUDA = 4,
    BBE_ENODEV = 5,
    BBE_ENCCL = 6
};

/* Random-draw source. */
enum {
    BBE_MODE_NATIVE = 0, /* in-register Philox4x32-10, FP32 race state: statistically equivalent */
    BBE_MODE_INJECT = 1, /* recorded reference draws (CSR), FP64 state: bit-exact to the reference */
    BBE_MODE_MT = 2,     /* CPython MT19937 from per-sim seeds, FP64 state: bit-exact from seeds */
    BBE_MODE_NATIVE64 = 3 /* in-register Philox4x32-10, FP64 state and the reference's FP64 operations:
                             statistically equivalent (only the word generator differs), 53-bit draws */
};

enum { BBE_FAMILY_UNIFORM = 0, BBE_FAMILY_LOGNORMAL = 1 };

/* race.py:158-189 (RaceConfig); dt, conditions and betting_close do not enter a step. */
typedef struct {
    double track_length;
    int64_t tick_limit; /* race.py:165; run_race checks it absolutely, simulate_from relatively */
    int32_t n;          /* competitors, 1..BBE_MAX_COMPETITORS */
    int32_t _pad;
} bbe_race;

/* race.py:35-116 (UniformSteps / LogNormalSteps / Responsiveness / Competitor), with the two
 * per-competitor constants the reference recomputes every step hoisted by the host in double:
 *   pref_factor = preference_factor(conditions, preference, pref_sensitivity)   race.py:192-199
 *   bp_abs      = breakpoint * track_length                                      race.py:94      */
typedef struct {
    int32_t family; /* BBE_FAMILY_* */
    int32_t _pad;
    double lo, hi;            /* uniform */
    double mu, sigma, scale;  /* lognormal: scale * exp(N(mu, sigma)) */
    double pref_factor;
    double theta;             /* blocking threshold */
    double early_mult, late_mult, bp_abs;
} bbe_competitor;

/* race.py:207-230 (RaceState).  Ignored when from_start != 0 (run_race: positions 0, previous
 * steps primed by one free draw each, race.py:233-241). */
typedef struct {
    int64_t tick;
    const double* positions;     /* [n] */
    const double* prev_steps;    /* [n] */
    const int64_t* finish_ticks; /* [n], -1 = still racing (None) */
    int32_t from_start;
    int32_t _pad;
} bbe_state;

typedef struct {
    int64_t n_sims;
    int64_t sim_offset;   /* global index of this call's first sim (multi-GPU sharding) */
    uint64_t seed;        /* NATIVE: Philox key */
    int32_t mode;         /* BBE_MODE_* */
    int32_t lanes_per_slot_hint; /* 0 = auto; else competitors per lane K (tuning) */
    /* INJECT: draws of sim s are draws[draw_offsets[s] .. draw_offsets[s+1]) in consumption order */
    const double* draws;
    const int64_t* draw_offsets; /* [n_sims + 1] */
    /* MT: per-sim CPython seeds (e.g. rp_predict's getrandbits(64) stream); NULL -> derive_seed(
     * seed_master, "run", sim_offset + s) as run_batch does */
    const uint64_t* seeds;
    uint64_t seed_master;
    /* > 0: also count winners per group of group_size consecutive sims (the dry runs of one bettor
     * in a batched dispatch) into bbe_result.group_wins */
    int64_t group_size;
} bbe_request;

/* Outputs.  Tally pointers (host for bbe_simulate) may be NULL except wins. */
typedef struct {
    uint64_t* wins;          /* [n]   winner counts (rp_predict tally) */
    uint64_t* ranks;         /* [n*n] ranks[c*n + r] = sims where competitor c finished at rank r */
    uint64_t* perms;         /* [n!]  full finish-order histogram by Lehmer index (n <= 6) */
    int32_t* winner;         /* [n_sims] */
    int32_t* order;          /* [n_sims*n] finish order (competitor indices) */
    int64_t* finish_ticks;   /* [n_sims*n] */
    double* final_positions; /* [n_sims*n] (FP32 state widened in NATIVE mode) */
    int64_t* blocked;        /* [n_sims] blocked steps per sim */
    int64_t* draws_used;     /* [n_sims] (INJECT / MT) */
    uint64_t competitor_steps; /* total racing competitor-timesteps (ct) */
    uint64_t blocked_steps;
    int64_t first_diverged;  /* global sim index of the first diverged sim, -1 none */
    int64_t first_bad_draws; /* INJECT: first sim whose draw stream mismatched, -1 none */
    float kernel_ms;         /* device time of the race kernel(s) */
    int32_t lanes_per_slot;  /* K actually used */
    /* Trajectories (INJECT / MT only; run_race(record=True), race.py:378-389): positions and previous
     * steps after every tick, [n_sims][traj_cap+1][n] each (row t = after tick t, row 0 = the start);
     * rows past a sim's last tick are not written.  traj_cap = 0 disables recording. */
    double* traj_positions;
    double* traj_prev_steps;
    int32_t traj_cap;
    int32_t _pad;
    /* [ceil(n_sims / group_size) * n] winner counts per group (req.group_size > 0), or NULL */
    uint64_t* group_wins;
} bbe_result;

int bbe_simulate(const bbe_race* race, const bbe_competitor* comps, const bbe_state* state,
                 const bbe_request* req, bbe_result* out);

/* bbe_simulate over several GPUs from one host thread -- the run_batch(workers=N) analogue
 * (batch.py:110-124): the sims are split into `n_parts` contiguous shards (shard_range), part p runs
 * on device p % bbe_device_count() in its own host thread (parts on one device run in turn).
 * Tally-only requests (no per-sim output buffers; NATIVE, NATIVE64, or MT with seeds derived from
 * seed_master): each device adds its parts
 * into one device tally on its own stream, and ONE grouped NCCL all-reduce over the devices (SUM of
 * the counters fused with a MAX of the encoded first-failure fields) combines them over NVLink /
 * NVSwitch -- the SURVEY 8(b)/(e) contract; device 0's tally is the only D2H copy (BBE_ENCCL when
 * the collective fails).  Requests with per-sim outputs (or host-memory draws / seeds)
 * write those outputs at their global positions from each part and merge the tallies on the host
 * (SUM; first_diverged / first_bad_draws keep the smallest index).  Every per-sim stream is a pure
 * function of the global sim index, so results are identical for any n_parts.  n_parts <= 0 -> one
 * part per visible device.  kernel_ms = the slowest device. */
int bbe_simulate_multi(int32_t n_parts, const bbe_race* race, const bbe_competitor* comps, const bbe_state* state,
                       const bbe_request* req, bbe_result* out);

/* bbe_simulate split in two: _begin validates, uploads and enqueues everything and returns at once;
 * _end waits and fills `out`.  Host work between the two (e.g. advancing the bettor's stream past
 * the other d-1 dry-run seeds) overlaps the kernel.  Any number of calls may be in flight (each holds
 * its own stream and staging buffers; `out` identifies the call); the host buffers of `out` (and the
 * request's inputs) must stay valid until _end returns. */
int bbe_simulate_begin(const bbe_race* race, const bbe_competitor* comps, const bbe_state* state,
                       const bbe_request* req, bbe_result* out);
int bbe_simulate_end(bbe_result* out);

/* Device-resident variant.  All pointers in req/state are HOST except draws/draw_offsets/seeds,
 * which must be DEVICE pointers; per-sim output pointers in `dev_out` are DEVICE pointers or NULL.
 * Tallies are ADDED into d_tally (device, bbe_tally_len(n) u64, layout below) on `stream`
 * (a cudaStream_t, NULL = legacy default).  Asynchronous: read d_tally after the stream syncs. */
int bbe_simulate_async(const bbe_race* race, const bbe_competitor* comps, const bbe_state* state,
                       const bbe_request* req, const bbe_result* dev_out, uint64_t* d_tally, void* stream);

/* rp_predict (agents.py:153-166) in one call.  The bettor's CPython random.Random is given as its
 * MT19937 state (`state624`, 624 words) and position (`pos`, 0..624) -- random.Random.getstate()[1],
 * or the generator object's own fields -- and is advanced in place by exactly d getrandbits(64), as
 * the reference's loop advances it (agents.py:164).  wins[n] receives the winner counts of the d
 * continuations of `state`; the caller forms the Laplace probabilities (w + 1) / (d + n).
 *   mode BBE_MODE_MT:     dry run i replays random.Random(seed_i), seed_i the i-th getrandbits(64)
 *                         (simulate_from, race.py:393-406): the reference's own counts, bit for bit.
 *   mode BBE_MODE_NATIVE: the Philox stream keyed by seed_0 (statistically equal, FP32 state); the other d-1
 *                         draws only advance the stream, on the host while the GPU runs.
 *   mode BBE_MODE_NATIVE64: the same Philox stream with the reference's FP64 race arithmetic.
 * Synchronous.  BBE_EDIVERGED: a dry run exceeded tick_limit (first_diverged, if not NULL, receives
 * its index k in 0..d-1); the stream is left advanced by k + 1 draws, where the reference's loop
 * raises (agents.py:164).  Writes to the generator happen with the caller's GIL held when the call
 * is bound through ctypes.PyDLL; the GIL is dropped for the GPU wait after the last write. */
int bbe_rp_predict(const bbe_race* race, const bbe_competitor* comps, const bbe_state* state, int64_t d,
                   int32_t mode, uint32_t* state624, int32_t* pos, uint64_t* wins, int64_t* first_diverged);

/* Prepared race (NATIVE / NATIVE64): the parameter block is packed and uploaded once, on the current device,
 * so repeated device-resident launches of one race state (the bench's steps, a shard's calls) copy
 * nothing per launch.  bbe_launch_prepared adds the tallies of sims [sim_offset, sim_offset +
 * n_sims) into d_tally (device, bbe_tally_len(n) u64) on `stream`, asynchronously; a prepared race
 * serves one launch at a time (callers serialise).  bbe_prepared_kernel_ms: device time of the last
 * launch (waits for it), -1 if none. */
typedef struct bbe_prepared bbe_prepared;
int bbe_prepare(const bbe_race* race, const bbe_competitor* comps, const bbe_state* state, int32_t mode,
                int32_t lanes_per_slot_hint, bbe_prepared** out); /* mode: BBE_MODE_NATIVE or _NATIVE64 */
int bbe_launch_prepared(bbe_prepared* prepared, int64_t n_sims, int64_t sim_offset, uint64_t seed,
                        uint64_t* d_tally, void* stream);
float bbe_prepared_kernel_ms(bbe_prepared* prepared);
void bbe_release_prepared(bbe_prepared* prepared);

/* d_tally layout: [wins n][ranks n*n][perms n! or 0][ct][blocked][diverged count][bad-draw count]
 *                 [(2^63-1) - first_diverged, or 0 = none][(2^63-1) - first_bad_draws, or 0 = none]
 * Every field but the last two is SUM-reduced across shards; the last two are MAX-reduced (signed or
 * unsigned alike), which keeps the smallest failing sim index. */
int64_t bbe_tally_len(int32_t n);
int64_t bbe_tally_offset(int32_t n, int32_t field); /* field: 0 wins 1 ranks 2 perms 3 ct 4 blocked
                                                       5 n_diverged 6 n_bad 7 first_div 8 first_bad */

int bbe_derive_seeds(uint64_t master, int64_t first, int64_t count, uint64_t* out_host);

/* agents.py:164 draws each dry-run seed as rng.getrandbits(64) from the bettor's CPython
 * random.Random (MT19937).  This advances such a generator by `count` getrandbits(64) calls in
 * place -- `state625` is random.Random.getstate()[1] (624 state words + position) as uint32 --
 * and, when `out` is not NULL, stores the values drawn (low word first, as CPython builds them). */
int bbe_mt_getrandbits64(uint32_t* state625, int64_t count, uint64_t* out);

/* The same advance with the position held separately (as CPython's RandomObject stores it:
 * `int index; uint32_t state[624]`), writing only the first out_len values (out may be NULL). */
int bbe_mt_advance64(uint32_t* state624, int32_t* pos, int64_t count, uint64_t* out, int64_t out_len);

/* bbe_mt_advance64 for n_gen independent generators at once (a tick's batch of bettors, each with
 * its own d), spread over `threads` host threads (<= 0: all cores).  outs / out_lens may be NULL, or
 * hold per-generator output arrays (NULL entries allowed) and the number of values to store. */
int bbe_mt_advance64_many(int64_t n_gen, uint32_t* const* states, int32_t* const* pos, const int64_t* counts,
                          uint64_t* const* outs, const int64_t* out_lens, int32_t threads);

/* 1 if MT mode reproduces the host libm's exp() (used by random.lognormvariate) bit for bit: the
 * library found glibc's exp table in the loaded libm and verified its evaluation against exp().
 * 0 -> lognormal steps in MT mode may differ from the reference in the last bit. */
int bbe_mt_exp_exact(void);

/* Bytes of the race-parameter block copied host->device per call (the per-call H2D input). */
int64_t bbe_param_bytes(int32_t n);

/* Device time (ms) of the race kernel of the most recent call on the current device; synchronises
 * on that kernel's completion event. */
float bbe_last_kernel_ms(void);

const char* bbe_last_error(void);
int bbe_version(void);
int bbe_device_count(void);
/* Fills name (NUL-terminated, up to 63 chars), SM count and max SM clock (kHz). */
int bbe_device_info(int device, char* name64, int32_t* sm_count, int32_t* clock_khz);

#ifdef __cplusplus
}
#endif

#endif /* BBE_SIM_H */
