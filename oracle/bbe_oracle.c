/*
 * bbe_oracle.c -- CPU restatement of the reference race engine (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity checker for the B200 kernels.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product library
 * (paper_2108_02419_b200/_lib/libbbe_sim.so) never links or calls it.
 *
 * It restates, in plain C99, the reference's algorithm for the hot path:
 *   - CPython's random.Random (MT19937 + init_by_array seeding, random(), getrandbits(64),
 *     uniform(), normalvariate() (Kinderman-Monahan), lognormvariate()) -- the stdlib code the
 *     reference calls at race.py:47 (UniformSteps.draw), race.py:69 (LogNormalSteps.draw),
 *     seeding.py:62-64 (make_rng) and agents.py:164 (rng.getrandbits(64)).
 *     Third-party pin: CPython 3.12.3 Modules/_randommodule.c and Lib/random.py (the algorithms
 *     are unchanged since 3.2 for the pieces used here).
 *   - seeding.py:24-59 (splitmix64, fnv1a, derive_seed).
 *   - race.py:192-199 (preference_factor), :93-96 (Responsiveness.at), :233-241 (initial_state),
 *     :244-264 (_front_runner), :267-274 (_resolve_step), :287-320 (advance_race),
 *     :323-332 (_finish_order), :373-390 (run_race), :393-406 (simulate_from).
 *   - agents.py:153-166 (rp_predict) and batch.py:110-124 (run_batch seeds).
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against golden vectors
 * produced by running the reference itself (tests/golden/make_golden.py).
 *
 * Build: gcc -O2 -std=c99 -ffp-contract=off -fPIC -shared (see oracle/Makefile).  FP contraction
 * must stay off: Python floats never fuse multiply-add.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------ */
/* MT19937 as in CPython Modules/_randommodule.c                                               */
/* ------------------------------------------------------------------------------------------ */
#define MT_N 624
#define MT_M 397

typedef struct {
    uint32_t mt[MT_N];
    int index;
} orc_mt;

static void mt_init_genrand(orc_mt* s, uint32_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < MT_N; i++)
        s->mt[i] = 1812433253u * (s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) + (uint32_t)i;
    s->index = MT_N;
}

static void mt_init_by_array(orc_mt* s, const uint32_t* key, int keylen) {
    mt_init_genrand(s, 19650218u);
    int i = 1, j = 0;
    int k = MT_N > keylen ? MT_N : keylen;
    for (; k; k--) {
        s->mt[i] = (s->mt[i] ^ ((s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
        i++;
        j++;
        if (i >= MT_N) { s->mt[0] = s->mt[MT_N - 1]; i = 1; }
        if (j >= keylen) j = 0;
    }
    for (k = MT_N - 1; k; k--) {
        s->mt[i] = (s->mt[i] ^ ((s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
        i++;
        if (i >= MT_N) { s->mt[0] = s->mt[MT_N - 1]; i = 1; }
    }
    s->mt[0] = 0x80000000u;
    s->index = MT_N;
}

/* random.Random(seed) for a non-negative int seed < 2**64 (seeding.py:62-64 masks to 64 bits):
 * the key is the little-endian 32-bit words of the seed, at least one word. */
static void mt_seed_u64(orc_mt* s, uint64_t seed) {
    uint32_t key[2];
    key[0] = (uint32_t)seed;
    key[1] = (uint32_t)(seed >> 32);
    mt_init_by_array(s, key, key[1] ? 2 : 1);
}

static uint32_t mt_u32(orc_mt* s) {
    static const uint32_t mag01[2] = {0u, 0x9908b0dfu};
    uint32_t y;
    if (s->index >= MT_N) {
        int kk;
        for (kk = 0; kk < MT_N - MT_M; kk++) {
            y = (s->mt[kk] & 0x80000000u) | (s->mt[kk + 1] & 0x7fffffffu);
            s->mt[kk] = s->mt[kk + MT_M] ^ (y >> 1) ^ mag01[y & 1u];
        }
        for (; kk < MT_N - 1; kk++) {
            y = (s->mt[kk] & 0x80000000u) | (s->mt[kk + 1] & 0x7fffffffu);
            s->mt[kk] = s->mt[kk + (MT_M - MT_N)] ^ (y >> 1) ^ mag01[y & 1u];
        }
        y = (s->mt[MT_N - 1] & 0x80000000u) | (s->mt[0] & 0x7fffffffu);
        s->mt[MT_N - 1] = s->mt[MT_M - 1] ^ (y >> 1) ^ mag01[y & 1u];
        s->index = 0;
    }
    y = s->mt[s->index++];
    y ^= (y >> 11);
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= (y >> 18);
    return y;
}

/* random_random(): 53-bit float from two words */
static double mt_random(orc_mt* s) {
    uint32_t a = mt_u32(s) >> 5, b = mt_u32(s) >> 6;
    return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
}

/* getrandbits(64): words fill from the least significant end */
static uint64_t mt_getrandbits64(orc_mt* s) {
    uint64_t lo = mt_u32(s);
    uint64_t hi = mt_u32(s);
    return lo | (hi << 32);
}

static double mt_uniform(orc_mt* s, double a, double b) { return a + (b - a) * mt_random(s); }

static double nv_magicconst(void) { return 4 * exp(-0.5) / sqrt(2.0); }

/* Lib/random.py normalvariate: Kinderman-Monahan ratio of uniforms */
static double mt_normalvariate(orc_mt* s, double mu, double sigma) {
    const double NV = nv_magicconst();
    double z;
    for (;;) {
        double u1 = mt_random(s);
        double u2 = 1.0 - mt_random(s);
        z = NV * (u1 - 0.5) / u2;
        double zz = z * z / 4.0;
        if (zz <= -log(u2)) break;
    }
    return mu + z * sigma;
}

static double mt_lognormvariate(orc_mt* s, double mu, double sigma) {
    return exp(mt_normalvariate(s, mu, sigma));
}

/* ------------------------------------------------------------------------------------------ */
/* seeding.py:24-59                                                                            */
/* ------------------------------------------------------------------------------------------ */
uint64_t orc_splitmix64(uint64_t x) {
    x = x + 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

uint64_t orc_fnv1a(const uint8_t* data, int64_t len) {
    uint64_t h = 0xCBF29CE484222325ull;
    for (int64_t i = 0; i < len; i++) h = (h ^ data[i]) * 0x100000001B3ull;
    return h;
}

static uint64_t fnv_int(uint64_t v) { /* _encode(int) = b"i:" + 8 bytes big endian */
    uint8_t b[10] = {'i', ':'};
    for (int k = 0; k < 8; k++) b[2 + k] = (uint8_t)(v >> (56 - 8 * k));
    return orc_fnv1a(b, 10);
}

static uint64_t fnv_str(const char* str) { /* _encode(str) = b"s:" + utf8 */
    uint8_t b[256] = {'s', ':'};
    size_t n = strlen(str);
    if (n > 250) n = 250;
    memcpy(b + 2, str, n);
    return orc_fnv1a(b, (int64_t)n + 2);
}

/* derive_seed(master, "run", i) -- the per-run seed of batch.py:117-119 */
uint64_t orc_derive_seed_run(uint64_t master, uint64_t i) {
    uint64_t h = orc_splitmix64(master);
    h = orc_splitmix64(h ^ fnv_str("run"));
    h = orc_splitmix64(h ^ fnv_int(i));
    return h;
}

/* ------------------------------------------------------------------------------------------ */
/* Race engine (race.py)                                                                       */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int32_t family; /* 0 uniform (lo, hi), 1 lognormal (mu, sigma, scale) */
    int32_t _pad;
    double lo, hi, mu, sigma, scale;
    double preference, pref_sensitivity, theta;
    double early_mult, late_mult, breakpoint;
} orc_comp;

typedef struct {
    double track_length;
    double conditions;
    int64_t tick_limit;
    int32_t n;
    int32_t _pad;
} orc_race;

enum { ORC_OK = 0, ORC_EDIVERGED = 2, ORC_EDRAWS = 3, ORC_EINVAL = 1 };

/* ------------------------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers: as easy as 1, 2, 3"): */
/* the counter-based word generator of the NATIVE / NATIVE64 kernels.  Pinned to ATen's independent */
/* philox_engine (torch/include/ATen/core/PhiloxRNGEngine.h) by tests/golden/make_philox_golden.py. */
/* ------------------------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t* ctr_in, uint64_t key, uint32_t* out) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    for (int r = 0; r < 10; r++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1, n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* NATIVE64's draw of two words (common.cuh unit53): the top 53 bits of w0:w1 times 2^-53 */
static double unit53(uint32_t w0, uint32_t w1) {
    return (double)((((uint64_t)w0 << 32) | w1) >> 11) * (1.0 / 9007199254740992.0);
}

/* Draw source: an MT stream (the reference), a replay of recorded draw values, or the NATIVE64
 * Philox stream (counter-based: the draw of competitor c at the sim's relative tick rt). */
typedef struct {
    int philox;    /* 1: NATIVE64 stream keyed by `key` for global sim index `gs` */
    uint64_t key, gs;
    int64_t rt;    /* ticks this sim has advanced (-1: run_race's priming draws) */
    orc_mt* mt;
    const double* replay;
    int64_t replay_len;
    int64_t cursor;
    double* rec; /* optional record of every draw value, in consumption order */
    int64_t rec_cap;
    int underflow;
} orc_draws;

/* NATIVE64 draw (native64_kernel.cuh): counter (rt / 2, c, gs) -- word 0 = 0xFFFFFFFF for the
 * priming draws -- gives (x, y, z, w); a uniform takes lo + (hi - lo) * unit53 of (x, y) at even
 * rt and (z, w) at odd rt; a lognormal takes scale * exp(mu + z * sigma) with the Box-Muller normal
 * of u1 = 1 - unit53(x, y), u2 = unit53(z, w): the cosine branch at even rt, the sine at odd. */
static double draw_philox(const orc_draws* d, const orc_comp* cp, int c) {
    uint32_t ctr[4] = {d->rt < 0 ? 0xFFFFFFFFu : (uint32_t)(d->rt >> 1), (uint32_t)c, (uint32_t)d->gs,
                       (uint32_t)(d->gs >> 32)};
    uint32_t w[4];
    orc_philox4x32_10(ctr, d->key, w);
    int odd = d->rt >= 0 && (d->rt & 1);
    if (cp->family == 0) return cp->lo + (cp->hi - cp->lo) * (odd ? unit53(w[2], w[3]) : unit53(w[0], w[1]));
    double u1 = 1.0 - unit53(w[0], w[1]), u2 = unit53(w[2], w[3]);
    double r = sqrt(-2.0 * log(u1));
    double t = 3.141592653589793 * (2.0 * u2);
    double z = odd ? r * sin(t) : r * cos(t);
    return cp->scale * exp(cp->mu + z * cp->sigma);
}

static double draw_raw(orc_draws* d, const orc_comp* c, int ci) {
    double v;
    if (d->philox) {
        v = draw_philox(d, c, ci);
    } else if (d->replay) {
        if (d->cursor >= d->replay_len) { d->underflow = 1; v = c->family ? c->scale : c->lo; }
        else v = d->replay[d->cursor];
    } else if (c->family == 0) {
        v = mt_uniform(d->mt, c->lo, c->hi); /* race.py:46-47 */
    } else {
        v = c->scale * mt_lognormvariate(d->mt, c->mu, c->sigma); /* race.py:68-69 */
    }
    if (d->rec && d->cursor < d->rec_cap) d->rec[d->cursor] = v;
    d->cursor++;
    return v;
}

/* race.py:192-199 */
double orc_preference_factor(double conditions, double preference, double sensitivity) {
    double f = 1.0 - sensitivity * fabs(conditions - preference);
    if (f < 0.01) return 0.01;
    if (f > 1.0) return 1.0;
    return f;
}

/* race.py:93-96 */
static double resp_at(const orc_comp* c, double pos, double length) {
    if (pos < c->breakpoint * length) return c->early_mult;
    return c->late_mult;
}

typedef struct {
    int64_t tick;
    double* pos;
    double* prev;
    int64_t* fin; /* -1 = still racing (None) */
    int64_t blocked;
} orc_state;

/* race.py:233-241 */
static void initial_state(const orc_race* r, const orc_comp* comps, orc_draws* d, orc_state* st) {
    for (int c = 0; c < r->n; c++) {
        double pref = orc_preference_factor(r->conditions, comps[c].preference, comps[c].pref_sensitivity);
        double resp = resp_at(&comps[c], 0.0, r->track_length);
        st->prev[c] = resp * pref * draw_raw(d, &comps[c], c);
        st->pos[c] = 0.0;
        st->fin[c] = -1;
    }
    st->tick = 0;
    st->blocked = 0;
}

/* race.py:244-264: nearest still-racing rival strictly ahead; ties on gap -> lowest index */
static int front_runner(const orc_state* st, int n, int c, double* gap_out) {
    double pc = st->pos[c];
    int best_i = -1;
    double best_gap = -1.0;
    for (int i = 0; i < n; i++) {
        if (i == c || st->fin[i] >= 0) continue;
        double p = st->pos[i];
        if (p > pc) {
            double gap = p - pc;
            if (best_i < 0 || gap < best_gap) { best_i = i; best_gap = gap; }
        }
    }
    *gap_out = best_gap;
    return best_i;
}

/* race.py:287-320 (with _resolve_step race.py:267-274 inlined) */
static void advance(const orc_race* r, const orc_comp* comps, orc_draws* d, orc_state* st, double* steps) {
    int n = r->n;
    int64_t blocked = 0;
    for (int c = 0; c < n; c++) {
        if (st->fin[c] >= 0) continue;
        const orc_comp* cp = &comps[c];
        double resp = resp_at(cp, st->pos[c], r->track_length);
        double gap;
        int f = front_runner(st, n, c, &gap);
        if (f < 0 || gap > cp->theta) {
            double pref = orc_preference_factor(r->conditions, cp->preference, cp->pref_sensitivity);
            steps[c] = resp * pref * draw_raw(d, cp, c);
        } else {
            double a = st->prev[c], b = st->prev[f];
            steps[c] = resp * (b < a ? b : a); /* Python min(a, b) */
            blocked++;
        }
    }
    int64_t t = st->tick + 1;
    for (int c = 0; c < n; c++) {
        if (st->fin[c] >= 0) continue;
        double p = st->pos[c] + steps[c];
        if (p == st->pos[c]) p = nextafter(p, INFINITY);
        st->pos[c] = p;
        st->prev[c] = steps[c];
        if (p >= r->track_length) st->fin[c] = t;
    }
    st->tick = t;
    st->blocked += blocked;
}

static int all_finished(const orc_state* st, int n) {
    for (int c = 0; c < n; c++)
        if (st->fin[c] < 0) return 0;
    return 1;
}

/* race.py:323-332: sort by (finish_tick, L - pos, index) */
static void finish_order(const orc_race* r, const orc_state* st, int32_t* order) {
    int n = r->n;
    for (int c = 0; c < n; c++) order[c] = c;
    for (int a = 1; a < n; a++) { /* insertion sort, stable, n <= a few dozen */
        int32_t v = order[a];
        int b = a - 1;
        while (b >= 0) {
            int32_t u = order[b];
            double ku = r->track_length - st->pos[u], kv = r->track_length - st->pos[v];
            int less = st->fin[v] < st->fin[u] || (st->fin[v] == st->fin[u] && (kv < ku || (kv == ku && v < u)));
            if (!less) break;
            order[b + 1] = u;
            b--;
        }
        order[b + 1] = v;
    }
}

typedef struct {
    int64_t* finish_ticks; /* [n] */
    int32_t* order;        /* [n] */
    double* final_pos;     /* [n] */
    int64_t blocked;
    int64_t draws_used;
    int64_t n_ticks_run; /* ticks advanced by this call */
    int64_t ct;          /* competitor-timesteps (racing _resolve_step calls) */
} orc_out;

#define ORC_MAXN 256

static int run_core(const orc_race* r, const orc_comp* comps, orc_draws* d, orc_state* st, int from_start,
                    orc_out* out) {
    int n = r->n;
    double steps[ORC_MAXN];
    int rc = ORC_OK;
    int64_t start = st->tick;
    int64_t ct = 0;
    while (!all_finished(st, n)) {
        if (from_start ? (st->tick >= r->tick_limit) : (st->tick - start >= r->tick_limit)) {
            rc = ORC_EDIVERGED;
            break;
        }
        for (int c = 0; c < n; c++) ct += st->fin[c] < 0;
        d->rt = st->tick - start;
        advance(r, comps, d, st, steps);
    }
    if (d->replay && rc == ORC_OK && (d->underflow || d->cursor != d->replay_len)) rc = ORC_EDRAWS;
    if (out) {
        if (out->finish_ticks) memcpy(out->finish_ticks, st->fin, sizeof(int64_t) * n);
        if (out->final_pos) memcpy(out->final_pos, st->pos, sizeof(double) * n);
        if (out->order && rc != ORC_EDIVERGED) finish_order(r, st, out->order);
        out->blocked = st->blocked;
        out->draws_used = d->cursor;
        out->n_ticks_run = st->tick - start;
        out->ct = ct;
    }
    return rc;
}

/* run_race (race.py:373-390).  replay != NULL replays recorded draws instead of MT(seed). */
int orc_run_race(const orc_race* r, const orc_comp* comps, uint64_t seed, const double* replay,
                 int64_t replay_len, double* rec, int64_t rec_cap, orc_out* out) {
    int n = r->n;
    if (n < 1 || n > ORC_MAXN) return ORC_EINVAL;
    orc_mt mt;
    orc_draws d = {0};
    if (replay) { d.replay = replay; d.replay_len = replay_len; }
    else { mt_seed_u64(&mt, seed); d.mt = &mt; }
    d.rec = rec;
    d.rec_cap = rec_cap;
    double pos[ORC_MAXN], prev[ORC_MAXN];
    int64_t fin[ORC_MAXN];
    orc_state st = {0, pos, prev, fin, 0};
    initial_state(r, comps, &d, &st);
    return run_core(r, comps, &d, &st, 1, out);
}

/* simulate_from (race.py:393-406): clone state, fresh stream, no priming draws. */
int orc_simulate_from(const orc_race* r, const orc_comp* comps, int64_t tick, const double* pos0,
                      const double* prev0, const int64_t* fin0, uint64_t seed, const double* replay,
                      int64_t replay_len, double* rec, int64_t rec_cap, orc_out* out) {
    int n = r->n;
    if (n < 1 || n > ORC_MAXN) return ORC_EINVAL;
    orc_mt mt;
    orc_draws d = {0};
    if (replay) { d.replay = replay; d.replay_len = replay_len; }
    else { mt_seed_u64(&mt, seed); d.mt = &mt; }
    d.rec = rec;
    d.rec_cap = rec_cap;
    double pos[ORC_MAXN], prev[ORC_MAXN];
    int64_t fin[ORC_MAXN];
    memcpy(pos, pos0, sizeof(double) * n);
    memcpy(prev, prev0, sizeof(double) * n);
    memcpy(fin, fin0, sizeof(int64_t) * n);
    orc_state st = {tick, pos, prev, fin, 0};
    return run_core(r, comps, &d, &st, 0, out);
}

/* run_race / simulate_from on the NATIVE64 Philox stream (key, global sim index gs) instead of MT. */
int orc_run_race_px(const orc_race* r, const orc_comp* comps, uint64_t key, uint64_t gs, orc_out* out) {
    int n = r->n;
    if (n < 1 || n > ORC_MAXN) return ORC_EINVAL;
    orc_draws d = {0};
    d.philox = 1; d.key = key; d.gs = gs; d.rt = -1;
    double pos[ORC_MAXN], prev[ORC_MAXN];
    int64_t fin[ORC_MAXN];
    orc_state st = {0, pos, prev, fin, 0};
    initial_state(r, comps, &d, &st);
    return run_core(r, comps, &d, &st, 1, out);
}

int orc_simulate_from_px(const orc_race* r, const orc_comp* comps, int64_t tick, const double* pos0,
                         const double* prev0, const int64_t* fin0, uint64_t key, uint64_t gs, orc_out* out) {
    int n = r->n;
    if (n < 1 || n > ORC_MAXN) return ORC_EINVAL;
    orc_draws d = {0};
    d.philox = 1; d.key = key; d.gs = gs;
    double pos[ORC_MAXN], prev[ORC_MAXN];
    int64_t fin[ORC_MAXN];
    memcpy(pos, pos0, sizeof(double) * n);
    memcpy(prev, prev0, sizeof(double) * n);
    memcpy(fin, fin0, sizeof(int64_t) * n);
    orc_state st = {tick, pos, prev, fin, 0};
    return run_core(r, comps, &d, &st, 0, out);
}

/* Advance a live race (the session's race) k ticks from initial_state on make_rng(seed):
 * reproduces the reference's way of building mid-race states (e.g. SURVEY C2). */
int orc_advance_from_start(const orc_race* r, const orc_comp* comps, uint64_t seed, int64_t k,
                           int64_t* tick, double* pos, double* prev, int64_t* fin, int64_t* blocked) {
    int n = r->n;
    if (n < 1 || n > ORC_MAXN) return ORC_EINVAL;
    orc_mt mt;
    mt_seed_u64(&mt, seed);
    orc_draws d = {0};
    d.mt = &mt;
    orc_state st = {0, pos, prev, fin, 0};
    double steps[ORC_MAXN];
    initial_state(r, comps, &d, &st);
    for (int64_t i = 0; i < k && !all_finished(&st, n); i++) advance(r, comps, &d, &st, steps);
    *tick = st.tick;
    *blocked = st.blocked;
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* RNG probes (for pinning against CPython)                                                    */
/* ------------------------------------------------------------------------------------------ */
void orc_mt_random(uint64_t seed, int64_t k, double* out) {
    orc_mt mt;
    mt_seed_u64(&mt, seed);
    for (int64_t i = 0; i < k; i++) out[i] = mt_random(&mt);
}

void orc_mt_getrandbits64(uint64_t seed, int64_t k, uint64_t* out) {
    orc_mt mt;
    mt_seed_u64(&mt, seed);
    for (int64_t i = 0; i < k; i++) out[i] = mt_getrandbits64(&mt);
}

void orc_mt_lognormvariate(uint64_t seed, double mu, double sigma, int64_t k, double* out) {
    orc_mt mt;
    mt_seed_u64(&mt, seed);
    for (int64_t i = 0; i < k; i++) out[i] = mt_lognormvariate(&mt, mu, sigma);
}

void orc_mt_uniform(uint64_t seed, double a, double b, int64_t k, double* out) {
    orc_mt mt;
    mt_seed_u64(&mt, seed);
    for (int64_t i = 0; i < k; i++) out[i] = mt_uniform(&mt, a, b);
}

/* ------------------------------------------------------------------------------------------ */
/* Batches: rp_predict (agents.py:153-166) and run_batch (batch.py:110-124), multi-threaded    */
/* over sims for the CPU baseline.  Tallies: wins[n], ranks[n*n] (ranks[c*n + r] = #sims where */
/* competitor c finished at rank r), optional per-sim winner.                                 */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    const orc_race* r;
    const orc_comp* comps;
    int from_start;
    int64_t tick;
    const double* pos0;
    const double* prev0;
    const int64_t* fin0;
    const uint64_t* seeds; /* per-sim seeds, or NULL -> derive_seed(master, "run", i) */
    uint64_t master;
    int px;              /* 1: NATIVE64 Philox stream (key = master, global index sim_offset + s) */
    int64_t sim_offset;
    int32_t* order_out;  /* optional per-sim records [n_sims*n] / [n_sims] */
    int64_t* fin_out;
    double* fpos_out;
    int64_t* blk_out;
    int64_t lo, hi;
    int32_t* winners;
    uint64_t wins[ORC_MAXN];
    uint64_t* ranks; /* private [n*n] */
    int64_t ct, blocked, first_diverged;
    int rc;
} orc_job;

static void* batch_worker(void* arg) {
    orc_job* j = (orc_job*)arg;
    int n = j->r->n;
    int64_t fin[ORC_MAXN];
    int32_t order[ORC_MAXN];
    double fpos[ORC_MAXN];
    j->first_diverged = -1;
    for (int64_t s = j->lo; s < j->hi; s++) {
        orc_out out = {fin, order, fpos, 0, 0, 0, 0};
        int rc;
        if (j->px) {
            uint64_t gs = (uint64_t)(j->sim_offset + s);
            rc = j->from_start ? orc_run_race_px(j->r, j->comps, j->master, gs, &out)
                               : orc_simulate_from_px(j->r, j->comps, j->tick, j->pos0, j->prev0, j->fin0, j->master,
                                                      gs, &out);
        } else {
            uint64_t seed = j->seeds ? j->seeds[s] : orc_derive_seed_run(j->master, (uint64_t)s);
            rc = j->from_start ? orc_run_race(j->r, j->comps, seed, NULL, 0, NULL, 0, &out)
                               : orc_simulate_from(j->r, j->comps, j->tick, j->pos0, j->prev0, j->fin0, seed,
                                                   NULL, 0, NULL, 0, &out);
        }
        if (j->order_out) memcpy(j->order_out + s * n, order, sizeof(int32_t) * n);
        if (j->fin_out) memcpy(j->fin_out + s * n, fin, sizeof(int64_t) * n);
        if (j->fpos_out) memcpy(j->fpos_out + s * n, fpos, sizeof(double) * n);
        if (j->blk_out) j->blk_out[s] = out.blocked;
        if (rc != ORC_OK) {
            if (j->first_diverged < 0) j->first_diverged = s;
            j->rc = rc;
            break;
        }
        j->wins[order[0]]++;
        if (j->ranks)
            for (int k = 0; k < n; k++) j->ranks[order[k] * n + k]++;
        if (j->winners) j->winners[s] = order[0];
        j->ct += out.ct;
        j->blocked += out.blocked;
    }
    return NULL;
}

static int batch_run(const orc_race* r, const orc_comp* comps, int from_start, int64_t tick, const double* pos0,
                     const double* prev0, const int64_t* fin0, int64_t n_sims, const uint64_t* seeds, uint64_t master,
                     int px, int64_t sim_offset, int32_t* order_out, int64_t* fin_out, double* fpos_out,
                     int64_t* blk_out, int nthreads, uint64_t* wins, uint64_t* ranks, int32_t* winners, int64_t* ct,
                     int64_t* blocked, int64_t* first_diverged) {
    int n = r->n;
    if (n < 1 || n > ORC_MAXN || nthreads < 1) return ORC_EINVAL;
    if (nthreads > 256) nthreads = 256;
    orc_job* jobs = (orc_job*)calloc((size_t)nthreads, sizeof(orc_job));
    pthread_t th[256];
    for (int t = 0; t < nthreads; t++) {
        orc_job* j = &jobs[t];
        j->r = r; j->comps = comps; j->from_start = from_start; j->tick = tick;
        j->pos0 = pos0; j->prev0 = prev0; j->fin0 = fin0; j->seeds = seeds; j->master = master;
        j->px = px; j->sim_offset = sim_offset;
        j->order_out = order_out; j->fin_out = fin_out; j->fpos_out = fpos_out; j->blk_out = blk_out;
        j->lo = n_sims * t / nthreads; j->hi = n_sims * (t + 1) / nthreads;
        j->winners = winners;
        j->ranks = ranks ? (uint64_t*)calloc((size_t)n * n, sizeof(uint64_t)) : NULL;
        if (nthreads > 1) pthread_create(&th[t], NULL, batch_worker, j);
    }
    if (nthreads == 1) batch_worker(&jobs[0]);
    else for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    int rc = ORC_OK;
    *ct = 0; *blocked = 0; *first_diverged = -1;
    for (int c = 0; c < n; c++) wins[c] = 0;
    if (ranks) memset(ranks, 0, sizeof(uint64_t) * n * n);
    for (int t = 0; t < nthreads; t++) {
        orc_job* j = &jobs[t];
        for (int c = 0; c < n; c++) wins[c] += j->wins[c];
        if (ranks) { for (int k = 0; k < n * n; k++) ranks[k] += j->ranks[k]; free(j->ranks); }
        *ct += j->ct; *blocked += j->blocked;
        if (j->rc != ORC_OK && rc == ORC_OK) { rc = j->rc; *first_diverged = j->first_diverged; }
    }
    free(jobs);
    return rc;
}

int orc_batch(const orc_race* r, const orc_comp* comps, int from_start, int64_t tick, const double* pos0,
              const double* prev0, const int64_t* fin0, int64_t n_sims, const uint64_t* seeds, uint64_t master,
              int nthreads, uint64_t* wins, uint64_t* ranks, int32_t* winners, int64_t* ct, int64_t* blocked,
              int64_t* first_diverged) {
    return batch_run(r, comps, from_start, tick, pos0, prev0, fin0, n_sims, seeds, master, 0, 0, NULL, NULL, NULL,
                     NULL, nthreads, wins, ranks, winners, ct, blocked, first_diverged);
}

/* The NATIVE64 stream: sim s = global index sim_offset + s of the Philox stream keyed by `key`;
 * optional per-sim finish orders, finish ticks, final positions and blocked counts. */
int orc_batch_px(const orc_race* r, const orc_comp* comps, int from_start, int64_t tick, const double* pos0,
                 const double* prev0, const int64_t* fin0, int64_t n_sims, int64_t sim_offset, uint64_t key,
                 int nthreads, uint64_t* wins, uint64_t* ranks, int32_t* order_out, int64_t* fin_out,
                 double* fpos_out, int64_t* blk_out, int64_t* ct, int64_t* blocked, int64_t* first_diverged) {
    return batch_run(r, comps, from_start, tick, pos0, prev0, fin0, n_sims, NULL, key, 1, sim_offset, order_out,
                     fin_out, fpos_out, blk_out, nthreads, wins, ranks, NULL, ct, blocked, first_diverged);
}
