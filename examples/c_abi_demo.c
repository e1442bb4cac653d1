/* c_abi_demo.c -- the C-ABI (include/bbe_sim.h) used from plain C, no Python: a 10-runner race,
 * 20,000 dry runs from a mid-race state in each mode, win probabilities as rp_predict returns them
 * ((wins + 1) / (d + n), agents.py:166); then rp_predict itself (bbe_rp_predict) for a bettor whose
 * generator is CPython's random.Random(5), kept here as its MT19937 state.
 *
 *   gcc -O2 -Iinclude examples/c_abi_demo.c -Lpaper_2108_02419_b200/_lib -lbbe_sim \
 *       -Wl,-rpath,$PWD/paper_2108_02419_b200/_lib -o c_abi_demo && ./c_abi_demo
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "bbe_sim.h"

#define N 10

/* random.Random(5): MT19937 init_by_array with the one-word key {5} (CPython _randommodule.c) */
static void mt_seed_small(uint32_t mt[624], int32_t* pos, uint32_t key) {
    mt[0] = 19650218u;
    for (int i = 1; i < 624; ++i) mt[i] = 1812433253u * (mt[i - 1] ^ (mt[i - 1] >> 30)) + (uint32_t)i;
    int i = 1;
    for (int k = 624; k; --k) {
        mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key;
        if (++i >= 624) { mt[0] = mt[623]; i = 1; }
    }
    for (int k = 623; k; --k) {
        mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
        if (++i >= 624) { mt[0] = mt[623]; i = 1; }
    }
    mt[0] = 0x80000000u;
    *pos = 624;
}

int main(void) {
    bbe_race race = {2000.0, 1000000, N, 0};
    bbe_competitor comps[N];
    double pos[N], prev[N];
    int64_t fin[N];
    memset(comps, 0, sizeof comps);
    for (int c = 0; c < N; ++c) {
        comps[c].family = BBE_FAMILY_UNIFORM;
        comps[c].lo = 10.0 + (c % 3);
        comps[c].hi = 20.0 + (c % 4);
        comps[c].scale = 1.0;
        comps[c].pref_factor = 1.0;
        comps[c].theta = (c % 2) ? 8.0 : 0.0;
        comps[c].early_mult = 1.0;
        comps[c].late_mult = 1.0;
        comps[c].bp_abs = 1000.0;
        pos[c] = 900.0 + 12.5 * c;
        prev[c] = 15.0;
        fin[c] = -1;
    }
    bbe_state st = {65, pos, prev, fin, 0, 0};
    const int64_t d = 20000;
    uint64_t* seeds = (uint64_t*)malloc(sizeof(uint64_t) * d);
    if (!seeds) return 1;
    bbe_derive_seeds(11, 0, d, seeds);
    const int modes[4] = {BBE_MODE_NATIVE, BBE_MODE_NATIVE64, BBE_MODE_MT, BBE_MODE_NATIVE64};
    const char* names[4] = {"native", "native64", "mt", "multi64"};
    for (int m = 0; m < 4; ++m) {
        bbe_request rq;
        memset(&rq, 0, sizeof rq);
        rq.n_sims = d;
        rq.seed = 7;
        rq.mode = modes[m];
        rq.seeds = modes[m] == BBE_MODE_MT ? seeds : NULL;
        uint64_t wins[N];
        bbe_result out;
        memset(&out, 0, sizeof out);
        out.wins = wins;
        /* multi64: the same NATIVE64 request over every visible GPU (one part per device; the
         * device tallies are combined by one NCCL all-reduce when there is more than one) */
        const int rc = m == 3 ? bbe_simulate_multi(0, &race, comps, &st, &rq, &out)
                              : bbe_simulate(&race, comps, &st, &rq, &out);
        if (rc != BBE_OK) {
            fprintf(stderr, "bbe_simulate(%s) failed (%d): %s\n", names[m], rc, bbe_last_error());
            return 2;
        }
        uint64_t total = 0;
        printf("%-6s kernel %.3f ms, ct %llu, probs", names[m], out.kernel_ms,
               (unsigned long long)out.competitor_steps);
        for (int c = 0; c < N; ++c) {
            total += wins[c];
            printf(" %.17g", (double)(wins[c] + 1) / (double)(d + N));
        }
        printf("\n");
        if (total != (uint64_t)d) return 3;
    }
    free(seeds);

    /* rp_predict(state, config, d, random.Random(5)) in one call: the d dry-run seeds are the
     * bettor's getrandbits(64) draws, and its state is advanced in place exactly as the reference's */
    uint32_t mt[624];
    int32_t mpos;
    mt_seed_small(mt, &mpos, 5u);
    uint64_t wins[N];
    int64_t first_div = -1;
    const int rc = bbe_rp_predict(&race, comps, &st, d, BBE_MODE_MT, mt, &mpos, wins, &first_div);
    if (rc != BBE_OK) {
        fprintf(stderr, "bbe_rp_predict failed (%d): %s\n", rc, bbe_last_error());
        return 4;
    }
    printf("rp_mt  pos %d probs", (int)mpos);
    for (int c = 0; c < N; ++c) printf(" %.17g", (double)(wins[c] + 1) / (double)(d + N));
    printf("\n");
    return 0;
}
