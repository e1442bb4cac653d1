/* Probe: which evaluation order reproduces this machine's libm exp() bit for bit?
 *
 * CPython's random.lognormvariate calls libm exp (Lib/random.py); MT mode must reproduce it on the
 * GPU.  glibc's exp (sysdeps/ieee754/dbl-64/e_exp.c, the table-driven algorithm published by
 * Szabolcs Nagy / ARM optimized-routines) reads its constants from the __exp_data table, which this
 * probe locates in the libm file by its first constant (N/ln2 with N = 128).  Candidate evaluation
 * orders (with / without fused multiply-adds, as the FMA ifunc variant compiles them) are compared
 * against exp() on random arguments.  Dev tool only; build: gcc -O2 -ffp-contract=off -o p p.c -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static double T_inv, T_shift, T_hi, T_lo, C2, C3, C4, C5;
static uint64_t TAB[256];

static double asd(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static uint64_t asu(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }

static int load(const char* path) {
    FILE* f = fopen(path, "rb");
    if (!f) return -1;
    fseek(f, 0, SEEK_END);
    long sz = ftell(f);
    fseek(f, 0, SEEK_SET);
    unsigned char* b = malloc(sz);
    if (fread(b, 1, sz, f) != (size_t)sz) return -2;
    fclose(f);
    const uint64_t inv = 0x40671547652b82feull;
    for (long i = 0; i + 8 * 300 < sz; i += 8) {
        uint64_t v;
        memcpy(&v, b + i, 8);
        if (v != inv) continue;
        uint64_t q[300];
        memcpy(q, b + i, sizeof(q));
        if (q[1] != 0x4338000000000000ull) continue;
        /* tab starts where the pair (0, 0x3ff0000000000000) appears */
        for (int t = 8; t < 40; ++t) {
            if (q[t] == 0 && q[t + 1] == 0x3ff0000000000000ull) {
                T_inv = asd(q[0]); T_shift = asd(q[1]); T_hi = asd(q[2]); T_lo = asd(q[3]);
                C2 = asd(q[4]); C3 = asd(q[5]); C4 = asd(q[6]); C5 = asd(q[7]);
                memcpy(TAB, q + t, sizeof(TAB));
                printf("found __exp_data at file offset %ld, tab at +%d\n", i, t);
                free(b);
                return 0;
            }
        }
    }
    free(b);
    return -3;
}

static double variant(double x, int v) {
    double z, kd, r, r2, tmp, tail, scale;
    uint64_t ki, idx, top, sbits;
    if (v & 1) kd = fma(T_inv, x, T_shift);
    else { z = T_inv * x; kd = z + T_shift; }
    ki = asu(kd);
    kd -= T_shift;
    if (v & 2) r = fma(kd, T_lo, fma(kd, T_hi, x));
    else r = x + kd * T_hi + kd * T_lo;
    idx = 2 * (ki % 128);
    top = ki << 45;
    tail = asd(TAB[idx]);
    sbits = TAB[idx + 1] + top;
    r2 = r * r;
    if (v & 4) tmp = fma(r2 * r2, fma(r, C5, C4), fma(r2, fma(r, C3, C2), tail + r));
    else tmp = tail + r + r2 * (C2 + r * C3) + r2 * r2 * (C4 + r * C5);
    scale = asd(sbits);
    if (v & 8) return fma(scale, tmp, scale);
    return scale + scale * tmp;
}

int main(int argc, char** argv) {
    const char* path = argc > 1 ? argv[1] : "/lib/x86_64-linux-gnu/libm.so.6";
    if (load(path)) { printf("table not found\n"); return 1; }
    uint64_t s = 88172645463325252ull;
    long N = argc > 2 ? atol(argv[2]) : 20000000;
    long bad[16] = {0};
    for (long i = 0; i < N; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        double x = ((double)(s >> 11) / 9007199254740992.0) * 16.0 - 8.0;
        double ref = exp(x);
        for (int v = 0; v < 16; ++v)
            if (asu(variant(x, v)) != asu(ref)) bad[v]++;
    }
    for (int v = 0; v < 16; ++v)
        printf("variant %2d (fma kd %d, r %d, poly %d, final %d): %ld / %ld mismatches\n", v, v & 1, (v >> 1) & 1,
               (v >> 2) & 1, (v >> 3) & 1, bad[v], N);
    return 0;
}
