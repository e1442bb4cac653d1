// host_mt.cpp -- advance a CPython random.Random (MT19937) state on the host CPU.
//
// rp_predict draws each dry-run seed as rng.getrandbits(64) (agents.py:164): 2 words per seed, low
// word first.  Keeping the bettor's stream identical to the reference's means advancing it by 2d
// words per call -- 200k words for d = 100k.  The twist loops below are written so GCC vectorises
// them (AVX2 clone chosen at load time where the CPU has it, generic code otherwise).
#include <stdint.h>

#include <algorithm>

namespace {

inline uint32_t mix(uint32_t a, uint32_t b, uint32_t m) {
    const uint32_t y = (a & 0x80000000u) | (b & 0x7fffffffu);
    return m ^ (y >> 1) ^ ((0u - (y & 1u)) & 0x9908b0dfu);
}

inline uint32_t temper(uint32_t y) {
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    return y ^ (y >> 18);
}

// Regenerate the 624-word block in place (MT19937): words [0, 227) read only old words, words
// [227, 623) read words 227 positions back (already new), the last word wraps to word 0.
__attribute__((target_clones("avx2", "default"))) void twist(uint32_t* __restrict mt) {
    uint32_t nxt[624];
    for (int k = 0; k < 623; ++k) nxt[k] = mt[k + 1];  // old successors, so each loop is elementwise
    for (int k = 0; k < 227; ++k) mt[k] = mix(mt[k], nxt[k], mt[k + 397]);
    for (int k = 227; k < 454; ++k) mt[k] = mix(mt[k], nxt[k], mt[k - 227]);
    for (int k = 454; k < 623; ++k) mt[k] = mix(mt[k], nxt[k], mt[k - 227]);
    mt[623] = mix(mt[623], mt[0], mt[396]);
}

}  // namespace

// state: 624 words, idx: position in the block; stores the first min(count, out_len) values drawn;
// returns the new position.
extern "C" uint32_t bbe_host_mt_getrandbits64(uint32_t* mt, uint32_t idx, int64_t count, uint64_t* out,
                                              int64_t out_len) {
    if (out && out_len < count) {  // values for a prefix, then a plain advance
        const int64_t head = out_len < 0 ? 0 : out_len;
        idx = bbe_host_mt_getrandbits64(mt, idx, head, out, head);
        return bbe_host_mt_getrandbits64(mt, idx, count - head, nullptr, 0);
    }
    int64_t words = 2 * count;
    if (!out) {  // advance only: whole blocks need no tempering
        while (words > 0) {
            if (idx >= 624) {
                twist(mt);
                idx = 0;
            }
            const int64_t take = std::min<int64_t>(words, 624 - idx);
            idx += (uint32_t)take;
            words -= take;
        }
        return idx;
    }
    int64_t i = 0;
    while (i < count) {
        if (idx >= 623) {  // two words straddle the block edge: one word at a time
            uint32_t w[2];
            for (int j = 0; j < 2; ++j) {
                if (idx >= 624) {
                    twist(mt);
                    idx = 0;
                }
                w[j] = temper(mt[idx++]);
            }
            out[i++] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
            continue;
        }
        const int64_t pairs = std::min<int64_t>(count - i, (624 - idx) / 2);
        for (int64_t p = 0; p < pairs; ++p, idx += 2)
            out[i++] = (uint64_t)temper(mt[idx]) | ((uint64_t)temper(mt[idx + 1]) << 32);
    }
    return idx;
}
