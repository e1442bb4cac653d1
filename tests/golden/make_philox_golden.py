"""Known-answer vectors for Philox4x32-10 from an independent implementation: ATen's philox_engine
(torch/include/ATen/core/PhiloxRNGEngine.h, Salmon et al. SC'11).

The NATIVE / NATIVE64 kernels and the C oracle (oracle/bbe_oracle.c orc_philox4x32_10) draw from
Philox4x32-10 with counter (word0, competitor, sim_lo, sim_hi) and key = the request seed.  ATen's
engine is philox_engine(seed, subsequence, offset): key = seed, counter = (offset_lo, offset_hi,
subsequence_lo, subsequence_hi), so one block of ours is philox_engine(key, sim, (comp << 32) | word0)
and its first four outputs.  This script compiles a tiny C++ program against the torch headers,
evaluates a spread of (key, counter) pairs and writes tests/golden/philox.json (committed).

Run here (needs g++ and the torch headers): python tests/golden/make_philox_golden.py
"""

from __future__ import annotations

import json
import os
import subprocess
import tempfile

import torch

HERE = os.path.dirname(os.path.abspath(__file__))

SRC = r"""
#include <ATen/core/PhiloxRNGEngine.h>
#include <cstdio>
#include <cstdint>
int main() {
    unsigned long long key; unsigned c0, c1, c2, c3;
    while (std::scanf("%llu %u %u %u %u", &key, &c0, &c1, &c2, &c3) == 5) {
        const uint64_t sub = (uint64_t)c2 | ((uint64_t)c3 << 32);
        const uint64_t off = (uint64_t)c0 | ((uint64_t)c1 << 32);
        at::philox_engine e(key, sub, off);
        unsigned a = e(), b = e(), c = e(), d = e();
        std::printf("%u %u %u %u\n", a, b, c, d);
    }
    return 0;
}
"""


def main():
    inc = os.path.join(os.path.dirname(torch.__file__), "include")
    cases = [
        (0, (0, 0, 0, 0)),
        (0xFFFFFFFFFFFFFFFF, (0xFFFFFFFF,) * 4),
        (0x299F31D0A4093822, (0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344)),
        (20260818, (0, 3, 12345, 0)),
        (20260818, (0xFFFFFFFF, 7, 99, 1)),  # a priming-draw counter
        (11, (40, 19, 0xFFFFFFFF, 0x3B)),
    ]
    import random

    rng = random.Random(2108_02419)
    for _ in range(58):
        cases.append((rng.getrandbits(64), tuple(rng.getrandbits(32) for _ in range(4))))
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "p.cpp")
        exe = os.path.join(tmp, "p")
        with open(src, "w") as fh:
            fh.write(SRC)
        subprocess.run(["g++", "-O1", "-std=c++17", "-I", inc, src, "-o", exe], check=True)
        inp = "".join(f"{k} {c[0]} {c[1]} {c[2]} {c[3]}\n" for k, c in cases)
        out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
    vectors = []
    for (k, c), line in zip(cases, out):
        vectors.append({"key": k, "counter": list(c), "out": [int(x) for x in line.split()]})
    with open(os.path.join(HERE, "philox.json"), "w") as fh:
        json.dump({"source": "ATen philox_engine (torch " + torch.__version__ + ")", "vectors": vectors}, fh, indent=0)
    print(f"wrote {len(vectors)} vectors")


if __name__ == "__main__":
    main()
