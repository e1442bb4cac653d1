"""FP32-state bias probe on the very same draws ("next" 1): the C5 field (20 x U(10,20),
L = 2000, from the start) through the NATIVE64 kernel twice -- the product build (FP64 state) and a
BBE_N64_F32_PROBE build that rounds every draw, step and position to FP32 after each operation --
with identical Philox draws, and counts the simulations whose winner differs.

  BBE_LIB=paper_2108_02419_b200/_lib/ab/libbbe_f32probe.so python tools/f32_probe.py write DIR N CHUNK
  python tools/f32_probe.py compare DIR N CHUNK          (product library; prints a JSON report)
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2108_02419_b200 import sim  # noqa: E402
from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps  # noqa: E402

SEED = 20260818


def main():
    what, d, n, chunk = sys.argv[1], sys.argv[2], int(float(sys.argv[3])), int(float(sys.argv[4]))
    cfg = RaceConfig(2000.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(20)))
    os.makedirs(d, exist_ok=True)
    flips = 0
    wins64 = np.zeros(20, np.int64)
    wins32 = np.zeros(20, np.int64)
    ct64 = ct32 = 0
    for i in range(n // chunk):
        r = sim.simulate_batch(None, cfg, chunk, SEED, mode="native64", winners=True, sim_offset=i * chunk)
        w = r.winner.astype(np.uint8)
        path = os.path.join(d, f"probe_{i}.npy")
        if what == "write":
            np.save(path, w)
            np.save(os.path.join(d, f"probe_{i}_meta.npy"), np.array([r.competitor_steps], np.int64))
            continue
        w32 = np.load(path)
        flips += int((w32 != w).sum())
        wins64 += np.bincount(w, minlength=20)
        wins32 += np.bincount(w32, minlength=20)
        ct64 += r.competitor_steps
        ct32 += int(np.load(os.path.join(d, f"probe_{i}_meta.npy"))[0])
        os.remove(path)
    if what == "compare":
        p = wins64 / n
        se = math.sqrt(2 * p.max() * (1 - p.max()) / n)
        print(json.dumps({
            "sims": n, "field": "C5: 20 x U(10,20), L = 2000, from the start", "seed": SEED,
            "winner_flips": flips, "winner_flips_per_1e9": flips * 1e9 / n,
            "max_abs_win_prob_diff": float(np.abs(wins64 - wins32).max() / n),
            "binomial_se_of_a_difference_at_max_p": se,
            "ct_per_race": [ct64 / n, ct32 / n],
            "note": "same Philox draws; FP64 state (product NATIVE64) vs FP32-rounded state (BBE_N64_F32_PROBE build)"}))


if __name__ == "__main__":
    main()
