"""Launch one MT-mode batch of a BASELINE field a few times (seeding + exact race kernel) -- the
command ncu profiles.   usage: python tools/profile_mt.py FIELD [sims] [reps]   (FIELD as profile_cfg.py;
env BBE_K = competitors-per-lane hint)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402

from paper_2108_02419_b200 import sim  # noqa: E402
from profile_cfg import field  # noqa: E402

name = sys.argv[1]
sims = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
state, cfg = field(name)
for i in range(reps):
    seeds = np.arange(1, sims + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15) + np.uint64(i)
    r = sim.simulate_batch(state, cfg, sims, mode="mt", seeds=seeds, ranks=False,
                           lanes_per_slot=int(os.environ.get("BBE_K", "0")))
    print(f"{name} mt launch {i}: {r.kernel_ms:.3f} ms (seed + race), ct={r.competitor_steps}", flush=True)
