"""Where the time of one MT-exact rp_predict(d = 100k) call goes (C2): host seed stream, the call
(seed H2D + seeding + race kernels + tally D2H), device time."""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from golden_io import c2, config_from_dict, state_from_dict  # noqa: E402
from paper_2108_02419_b200.agents import dry_run_seeds, rp_predict  # noqa: E402
from paper_2108_02419_b200.sim import simulate_batch  # noqa: E402

g = c2()
cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
d = 100_000
rng = random.Random(11)
for _ in range(3):
    rp_predict(st, cfg, d, rng)
R = 20
acc = np.zeros(4)
for _ in range(R):
    t0 = time.perf_counter()
    seeds = dry_run_seeds(rng, d)
    t1 = time.perf_counter()
    res = simulate_batch(st, cfg, d, mode="mt", seeds=seeds, ranks=False)
    t2 = time.perf_counter()
    acc += (t1 - t0, t2 - t1, t2 - t0, res.kernel_ms / 1e3)
t0 = time.perf_counter()
for _ in range(R):
    rp_predict(st, cfg, d, rng)
t_rp = (time.perf_counter() - t0) / R
for name, a in zip(("seeds (host MT, 800 KB out)", "simulate_batch (H2D + kernels + D2H)", "sum", "kernels (events)"), acc):
    print(f"{name:40s} {a / R * 1e3:8.3f} ms")
print(f"{'rp_predict(mode=mt)':40s} {t_rp * 1e3:8.3f} ms")
