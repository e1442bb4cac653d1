"""Time rp_predict(mode='native') at the bench workload (C2, d = 100k): median of 200 calls."""
import os
import random
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_io import c2, config_from_dict, state_from_dict  # noqa: E402
from paper_2108_02419_b200 import sim  # noqa: E402
from paper_2108_02419_b200.agents import rp_predict  # noqa: E402

g = c2()
cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
rng = random.Random(11)
for d in (100_000, 1_000):
    for _ in range(20):
        rp_predict(st, cfg, d, rng, mode="native")
    ts = []
    for _ in range(200):
        t0 = time.perf_counter()
        rp_predict(st, cfg, d, rng, mode="native")
        ts.append(time.perf_counter() - t0)
    k = sim.simulate_batch(st, cfg, d, 5, ranks=False).kernel_ms
    print(f"d={d}: rp_predict native median {statistics.median(ts) * 1e6:.1f} us, min {min(ts) * 1e6:.1f} us; "
          f"kernel {k * 1e3:.1f} us")
