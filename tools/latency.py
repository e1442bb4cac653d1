"""Per-call latency of the public API (rp_predict) for small and large d, both modes.

usage: python tools/latency.py [reps]
"""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_io import c2, config_from_dict, state_from_dict  # noqa: E402
from paper_2108_02419_b200.agents import rp_predict  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
g = c2()
cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
for mode in ("native", "mt"):
    for d in (1, 64, 1000, 10000, 100000):
        rng = random.Random(5)
        r = max(3, reps if d <= 10000 else reps // 10)
        for _ in range(3):
            rp_predict(st, cfg, d, rng, mode=mode)
        t0 = time.perf_counter()
        for _ in range(r):
            rp_predict(st, cfg, d, rng, mode=mode)
        dt = (time.perf_counter() - t0) / r
        print(f"{mode:6s} d={d:6d}: {dt * 1e6:9.1f} us/call  {d / dt / 1e6:8.2f} M races/s")
