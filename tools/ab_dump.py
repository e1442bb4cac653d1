"""Dump per-sim native/MT results of a C2 batch and a from-start derby20 batch (A/B builds must be
bit-identical when they only change the schedule): python tools/ab_dump.py OUT.npz [mode]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from golden_io import c2, config_from_dict, state_from_dict  # noqa: E402
from paper_2108_02419_b200 import sim  # noqa: E402
from paper_2108_02419_b200.batch import resize_race  # noqa: E402

mode = sys.argv[2] if len(sys.argv) > 2 else "native"
g = c2()
cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
kw = dict(seeds=np.arange(1, 30_001, dtype=np.uint64)) if mode == "mt" else {}
r = sim.simulate_batch(st, cfg, 30_000, 77, mode=mode, records=True, **kw)
cfg20 = resize_race(cfg, 20)
r2 = sim.simulate_batch(None, cfg20, 20_000, 78, mode=mode, records=True,
                        **(dict(seeds=np.arange(5, 20_005, dtype=np.uint64)) if mode == "mt" else {}))
np.savez(sys.argv[1], order=r.order, fin=r.finish_ticks, pos=r.final_positions, wins=r.wins, ranks=r.ranks,
         ct=r.competitor_steps, blk=r.blocked_steps, order2=r2.order, fin2=r2.finish_ticks, pos2=r2.final_positions)
print("dumped", sys.argv[1], r.competitor_steps, r2.competitor_steps)
