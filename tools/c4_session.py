"""Time the C4 dry-run session (100 RP bettors, every wake predicting with d dry runs) per mode.

usage: python tools/c4_session.py [d ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_io import c2, config_from_dict  # noqa: E402
from paper_2108_02419_b200.batch import resize_race  # noqa: E402
from paper_2108_02419_b200.session import run_dry_run_session  # noqa: E402

derby5 = resize_race(config_from_dict(c2()["config"]), 5)
for d in [int(x) for x in sys.argv[1:]] or [1000]:
    for mode in ("mt", "native"):
        run_dry_run_session(derby5, n_agents=100, d=d, master_seed=20260818, opening_period=5.0, mode=mode)
        r = run_dry_run_session(derby5, n_agents=100, d=d, master_seed=20260818, opening_period=5.0, mode=mode)
        print(f"d={d} {mode}: {r.launches} launches, {r.sims} sims, {r.seconds:.3f} s, "
              f"{r.sims_per_second / 1e6:.1f} M races/s")
