"""MT-mode throughput of one field under each competitors-per-lane layout (lanes_per_slot hint), from
the start line with run_batch's device-derived seeds; checks that every layout gives the same tallies.
usage: python tools/mt_layout_probe.py FIELD [sims]   (FIELD as profile_cfg.py)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from paper_2108_02419_b200 import sim  # noqa: E402
from profile_cfg import field  # noqa: E402

name = sys.argv[1]
sims = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1_000_000
state, cfg = field(name)
ref = None
for k in (0, 1, 2, 3, 4):
    if (len(cfg.competitors) + max(k, 1) - 1) // max(k, 1) > 32:
        continue
    best = None
    for r in range(3):
        res = sim.simulate_batch(state, cfg, sims, mode="mt", seed_master=20260818, lanes_per_slot=k)
        best = res.kernel_ms if best is None else min(best, res.kernel_ms)
    same = ref is None or (res.wins == ref.wins).all()
    ref = ref or res
    print(f"{name} mt K hint {k} (layout K={res.lanes_per_slot}): {best:.3f} ms, {sims / best / 1e3:.1f} M races/s, "
          f"{res.competitor_steps / best / 1e6:.1f} G ct/s, tallies equal: {same}", flush=True)
