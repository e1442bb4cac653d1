"""MT-exact throughput on a uniform-only field (C1: 5 x U(10,20), L=2000, from the start) and on C2."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_io import c2, config_from_dict, state_from_dict  # noqa: E402
from paper_2108_02419_b200 import sim  # noqa: E402
from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps  # noqa: E402

c1 = RaceConfig(2000.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(5)))
g = c2()
cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
for name, state, conf, n in (("C1 mt 100k", None, c1, 100_000), ("C2 mt 100k", st, cfg, 100_000)):
    for i in range(4):
        r = sim.simulate_batch(state, conf, n, mode="mt", seed_master=20260818 + i, ranks=False)
    print(f"{name}: {r.kernel_ms:.3f} ms device (seed + race), {n / r.kernel_ms / 1e3:.1f} M races/s, "
          f"{r.competitor_steps / r.kernel_ms / 1e6:.1f} G ct/s")
