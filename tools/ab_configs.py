"""Native kernel time (median of 7 launches, CUDA events) on the bench's configs, for A/B builds:
BBE_LIB=... python tools/ab_configs.py TAG"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from golden_io import c2, config_from_dict, state_from_dict  # noqa: E402
from paper_2108_02419_b200 import sim  # noqa: E402
from paper_2108_02419_b200.batch import resize_race  # noqa: E402
from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps  # noqa: E402

g = c2()
cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])


def uni(n):
    return RaceConfig(2000.0, tuple(Competitor(f"c{i}", UniformSteps(10.0, 20.0)) for i in range(n)))


cases = [("C2 derby10 mid-race 1e5", st, cfg, 100_000), ("C1 5xU from start 1e6", None, uni(5), 1_000_000),
         ("C3 20xU from start 1e6", None, uni(20), 1_000_000),
         ("derby20 from start 1e6", None, resize_race(cfg, 20), 1_000_000),
         ("derby5 from start 1e6", None, resize_race(cfg, 5), 1_000_000)]
out = []
for name, s0, c, ns in cases:
    L = sim.DeviceLauncher(s0, c)
    tally = torch.zeros(L.tally_len, dtype=torch.int64, device="cuda")
    ts = []
    for i in range(9):
        tally.zero_()
        L.launch(tally.data_ptr(), ns, 100 + i, stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        ts.append(L.last_kernel_ms())
    out.append(f"{name}: {statistics.median(ts[2:]):.3f} ms")
print(sys.argv[1] if len(sys.argv) > 1 else "", " | ".join(out))
