"""Native kernel time vs race length, for the ticks-per-block choice (pick_ticks in bbe_sim.cu).
Run once per BBE_TICKS value (4, 8, 16; unset = the automatic choice):
  for t in 4 8 16 auto; do BBE_TICKS=$t python tools/ticks_sweep.py $t; done"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from golden_io import c2, config_from_dict  # noqa: E402
from paper_2108_02419_b200 import sim  # noqa: E402
from paper_2108_02419_b200.batch import resize_race  # noqa: E402
from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps  # noqa: E402

derby = config_from_dict(c2()["config"])
row = []
for field in ("5xU", "derby10", "20xU"):
    for L in (100.0, 250.0, 500.0, 1000.0, 2000.0, 4000.0):
        if field == "derby10":
            cfg = RaceConfig(L, resize_race(derby, 10).competitors)
        else:
            n = 5 if field == "5xU" else 20
            cfg = RaceConfig(L, tuple(Competitor(f"c{i}", UniformSteps(10.0, 20.0)) for i in range(n)))
        sims = int(4e8 / (L * (5 if field == "5xU" else 10 if field == "derby10" else 20)))
        Lh = sim.DeviceLauncher(None, cfg)
        tally = torch.zeros(Lh.tally_len, dtype=torch.int64, device="cuda")
        ts = []
        for i in range(7):
            tally.zero_()
            Lh.launch(tally.data_ptr(), sims, 100 + i, stream=torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            ts.append(Lh.last_kernel_ms())
        ct = int(tally[Lh.off["ct"]])
        row.append(f"{field} L={int(L)}: {ct / (statistics.median(ts[2:]) * 1e-3) / 1e9:.0f} Gct/s")
print(sys.argv[1] if len(sys.argv) > 1 else "", " | ".join(row))
