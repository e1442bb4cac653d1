"""Time every competitors-per-lane layout K for a range of field sizes (native, from the start line,
L = 2000): the data behind bbe_sim.cu choose_k.

usage: python tools/k_sweep.py [sims]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402
from golden_io import c2, config_from_dict  # noqa: E402

from paper_2108_02419_b200 import sim  # noqa: E402
from paper_2108_02419_b200.batch import resize_race  # noqa: E402
from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps  # noqa: E402

sims = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
derby10 = config_from_dict(c2()["config"])
stream = torch.cuda.current_stream()
print("| field | n | " + " | ".join(f"K={k} ms" for k in (1, 2, 3, 4)) + " | auto K |")
print("|---|---|---|---|---|---|---|")
for kind in ("uniform", "derby"):
    for n in [int(x) for x in os.environ.get("K_SWEEP_N", "").split(",") if x] or (6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 20, 21, 24, 28, 32, 33, 40, 48, 64, 96, 128):
        if kind == "uniform":
            cfg = RaceConfig(2000.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(n)))
        else:
            cfg = resize_race(derby10, n)
        cells = []
        for k in (1, 2, 3, 4):
            if -(-n // k) > 32:
                cells.append("-")
                continue
            dl = sim.DeviceLauncher(None, cfg, lanes_per_slot=k)
            tally = torch.zeros(dl.tally_len, dtype=torch.int64, device="cuda")
            dl.launch(tally.data_ptr(), min(sims, 50_000), 1, stream=stream.cuda_stream)
            best = 1e9
            for rep in range(2):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                dl.launch(tally.data_ptr(), sims, 2 + rep, stream=stream.cuda_stream)
                e1.record(stream)
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            cells.append(f"{best:.2f}")
        r = sim.simulate_batch(None, cfg, 1000, 1, ranks=False)
        print(f"| {kind} | {n} | " + " | ".join(cells) + f" | {r.lanes_per_slot} |", flush=True)
