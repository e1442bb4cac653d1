"""Launch the bench workload (C2, 100k continuations) a few times -- the command profiled by ncu.

usage: python tools/profile_c2.py [sims] [reps]     env: BBE_K (lanes-per-slot hint), BBE_MODE (native|mt)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from golden_io import c2, config_from_dict, state_from_dict  # noqa: E402
from paper_2108_02419_b200 import sim  # noqa: E402

sims = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mode = os.environ.get("BBE_MODE", "native")
g = c2()
cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
if mode == "native":
    L = sim.DeviceLauncher(st, cfg, lanes_per_slot=int(os.environ.get("BBE_K", "0")))
    tally = torch.zeros(L.tally_len, dtype=torch.int64, device="cuda")
    for i in range(reps):
        tally.zero_()
        L.launch(tally.data_ptr(), sims, 1000 + i, stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        print(f"launch {i}: {L.last_kernel_ms():.3f} ms, ct={int(tally[L.off['ct']])}")
else:
    for i in range(reps):
        seeds = np.arange(1, sims + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15) + np.uint64(i)
        r = sim.simulate_batch(st, cfg, sims, mode=mode, seeds=seeds, ranks=False)
        print(f"launch {i}: {r.kernel_ms:.3f} ms (seed + race kernels), ct={r.competitor_steps}")
