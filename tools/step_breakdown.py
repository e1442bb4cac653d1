"""What the bench's device step (C2, 100k sims) spends outside the race kernel: the step timed as in
bench.py (events around tally zeroing + bbe_simulate_async), and variants without the zeroing."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from golden_io import c2, config_from_dict, state_from_dict  # noqa: E402
from paper_2108_02419_b200 import sim  # noqa: E402

g = c2()
cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
L = sim.DeviceLauncher(st, cfg)
tally = torch.zeros(L.tally_len, dtype=torch.int64, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()


def run(zero: bool, reps: int = 60):
    ts, ks = [], []
    for i in range(reps):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        if zero:
            tally.zero_()
        L.launch(tally.data_ptr(), 100_000, 7 + i, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        ks.append(L.last_kernel_ms())
    return statistics.median(ts[5:]), statistics.median(ks[5:])


for zero in (True, False, True, False):
    t, k = run(zero)
    print(f"zero={zero}: step {t * 1e3:.1f} us, kernel {k * 1e3:.1f} us, outside {1e3 * (t - k):.1f} us")
