"""C3 roofline sweep: races/s, ct/s and issue-roofline fraction of the NATIVE (FP32
state) or NATIVE64 (FP64 state) kernel over competitor count n and track length L, from the start line.

Fields: `uniform` = n x U(10, 20) (theta = 0: no front-runner scan), `derby` = derby.json resized to
n (blocking theta = 8 runners, lognormal runners).  Writes a markdown table to stdout.

usage: python tools/sweep.py [sims] [native|native64]
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

PEAK = 148 * 128 * 1.965e9  # lane-ops/s (bench.py: MEASURED_PEAKS sm_max_mhz)
sims = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
mode = sys.argv[2] if len(sys.argv) > 2 else "native"
derby10 = config_from_dict(c2()["config"])


def ops_per_ct(n, f_free, scan):
    # bench.py ops_per_ct: a draw is one Philox word (+2) in FP32 state, two (+4) in FP64 state
    return (4 * (n - 1) if scan else 0) + 13 + (44 if mode == "native64" else 22) * f_free


def field(kind, n, L):
    if kind == "uniform":
        return RaceConfig(L, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(n)))
    base = resize_race(derby10, n)
    return RaceConfig(L, base.competitors, conditions=base.conditions)


stream = torch.cuda.current_stream()
print(f"# {mode} kernel sweep: {sims:,} races from the start line per point (B200, CUDA events)\n")
print("| field | n | L | ms | M races/s | G ct/s | roofline frac |")
print("|---|---|---|---|---|---|---|")
for kind in ("uniform", "derby"):
    for n in (2, 3, 4, 5, 8, 10, 12, 16, 20, 24, 32, 40):
        for L in (250.0, 500.0, 1000.0, 2000.0, 4000.0):
            cfg = field(kind, n, L)
            dl = sim.DeviceLauncher(None, cfg, native_mode=mode)
            tally = torch.zeros(dl.tally_len, dtype=torch.int64, device="cuda")
            dl.launch(tally.data_ptr(), min(sims, 100_000), 1, stream=stream.cuda_stream, mode=mode)
            torch.cuda.synchronize()
            tally.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dl.launch(tally.data_ptr(), sims, 2, stream=stream.cuda_stream, mode=mode)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            t = tally.cpu()
            ct, blocked = int(t[dl.off["ct"]]), int(t[dl.off["blocked"]])
            scan = any(c.theta > 0 for c in cfg.competitors)
            frac = ct * ops_per_ct(n, 1 - blocked / ct, scan) / (ms / 1e3) / PEAK
            print(f"| {kind} | {n} | {L:.0f} | {ms:.2f} | {sims / ms / 1e3:.1f} | {ct / ms / 1e6:.1f} | {frac:.3f} |")
