"""Device time of NATIVE (FP32 state) vs NATIVE64 (FP64 state) on the BASELINE configs (CUDA events
around prepared launches; one warm-up each).  Usage: python tools/n64_timing.py [--c5 1e8]"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from golden_io import c2, config_from_dict, state_from_dict  # noqa: E402
from paper_2108_02419_b200 import sim  # noqa: E402
from paper_2108_02419_b200.batch import resize_race  # noqa: E402
from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps  # noqa: E402


def uniform_field(n):
    return RaceConfig(2000.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(n)))


def time_launch(state, cfg, n_sims, mode, reps=3, lanes=0):
    L = sim.DeviceLauncher(state, cfg, native_mode=mode, lanes_per_slot=lanes)
    t = torch.zeros(L.tally_len, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    L.launch(t.data_ptr(), min(n_sims, 200_000), 1, stream=s, mode=mode)
    torch.cuda.synchronize()
    best = None
    for r in range(reps):
        t.zero_()
        L.launch(t.data_ptr(), n_sims, 2 + r, stream=s, mode=mode)
        ms = L.last_kernel_ms()
        best = ms if best is None else min(best, ms)
    ct = int(t[L.off["ct"]].item())
    return best, ct


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c5", type=float, default=1e8)
    ap.add_argument("--lanes", type=int, default=0)
    args = ap.parse_args()
    g = c2()
    derby10 = config_from_dict(g["config"])
    st = state_from_dict(g["state"])
    runs = [("C1 5xU 1e6", None, uniform_field(5), 10**6),
            ("C2 derby10 mid 1e5", st, derby10, 10**5),
            ("C2 derby10 mid 1e6", st, derby10, 10**6),
            ("C3 20xU 1e7", None, uniform_field(20), 10**7),
            ("C5 20xU", None, uniform_field(20), int(args.c5)),
            ("derby20 1e6", None, resize_race(resize_race(derby10, 5), 20), 10**6)]
    for name, state, cfg, n in runs:
        row = [name]
        for mode in ("native", "native64"):
            ms, ct = time_launch(state, cfg, n, mode, lanes=args.lanes)
            row.append(f"{mode}: {ms:8.3f} ms {ct / ms / 1e9:7.3f} Tct/s {n / ms / 1e3:9.1f} Mraces/s")
        print(" | ".join(row), flush=True)


if __name__ == "__main__":
    main()
