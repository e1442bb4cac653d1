"""Launch one BASELINE workload a few times through a prepared race -- the command ncu profiles.

usage: python tools/profile_cfg.py FIELD MODE [sims] [reps]
  FIELD: c1 (5 x U(10,20) from the start), c2 (derby10 mid-race), c3 (20 x U(10,20) from the start),
         derby20 (derby.json resized to 20, from the start), c5 (= the c3 field)
  MODE:  native | native64
"""
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


def field(name):
    g = c2()
    derby10 = config_from_dict(g["config"])
    if name == "c2":
        return state_from_dict(g["state"]), derby10
    if name == "derby20":
        return None, resize_race(resize_race(derby10, 5), 20)
    if name.startswith("derby"):  # derbyN: derby.json resized to N, from the start line
        return None, resize_race(resize_race(derby10, 5), int(name[5:]))
    n = {"c1": 5, "c3": 20, "c5": 20}[name]
    return None, RaceConfig(2000.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(n)))


def main():
    name, mode = sys.argv[1], sys.argv[2]
    sims = int(float(sys.argv[3])) if len(sys.argv) > 3 else 100_000
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    state, cfg = field(name)
    L = sim.DeviceLauncher(state, cfg, native_mode=mode, lanes_per_slot=int(os.environ.get("BBE_K", "0")))
    tally = torch.zeros(L.tally_len, dtype=torch.int64, device="cuda")
    for i in range(reps):
        tally.zero_()
        L.launch(tally.data_ptr(), sims, 1000 + i, stream=torch.cuda.current_stream().cuda_stream, mode=mode)
        torch.cuda.synchronize()
        print(f"{name} {mode} launch {i}: {L.last_kernel_ms():.3f} ms, ct={int(tally[L.off['ct']])}, "
              f"blocked={int(tally[L.off['blocked']])}", flush=True)


if __name__ == "__main__":
    main()
