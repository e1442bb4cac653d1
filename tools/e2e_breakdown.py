"""Where the time of one native rp_predict(d = 100k) call goes (C2): host steps around the kernel."""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_io import c2, config_from_dict, state_from_dict  # noqa: E402
from paper_2108_02419_b200.agents import dry_run_seeds, rp_predict  # noqa: E402
from paper_2108_02419_b200.sim import simulate_batch_begin  # noqa: E402

g = c2()
cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
d, n = 100_000, 10
rng = random.Random(11)
for _ in range(5):
    rp_predict(st, cfg, d, rng, mode="native")
acc = [0.0] * 6
R = 50
for _ in range(R):
    t0 = time.perf_counter()
    key = int(dry_run_seeds(rng, 1)[0])
    t1 = time.perf_counter()
    pending = simulate_batch_begin(st, cfg, d, key, mode="native", ranks=False)
    t2 = time.perf_counter()
    dry_run_seeds(rng, d - 1, want=False)
    t3 = time.perf_counter()
    res = pending.end()
    t4 = time.perf_counter()
    probs = tuple((int(w) + 1) / (d + n) for w in res.wins)
    t5 = time.perf_counter()
    for i, dt in enumerate((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t5 - t0)):
        acc[i] += dt
names = ("first seed", "begin (pack + H2D + launch)", "advance d-1 (overlaps)", "end (wait + D2H)", "probs", "total")
for name, a in zip(names, acc):
    print(f"{name:30s} {a / R * 1e6:8.1f} us")
print(f"kernel (events) {res.kernel_ms * 1e3:.1f} us")
