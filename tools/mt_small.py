"""Small MT-exact rp_predict calls (d = 64 and 1) -- the command behind the per-launch latency list."""
import sys, random; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from golden_io import c2, config_from_dict, state_from_dict
from paper_2108_02419_b200.agents import rp_predict
g=c2(); cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
rng=random.Random(3)
for _ in range(4): rp_predict(st, cfg, 64, rng, mode="mt")
for _ in range(4): rp_predict(st, cfg, 1, rng, mode="mt")
