"""Rank-marginal diagnostic for a 40-runner derby field: native tallies of every layout K against a
200k-race oracle batch, and the mean rank of exchangeable siblings (same template)."""
import sys, math
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
import oracle
from golden_io import c2, config_from_dict
from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.race import Competitor, RaceConfig
g = c2(); base = config_from_dict(g["config"])
n = 40
comps = tuple(Competitor(f"c{i + 1}", base.competitors[i % 5].steps, base.competitors[i % 5].preference,
                         base.competitors[i % 5].pref_sensitivity, base.competitors[i % 5].theta,
                         base.competitors[i % 5].responsiveness) for i in range(n))
cfg = RaceConfig(2000.0, comps, conditions=base.conditions)
ref = oracle.batch(cfg, 200_000, master=424242, threads=16)
rr = ref["ranks"] / 200_000
for k in (2, 3, 4):
    res = sim.simulate_batch(None, cfg, 2_000_000, 987654321 + k, lanes_per_slot=k)
    rg = res.ranks / 2_000_000
    se = np.sqrt(np.maximum(rr * (1 - rr), 1e-12) * (1 / 200_000 + 1 / 2_000_000))
    z = np.abs(rg - rr) / se
    i, j = np.unravel_index(np.argmax(z), z.shape)
    print(f"K={k}: max z {z.max():.2f} at competitor {i} rank {j}: gpu {rg[i, j]:.5f} ref {rr[i, j]:.5f}; "
          f"win max z {np.max(np.abs(rg[:, 0] - rr[:, 0]) / se[:, 0]):.2f}; mean ct gpu {res.competitor_steps / 2e6:.2f} ref {ref['ct'] / 2e5:.2f}")
    # exchangeable siblings of template 0 (c0, c5, ..., c35): mean rank
    sib = [c for c in range(n) if c % 5 == 0]
    mr = (rg[sib] * np.arange(n)).sum(axis=1)
    print("   mean rank of template-0 siblings gpu:", np.round(mr, 3))
mr = (rr[[c for c in range(n) if c % 5 == 0]] * np.arange(n)).sum(axis=1)
print("   mean rank of template-0 siblings ref:", np.round(mr, 3))
