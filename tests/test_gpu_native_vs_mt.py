"""The Philox modes (NATIVE, NATIVE64) against MT mode on random configs at GPU scale.

MT mode is bit-identical to the reference (tests/test_gpu_mt.py, test_gpu_fuzz.py), so it stands in
for the reference at sample sizes the CPU cannot reach.  For each random field (mixed step families,
blocking, responsiveness, preferences; n up to 40, every lane layout) the native win probabilities
must agree with MT's within binomial bounds (two-sample z, Bonferroni over every competitor of every
config, alpha = 0.01), and so must the mean race length in competitor-timesteps.
"""

import math
import random

import numpy as np
import pytest
from scipy.stats import norm

from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.race import Competitor, LogNormalSteps, RaceConfig, Responsiveness, UniformSteps

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["native", "native64"], autouse=True)
def philox_mode(request, monkeypatch):
    """Both Philox modes (FP32 and FP64 state): simulate_batch calls without an explicit mode run in it."""
    orig = sim.simulate_batch

    def simulate_batch(*args, **kwargs):
        kwargs.setdefault("mode", request.param)
        return orig(*args, **kwargs)

    monkeypatch.setattr(sim, "simulate_batch", simulate_batch)
    return request.param


def random_field(rng: random.Random) -> RaceConfig:
    n = rng.choice([2, 3, 5, 8, 10, 12, 17, 20, 33, 40])
    comps = []
    for i in range(n):
        if rng.random() < 0.7:
            lo = rng.uniform(5.0, 12.0)
            steps = UniformSteps(lo, lo + rng.uniform(2.0, 10.0))
        else:
            steps = LogNormalSteps(rng.uniform(1.8, 2.6), rng.uniform(0.1, 0.4), 1.0)
        comps.append(Competitor(f"r{i}", steps, preference=rng.random(), pref_sensitivity=rng.uniform(0.0, 0.6),
                                theta=rng.choice([0.0, 0.0, rng.uniform(2.0, 9.0)]),
                                responsiveness=Responsiveness(rng.uniform(0.8, 1.2), rng.uniform(0.8, 1.2),
                                                              rng.random())))
    return RaceConfig(rng.uniform(300.0, 1500.0), tuple(comps), conditions=rng.random())


def test_native_matches_mt_on_random_fields():
    rng = random.Random(4242)
    configs = [random_field(rng) for _ in range(16)]
    total_k = sum(c.n_competitors for c in configs)
    crit = norm.ppf(1 - 0.01 / (2 * total_k))
    n_nat, n_mt = 1_000_000, 100_000
    for idx, cfg in enumerate(configs):
        nat = sim.simulate_batch(None, cfg, n_nat, 1000 + idx, ranks=False)
        mt = sim.simulate_batch(None, cfg, n_mt, mode="mt", seed_master=2000 + idx, ranks=False)
        for c in range(cfg.n_competitors):
            a, b = int(nat.wins[c]), int(mt.wins[c])
            p = (a + b) / (n_nat + n_mt)
            if min(p, 1 - p) * n_mt < 10:
                continue  # too rare (or too certain) for the normal approximation
            z = abs(a / n_nat - b / n_mt) / math.sqrt(p * (1 - p) * (1 / n_nat + 1 / n_mt))
            assert z <= crit, f"config {idx} (n={cfg.n_competitors}) competitor {c}: |z| {z:.2f} > {crit:.2f}"
        ct_nat, ct_mt = nat.competitor_steps / n_nat, mt.competitor_steps / n_mt
        assert abs(ct_nat - ct_mt) / ct_mt < 0.002, (idx, ct_nat, ct_mt)
    assert np.isfinite(crit)


def test_native_matches_mt_from_mid_race_states():
    """The same comparison for continuations (simulate_from / rp_predict): mid-race states taken from
    a recorded MT race of each field."""
    from paper_2108_02419_b200.race import RaceState

    rng = random.Random(777)
    cases = []
    for _ in range(12):
        cfg = random_field(rng)
        traj, prevs = sim.run_race(cfg, rng.getrandbits(64), record=True, with_prev_steps=True)
        t = max(1, int(traj.n_ticks * rng.uniform(0.3, 0.8)))
        st = RaceState(t, list(traj.ticks[t]), [float(x) for x in prevs[t]],
                       [f if f <= t else None for f in traj.finish_ticks])
        if all(f is not None for f in st.finish_ticks):
            continue
        cases.append((cfg, st))
    total_k = sum(c.n_competitors for c, _ in cases)
    crit = norm.ppf(1 - 0.01 / (2 * total_k))
    n_nat, n_mt = 1_000_000, 100_000
    for idx, (cfg, st) in enumerate(cases):
        nat = sim.simulate_batch(st, cfg, n_nat, 3000 + idx, ranks=False)
        mt = sim.simulate_batch(st, cfg, n_mt, mode="mt", seed_master=4000 + idx, ranks=False)
        for c in range(cfg.n_competitors):
            a, b = int(nat.wins[c]), int(mt.wins[c])
            p = (a + b) / (n_nat + n_mt)
            if min(p, 1 - p) * n_mt < 10:
                continue
            z = abs(a / n_nat - b / n_mt) / math.sqrt(p * (1 - p) * (1 / n_nat + 1 / n_mt))
            assert z <= crit, f"case {idx} (n={cfg.n_competitors}, tick {st.tick}) competitor {c}: |z| {z:.2f}"
        ct_nat, ct_mt = nat.competitor_steps / n_nat, mt.competitor_steps / n_mt
        assert abs(ct_nat - ct_mt) / ct_mt < 0.003, (idx, ct_nat, ct_mt)
