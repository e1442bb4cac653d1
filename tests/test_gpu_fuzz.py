"""Random-config parity fuzz (exact modes vs the oracle), in the spirit of the reference's randomized
termination criterion (tests/test_acceptance.py:70-123) but with its own generator: fields of 1..40
competitors, mixed step families, blocking thresholds, responsiveness and preference, short tracks.

For every config the MT kernel must reproduce the oracle race bit for bit from the start line
(run_race) and from a mid-race state (simulate_from), and the inject kernel must do the same from the
oracle's recorded draws.  Any K (competitors per lane) layout the field needs is exercised.
"""

import random

import numpy as np
import pytest

import oracle
from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.race import (
    Competitor,
    LogNormalSteps,
    RaceConfig,
    RaceState,
    Responsiveness,
    UniformSteps,
)

pytestmark = pytest.mark.gpu


def random_config(rng: random.Random) -> RaceConfig:
    n = rng.choice([1, 2, 3, 5, 7, 10, 13, 20, 31, 33, 40])
    comps = []
    for i in range(n):
        if rng.random() < 0.6:
            lo = rng.uniform(0.5, 6.0)
            steps = UniformSteps(lo, lo + rng.choice([0.0, rng.uniform(0.0, 6.0)]))
        else:
            steps = LogNormalSteps(rng.uniform(-0.5, 1.5), rng.uniform(0.0, 0.8), rng.uniform(0.3, 3.0))
        comps.append(Competitor(f"r{i}", steps, preference=rng.random(), pref_sensitivity=rng.uniform(0.0, 0.9),
                                theta=rng.choice([0.0, 0.0, rng.uniform(0.0, 6.0)]),
                                responsiveness=Responsiveness(rng.uniform(0.4, 1.6), rng.uniform(0.4, 1.6),
                                                              rng.random())))
    return RaceConfig(rng.uniform(15.0, 90.0), tuple(comps), conditions=rng.random())


def _same(r, i, o):
    assert r.order[i].tolist() == o.order.tolist()
    assert r.finish_ticks[i].tolist() == o.finish_ticks.tolist()
    assert r.final_positions[i].tolist() == o.final_positions.tolist()
    assert int(r.blocked[i]) == o.blocked


@pytest.mark.parametrize("block", range(4))
def test_random_configs_bit_exact(block):
    rng = random.Random(7000 + block)
    for _ in range(40):
        cfg = random_config(rng)
        n = cfg.n_competitors
        seeds = np.array([rng.getrandbits(64) for _ in range(3)], np.uint64)
        # from the start line: MT from the seeds, inject from the oracle's recorded draws
        r = sim.simulate_batch(None, cfg, 3, mode="mt", seeds=seeds, records=True)
        recs = [oracle.run_race(cfg, int(s), record=True) for s in seeds]
        for i, o in enumerate(recs):
            _same(r, i, o)
        offs = np.zeros(4, np.int64)
        offs[1:] = np.cumsum([o.draws_used for o in recs])
        r = sim.simulate_batch(None, cfg, 3, mode="inject", draws=np.concatenate([o.draws for o in recs]),
                               draw_offsets=offs, records=True)
        for i, o in enumerate(recs):
            _same(r, i, o)
        # from a mid-race state of the first race
        k = rng.randint(1, max(1, int(recs[0].n_ticks_run) - 1))
        tick, pos, prev, fin, _ = oracle.advance_from_start(cfg, int(seeds[0]), k)
        st = RaceState(tick, pos.tolist(), prev.tolist(), [None if f < 0 else int(f) for f in fin])
        if all(f is not None for f in st.finish_ticks):
            continue
        r = sim.simulate_batch(st, cfg, 3, mode="mt", seeds=seeds[::-1].copy(), records=True)
        for i, s in enumerate(seeds[::-1]):
            _same(r, i, oracle.simulate_from(st, cfg, int(s)))
        assert n == len(r.ids)


def random_degenerate_config(rng: random.Random) -> RaceConfig:
    """U(v, v) steps on a half-integer grid, responsiveness in {1, 2} (a blocked step never shrinks
    below the grid), no preference effect: every FP32 operation is exact, so native mode must equal
    the reference race bit for bit."""
    n = rng.choice([1, 2, 4, 6, 9, 10, 12, 17, 20, 24, 32, 40, 64])
    comps = tuple(
        Competitor(f"d{i}", UniformSteps(v, v), theta=rng.choice([0.0, 1.0, 2.5, 4.0]),
                   responsiveness=Responsiveness(rng.choice([1.0, 2.0]), rng.choice([1.0, 2.0]),
                                                 rng.choice([0.0, 0.25, 0.5, 1.0])))
        for i, v in enumerate(rng.choice([0.5, 1.0, 1.5, 2.0, 3.0, 4.5]) for _ in range(n)))
    return RaceConfig(float(rng.choice([24, 40, 64])), comps)


@pytest.mark.parametrize("block", range(2))
def test_random_degenerate_configs_native_exact(block):
    rng = random.Random(9100 + block)
    for _ in range(40):
        cfg = random_degenerate_config(rng)
        n = cfg.n_competitors
        o = oracle.run_race(cfg, 1)  # draws do not matter: U(v, v)
        for k in (0, 1, 2, 3, 4):
            if k and -(-n // k) > 32:
                continue
            r = sim.simulate_batch(None, cfg, 2, 5, records=True, lanes_per_slot=k)
            _same(r, 0, o)
        # mid-race, with state positions on the same grid
        pos = [rng.randint(0, 20) * 0.5 for _ in range(n)]
        st = RaceState(2, pos, [rng.randint(1, 8) * 0.5 for _ in range(n)], [None] * n)
        o = oracle.simulate_from(st, cfg, 1)
        r = sim.simulate_batch(st, cfg, 2, 5, records=True)
        _same(r, 0, o)
