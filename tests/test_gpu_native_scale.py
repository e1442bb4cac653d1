"""Native-RNG parity at the BASELINE configs' scale (north_star: "in native-RNG mode, win
probabilities must agree with the reference's within stated binomial confidence bounds").

MT mode is bit-identical to the reference (tests/test_gpu_mt.py, test_gpu_fuzz.py,
test_session_exchange.py), so 10^7 MT sims ARE 10^7 reference sims.  Against them, 10^8 sims of each
Philox mode -- NATIVE64 (FP64 state, the bench headline) and NATIVE (FP32 state) -- on the metric's
fields:
  C1  5 x U(10,20), L = 2000, from the start line (BASELINE configs[0]; config.py:433-443)
  C3  20 x U(10,20), L = 2000, from the start line (configs[2] and the C5 field of configs[4])
  derby20  derby.json resized to 20 (blocking, lognormal, closers), from the start line
  C2  derby10 mid-race (tick 65) continuation (configs[1])
  lognormal8  every runner lognormal (Box-Muller vs the reference's Kinderman-Monahan), from the start
  blocking12  every runner blocking (theta = 6), from the start
Tests: two-sample binomial z on every win probability and every rank-marginal cell, Bonferroni over
all cells of the file at alpha = 0.01 (tests/test_acceptance.py:394-424 calibrates the same way), and
a z test on the mean race length in competitor-timesteps (variance from a recorded MT subsample).

Scale probe (C5 field, 10^9 vs 10^9): NATIVE (FP32 state, 23-bit draws) against NATIVE64 -- the
binomial standard error of a difference is ~1e-5 there, the tightest bound any BASELINE config sets;
FP32 bias (position rounding near L = 2000, the overshoot tie-break, 23-bit uniforms) must stay below it.
Set BBE_REPORT=path to write the measured differences as JSON (DESIGN.md §2 quotes them).
"""

import json
import math
import os

import numpy as np
import pytest
from scipy.stats import norm

from golden_io import c2, config_from_dict, state_from_dict
from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.batch import resize_race
from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps

pytestmark = pytest.mark.gpu

N_NAT = 10**8
N_MT = 10**7
N_PROBE = 10**9
ALPHA = 0.01
REPORT = {}


def uniform_field(n):
    return RaceConfig(2000.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(n)))


def lognormal_field(n=8):
    """Every runner lognormal (the Box-Muller law of the Philox modes against the reference's
    Kinderman-Monahan normalvariate), mixed mu / sigma / scale, a few blockers."""
    from paper_2108_02419_b200.race import LogNormalSteps

    comps = tuple(Competitor(f"l{i}", LogNormalSteps(2.3 + 0.05 * i, 0.15 + 0.04 * (i % 4), 1.0 + 0.1 * (i % 3)),
                             theta=6.0 if i % 3 == 0 else 0.0) for i in range(n))
    return RaceConfig(1500.0, comps)


def blocking_field(n=12):
    """Every runner blocks (theta = 6): the front-runner scan and blocked steps on every tick."""
    return RaceConfig(1200.0, tuple(Competitor(f"b{i}", UniformSteps(9.0 + 0.3 * i, 16.0), theta=6.0,
                                               preference=0.1 * (i % 10), pref_sensitivity=0.3)
                                    for i in range(n)), conditions=0.4)


def fields():
    g = c2()
    derby10 = config_from_dict(g["config"])
    return {"C1": (None, uniform_field(5)), "C3": (None, uniform_field(20)),
            "derby20": (None, resize_race(resize_race(derby10, 5), 20)),
            "C2": (state_from_dict(g["state"]), derby10),
            "lognormal8": (None, lognormal_field()), "blocking12": (None, blocking_field())}


# every cell tested in this file: per field and mode, n wins + n^2 rank cells + 1 mean-ct test; plus
# the probe's 20 + 400 cells
_N_TESTS = sum(2 * (len(c.competitors) + len(c.competitors) ** 2 + 1) for _, c in fields().values()) + 420
CRIT = norm.ppf(1 - ALPHA / (2 * _N_TESTS))


def z_two_sample(a, na, b, nb):
    p = (a + b) / (na + nb)
    if min(p, 1 - p) * min(na, nb) < 10:
        return 0.0  # too rare for the normal approximation
    return abs(a / na - b / nb) / math.sqrt(p * (1 - p) * (1 / na + 1 / nb))


def compare_tallies(x, nx, y, ny, n):
    zs = [z_two_sample(int(x.wins[c]), nx, int(y.wins[c]), ny) for c in range(n)]
    zr = [z_two_sample(int(x.ranks[c, r]), nx, int(y.ranks[c, r]), ny) for c in range(n) for r in range(n)]
    dp = max(abs(int(x.wins[c]) / nx - int(y.wins[c]) / ny) for c in range(n))
    return max(zs), max(zr), dp


@pytest.fixture(scope="module")
def mt_runs():
    out = {}
    for i, (name, (state, cfg)) in enumerate(fields().items()):
        mt = sim.simulate_batch(state, cfg, N_MT, mode="mt", seed_master=20260818 + i)
        rec = sim.simulate_batch(state, cfg, 100_000, mode="mt", seed_master=777 + i, records=True, ranks=False)
        t0 = 0 if state is None else state.tick
        racing = np.array([f is None for f in (state.finish_ticks if state else [None] * cfg.n_competitors)])
        ct_per_sim = ((rec.finish_ticks - t0) * racing[None, :]).sum(axis=1)
        out[name] = (mt, float(ct_per_sim.std()))
    return out


@pytest.mark.parametrize("mode", ["native64", "native"])
@pytest.mark.parametrize("name", ["C1", "C3", "derby20", "C2", "lognormal8", "blocking12"])
def test_native_modes_match_reference_stream_at_scale(mt_runs, name, mode):
    state, cfg = fields()[name]
    n = cfg.n_competitors
    mt, ct_sd = mt_runs[name]
    nat = sim.simulate_batch(state, cfg, N_NAT, 4242 + n, mode=mode)
    assert int(nat.wins.sum()) == N_NAT and int(mt.wins.sum()) == N_MT
    zw, zr, dp = compare_tallies(nat, N_NAT, mt, N_MT, n)
    m_nat, m_mt = nat.competitor_steps / N_NAT, mt.competitor_steps / N_MT
    z_ct = abs(m_nat - m_mt) / (ct_sd * math.sqrt(1 / N_NAT + 1 / N_MT)) if ct_sd > 0 else 0.0
    REPORT[f"{name}/{mode}"] = {"max_z_wins": zw, "max_z_ranks": zr, "max_abs_dp_win": dp, "z_mean_ct": z_ct,
                               "mean_ct": [m_nat, m_mt], "crit": CRIT, "n": [N_NAT, N_MT]}
    assert zw <= CRIT, f"{name} {mode}: win |z| {zw:.2f} > {CRIT:.2f}"
    assert zr <= CRIT, f"{name} {mode}: rank |z| {zr:.2f} > {CRIT:.2f}"
    assert z_ct <= CRIT, f"{name} {mode}: mean ct {m_nat} vs {m_mt} (|z| {z_ct:.2f})"


def test_fp32_state_bias_below_binomial_error_at_1e9():
    """C5 field at 10^9 sims per mode: FP32-state NATIVE vs FP64-state NATIVE64."""
    cfg = uniform_field(20)
    a = sim.simulate_batch(None, cfg, N_PROBE, 99, mode="native")
    b = sim.simulate_batch(None, cfg, N_PROBE, 99, mode="native64")
    zw, zr, dp = compare_tallies(a, N_PROBE, b, N_PROBE, 20)
    p = float(b.wins.max()) / N_PROBE
    se = math.sqrt(2 * p * (1 - p) / N_PROBE)
    REPORT["C5_probe/native_vs_native64"] = {"max_z_wins": zw, "max_z_ranks": zr, "max_abs_dp_win": dp,
                                             "se_diff_at_max_p": se, "crit": CRIT, "n": [N_PROBE, N_PROBE],
                                             "ct_per_race": [a.competitor_steps / N_PROBE, b.competitor_steps / N_PROBE]}
    assert zw <= CRIT and zr <= CRIT, (zw, zr)


def teardown_module(module):
    path = os.environ.get("BBE_REPORT")
    if path and REPORT:
        with open(path, "w") as fh:
            json.dump(REPORT, fh, indent=1)
