"""The Philox kernels -- NATIVE (FP32 state) and NATIVE64 (FP64 state, the bench headline; every test
runs once per mode): exact where the reference is RNG-independent, statistically equal to the
reference elsewhere, and reproducible under any sharding of the simulation index range.

Statistical bar (north star): per-competitor win probabilities agree with the reference's within
binomial confidence bounds -- two-sample z-test, Bonferroni over competitors, alpha = 0.01 -- and the
full finish-order PMF passes the reference's own chi-square homogeneity test (batch.py:181-203) for
n <= 6, mirroring acceptance criterion 10 (tests/test_acceptance.py:394-424).
"""

import math

import numpy as np
import pytest
from scipy.stats import chi2_contingency, norm

import oracle
from golden_io import c2, config_from_dict, state_from_dict
from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.agents import rp_predict
from paper_2108_02419_b200.race import (
    Competitor,
    LogNormalSteps,
    RaceConfig,
    RaceState,
    Responsiveness,
    UniformSteps,
)

pytestmark = pytest.mark.gpu
ALPHA = 0.01


@pytest.fixture(params=["native", "native64"], autouse=True)
def philox_mode(request, monkeypatch):
    """Every test of this module once per Philox mode: simulate_batch calls without an explicit mode
    run in this one."""
    orig = sim.simulate_batch

    def simulate_batch(*args, **kwargs):
        kwargs.setdefault("mode", request.param)
        return orig(*args, **kwargs)

    monkeypatch.setattr(sim, "simulate_batch", simulate_batch)
    return request.param


def binomial_agreement(wins_a, n_a, wins_b, n_b, alpha=ALPHA, min_expected=10):
    """Two-sample z-test per competitor, Bonferroni over competitors; returns (ok, max |z|, crit).

    Cells whose pooled rate predicts fewer than ``min_expected`` counts in the smaller sample are
    skipped: the normal approximation does not hold there (rare ranks of large fields)."""
    k = len(wins_a)
    crit = norm.ppf(1 - alpha / (2 * k))
    zmax = 0.0
    for wa, wb in zip(wins_a, wins_b):
        pa, pb = wa / n_a, wb / n_b
        p = (wa + wb) / (n_a + n_b)
        if p * min(n_a, n_b) < min_expected:
            continue
        se = math.sqrt(max(p * (1 - p), 1e-300) * (1 / n_a + 1 / n_b))
        z = 0.0 if se == 0 else abs(pa - pb) / se
        zmax = max(zmax, z)
    return zmax <= crit, zmax, crit


def test_degenerate_races_exact_in_native_mode():
    fixed = lambda v: UniformSteps(v, v)  # noqa: E731
    a, b = Competitor("c1", fixed(11.0)), Competitor("c2", fixed(12.0))
    res = sim.simulate_batch(None, RaceConfig(22.0, (a, b)), 64, 3, records=True)
    assert (res.order == [1, 0]).all() and (res.finish_ticks == [2, 2]).all()
    cfg2 = RaceConfig(22.0, (Competitor("c1", fixed(11.0)), Competitor("c2", fixed(11.0))))
    res = sim.simulate_batch(None, cfg2, 64, 3, records=True)
    assert (res.order == [0, 1]).all()
    # blocked branch copies min(prev) * resp, no draw: 10 + min(11, 15) = 21 on the first tick
    c0 = Competitor("c1", fixed(5.0), theta=5.0)
    c1 = Competitor("c2", fixed(3.0))
    st = RaceState(0, [10.0, 12.0], [11.0, 15.0], [None, None])
    res = sim.simulate_batch(st, RaceConfig(21.0, (c0, c1)), 8, 1, records=True)
    assert (res.finish_ticks[:, 0] == 1).all() and (res.blocked == 1).all()


def test_laplace_counts_exact():
    """tests/test_agents.py:89-95: a runner that is home every time gives (d+1)/(d+n), 1/(d+n)."""
    import random

    cfg = RaceConfig(200.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(2)))
    st = RaceState(5, [190.0, 10.0], [15.0, 15.0], [None, None])
    assert rp_predict(st, cfg, 20, random.Random(1)) == ((20 + 1) / 22, 1 / 22)
    assert rp_predict(st, cfg, 0, random.Random(1)) == (0.5, 0.5)


def test_far_ahead_leader_always_wins():
    cfg = RaceConfig(200.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(2)))
    st = RaceState(5, [150.0, 10.0], [15.0, 15.0], [None, None])
    res = sim.simulate_batch(st, cfg, 100_000, 7)
    assert res.wins.tolist() == [100_000, 0]


def test_frozen_two_distribution_probability():
    """tests/test_race.py:264-272: P(U(10,20) beats U(1,25), L=500) = 0.93865 +- 0.0005."""
    cfg = RaceConfig(500.0, (Competitor("c1", UniformSteps(10.0, 20.0)), Competitor("c2", UniformSteps(1.0, 25.0))))
    N = 2_000_000
    res = sim.simulate_batch(None, cfg, N, 12345)
    p = res.wins[0] / N
    se = math.sqrt(0.93865 * (1 - 0.93865) / N)
    assert abs(p - 0.93865) < 0.0005 + 4 * se, p


def test_identical_competitors_split_evenly():
    cfg = RaceConfig(150.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(4)))
    N = 1_000_000
    res = sim.simulate_batch(None, cfg, N, 2)
    three_sigma = 3 * math.sqrt(0.25 * 0.75 / N)
    assert all(abs(w / N - 0.25) < three_sigma for w in res.wins)
    assert (res.ranks.sum(axis=0) == N).all() and (res.ranks.sum(axis=1) == N).all()


@pytest.mark.parametrize("which", ["c2_midrace", "derby5_start", "derby12_start", "derby20_start", "derby40_start",
                                   "uniform10_start", "fuzz_mix"])
def test_win_probabilities_match_reference_within_binomial_bounds(which):
    g = c2()
    if which == "c2_midrace":
        cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    elif which.startswith("derby"):
        import json
        import os

        from golden_io import GOLDEN  # noqa: F401

        base = config_from_dict(g["config"])
        n = int(which[len("derby"):-len("_start")])  # layouts: K = 1 (5), 2 (12, 20, 40)
        comps = tuple(
            Competitor(f"c{i + 1}", base.competitors[i % 5].steps, base.competitors[i % 5].preference,
                       base.competitors[i % 5].pref_sensitivity, base.competitors[i % 5].theta,
                       base.competitors[i % 5].responsiveness)
            for i in range(n))
        cfg, st = RaceConfig(2000.0, comps, conditions=base.conditions), None
    elif which == "uniform10_start":  # theta = 0 everywhere: the scan-free K = 2 kernel
        cfg, st = RaceConfig(500.0, tuple(Competitor(f"c{i + 1}", UniformSteps(8.0 + i % 4, 20.0)) for i in range(10))), None
    else:
        comps = (
            Competitor("a", UniformSteps(2.0, 6.0), theta=3.0),
            Competitor("b", LogNormalSteps(1.0, 0.5, 0.9), preference=0.2, pref_sensitivity=0.6),
            Competitor("c", UniformSteps(3.0, 4.5), theta=1.0, responsiveness=Responsiveness(0.7, 1.4, 0.5)),
            Competitor("d", LogNormalSteps(0.5, 0.2, 2.0), theta=6.0),
        )
        cfg, st = RaceConfig(60.0, comps, conditions=0.7), None
    n_ref = 20_000
    ref = oracle.batch(cfg, n_ref, state=st, master=424242, threads=8)
    assert ref["rc"] == 0
    n_gpu = 1_000_000
    res = sim.simulate_batch(st, cfg, n_gpu, 987654321)
    ok, z, crit = binomial_agreement(res.wins.tolist(), n_gpu, ref["wins"].tolist(), n_ref)
    assert ok, f"max |z| {z:.2f} > {crit:.2f}: gpu {res.wins / n_gpu} ref {ref['wins'] / n_ref}"
    # rank marginals too (each competitor's rank distribution), Bonferroni over n*n cells
    n = cfg.n_competitors
    for c in range(n):
        ok, z, crit = binomial_agreement(res.ranks[c].tolist(), n_gpu, ref["ranks"][c].tolist(), n_ref,
                                         alpha=ALPHA / n)
        assert ok, f"rank marginal of {c}: |z| {z:.2f} > {crit:.2f}"
    # competitor-timesteps per sim agree in mean (same race lengths)
    ct_gpu, ct_ref = res.competitor_steps / n_gpu, ref["ct"] / n_ref
    assert abs(ct_gpu - ct_ref) / ct_ref < 0.01


def test_full_order_pmf_chi_square_like_compare_pmf():
    comps = tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0) if i != 2 else UniformSteps(1.0, 25.0),
                             theta=4.0 if i == 1 else 0.0) for i in range(4))
    cfg = RaceConfig(150.0, comps)
    n_ref = 20_000
    import itertools

    ref_counts = {p: 0 for p in itertools.permutations(range(4))}
    for i in range(n_ref):
        r = oracle.run_race(cfg, oracle.derive_seed_run(10, i))
        ref_counts[tuple(r.order.tolist())] += 1
    res = sim.simulate_batch(None, cfg, 400_000, 77, perms=True)
    keys = list(itertools.permutations(range(4)))
    row_a = [int(c) for c in res.perms]
    row_b = [ref_counts[k] for k in keys]
    cols = [i for i in range(len(keys)) if row_a[i] + row_b[i] > 0]
    stat, p, dof, _ = chi2_contingency([[row_a[i] for i in cols], [row_b[i] for i in cols]], correction=False)
    assert p > ALPHA, (stat, p, dof)
    # the Lehmer-indexed histogram is layout-independent (2-4 competitors per lane)
    for k in (2, 3, 4):
        other = sim.simulate_batch(None, cfg, 400_000, 77, perms=True, lanes_per_slot=k)
        assert (other.perms == res.perms).all() and (other.ranks == res.ranks).all()


def test_sharding_and_lane_layout_invariance():
    """Same Philox counters => bit-identical tallies for any split of [0, N) (tests/test_batch.py:38-42)."""
    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    N = 300_000
    whole = sim.simulate_batch(st, cfg, N, 5)
    parts = [sim.simulate_batch(st, cfg, hi - lo, 5, sim_offset=lo)
             for lo, hi in [(0, 70_001), (70_001, 150_000), (150_000, N)]]
    assert (sum(p.wins for p in parts) == whole.wins).all()
    assert (sum(p.ranks for p in parts) == whole.ranks).all()
    assert sum(p.competitor_steps for p in parts) == whole.competitor_steps
    for k in (1, 2, 3):
        other = sim.simulate_batch(st, cfg, N, 5, lanes_per_slot=k)
        assert (other.wins == whole.wins).all() and other.competitor_steps == whole.competitor_steps


def test_divergence_reports_first_sim():
    cfg = RaceConfig(100.0, tuple(Competitor(f"c{i + 1}", UniformSteps(1.0, 1.0)) for i in range(2)),
                     tick_limit=10)
    with pytest.raises(sim.SimDivergedError) as e:
        sim.simulate_batch(None, cfg, 1000, 1)
    assert e.value.sim_index == 0


def test_records_consistent_with_tallies():
    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    res = sim.simulate_batch(st, cfg, 20_000, 9, records=True)
    n = cfg.n_competitors
    assert np.bincount(res.winner, minlength=n).tolist() == res.wins.tolist()
    assert (res.order[:, 0] == res.winner).all()
    assert (np.sort(res.order, axis=1) == np.arange(n)).all()
    assert (res.final_positions >= cfg.track_length).all()
    assert int(res.blocked.sum()) == res.blocked_steps
    ticks_run = res.finish_ticks.max(axis=1) - st.tick
    assert (ticks_run > 0).all()


def test_simulate_sharded_single_rank_matches_batch(philox_mode):
    from paper_2108_02419_b200.parallel import simulate_sharded

    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    t = simulate_sharded(st, cfg, 50_000, 3, mode=philox_mode)
    r = sim.simulate_batch(st, cfg, 50_000, 3)
    assert (t.wins == r.wins).all() and (t.ranks == r.ranks).all()
    assert t.competitor_steps == r.competitor_steps and t.first_diverged == -1
    # MT mode: run_batch's per-run seeds, derived on the device -- the reference's own tallies
    t = simulate_sharded(None, cfg, 3_000, 9, mode="mt")
    ob = oracle.batch(cfg, 3_000, master=9, threads=8)
    assert t.wins.tolist() == ob["wins"].tolist() and t.competitor_steps == ob["ct"]


def test_criterion_10_calibration_gpu_vs_reference():
    """tests/test_acceptance.py:394-424 with the GPU on one side: the chi-square PMF comparison of a
    native-mode batch against a reference (oracle) batch of the same config rejects at most 5/100
    times at alpha = 0.01, and detects the swapped step law at least 95/100 times (R = 300)."""
    import itertools

    base = tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(3))
    cfg = RaceConfig(150.0, base)
    swapped = RaceConfig(150.0, base[:2] + (Competitor("c3", UniformSteps(1.0, 25.0)),))
    keys = list(itertools.permutations(range(3)))

    def ref_counts(seed):
        counts = np.zeros(6, np.int64)
        for i in range(300):
            counts[keys.index(tuple(oracle.run_race(cfg, oracle.derive_seed_run(seed, i)).order.tolist()))] += 1
        return counts

    def chi2_p(a, b):
        cols = [i for i in range(6) if a[i] + b[i] > 0]
        if len(cols) < 2:
            return 1.0
        return chi2_contingency([[a[i] for i in cols], [b[i] for i in cols]], correction=False)[1]

    false_rejects = detections = 0
    for trial in range(100):
        ref = ref_counts(1000 + trial)
        same = sim.simulate_batch(None, cfg, 300, 5000 + trial, perms=True).perms.astype(np.int64)
        other = sim.simulate_batch(None, swapped, 300, 9000 + trial, perms=True).perms.astype(np.int64)
        false_rejects += chi2_p(ref, same) < ALPHA
        detections += chi2_p(ref, other) < ALPHA
    assert false_rejects <= 5, false_rejects
    assert detections >= 95, detections


def test_layout_rule_and_layout_invariance_from_the_start():
    """choose_k picks the measured-best layout (profiles/r1_k_sweep.md) and every layout gives the
    same per-sim results: the FP32 frame does not depend on it (from-start races included)."""
    for n, scan, want in ((10, True, 1), (12, True, 1), (20, True, 2), (22, True, 1), (10, False, 2),
                          (5, False, 1), (24, False, 3), (40, True, 2), (40, False, 3), (48, False, 3), (64, False, 2),
                          (96, False, 3), (128, True, 4)):
        comps = tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0), theta=8.0 if (scan and i % 4 == 1) else 0.0)
                      for i in range(n))
        cfg = RaceConfig(2000.0, comps)
        r = sim.simulate_batch(None, cfg, 3000, 11, records=True)
        assert r.lanes_per_slot == want, (n, scan, r.lanes_per_slot)
        for k in (1, 2, 3, 4):
            if -(-n // k) > 32 or k == want:
                continue
            o = sim.simulate_batch(None, cfg, 3000, 11, records=True, lanes_per_slot=k)
            assert (o.order == r.order).all() and (o.finish_ticks == r.finish_ticks).all()
            assert (o.final_positions == r.final_positions).all() and (o.blocked == r.blocked).all()


@pytest.mark.parametrize("field", ["c2", "derby5_from_start"])
def test_prepared_race_equals_per_call_upload(field):
    """bbe_prepare / bbe_launch_prepared (parameters uploaded once) add the same tallies as
    bbe_simulate_async (parameters uploaded per call), for a whole range and for two shards -- every
    tally field, including the full-order bins of n <= 6 fields."""
    import ctypes

    import torch

    from paper_2108_02419_b200.batch import resize_race

    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    if field != "c2":
        cfg, st = resize_race(cfg, 5), None
    dl = sim.DeviceLauncher(st, cfg)
    s = torch.cuda.current_stream().cuda_stream
    a = torch.zeros(dl.tally_len, dtype=torch.int64, device="cuda")
    b = torch.zeros_like(a)
    dl.launch(a.data_ptr(), 50_000, 99, stream=s)  # prepared
    req = sim.BbeRequest(30_000, 0, 99, sim.MODES["native"], 0, None, None, None, 0, 0)
    for off, ns in ((0, 30_000), (30_000, 20_000)):
        req.n_sims, req.sim_offset = ns, off
        rc = sim.lib().bbe_simulate_async(ctypes.byref(dl.pk.race), dl.pk.comps, ctypes.byref(dl.st),
                                          ctypes.byref(req), None, ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(s))
        assert rc == 0, sim.last_error()
    torch.cuda.synchronize()
    assert torch.equal(a, b) and int(a[dl.off["ct"]]) > 0
    assert dl.last_kernel_ms() > 0.0
