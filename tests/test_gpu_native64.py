"""NATIVE64 (FP64 state, Philox draws) against the C oracle's NATIVE64 draw source.

The kernel performs the reference's FP64 operations in the reference's order
(race.py:233-332), so fed the same Philox words as the oracle (oracle/bbe_oracle.c draw_philox) it
must reproduce every race bit for bit: finish order, finish ticks, final positions, blocked counts
and the tallies.  Uniform fields are compared bitwise; fields with a lognormal runner use the
device's log/sincospi/exp inside Box-Muller (not glibc's), so their step values may differ in the
last bits -- orders, finish ticks and blocked counts must still match exactly, positions to 1e-12.
"""

import random

import numpy as np
import pytest

import oracle
from golden_io import c2, config_from_dict, plain_race, race_corpus, state_from_dict
from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.batch import resize_race
from paper_2108_02419_b200.race import (
    Competitor,
    LogNormalSteps,
    RaceConfig,
    RaceState,
    Responsiveness,
    UniformSteps,
)

pytestmark = pytest.mark.gpu


def has_lognormal(cfg) -> bool:
    return any(not hasattr(c.steps, "lo") for c in cfg.competitors)


def check(cfg, n_sims, key, state=None, sim_offset=0, lanes=0):
    r = sim.simulate_batch(state, cfg, n_sims, key, mode="native64", records=True, sim_offset=sim_offset,
                           lanes_per_slot=lanes)
    o = oracle.batch_px(cfg, n_sims, key, state=state, sim_offset=sim_offset, threads=8, records=True)
    assert o["rc"] == 0
    assert (r.order == o["order"]).all()
    assert (r.finish_ticks == o["finish_ticks"]).all()
    assert (r.blocked == o["blocked_per_sim"]).all()
    if has_lognormal(cfg):
        np.testing.assert_allclose(r.final_positions, o["final_positions"], rtol=1e-12, atol=0)
    else:
        assert (r.final_positions.view(np.int64) == o["final_positions"].view(np.int64)).all()
    assert (r.wins == o["wins"]).all()
    assert (r.ranks == o["ranks"]).all()
    assert r.competitor_steps == o["ct"] and r.blocked_steps == o["blocked"]
    return r


def uniform_field(n, L=2000.0):
    return RaceConfig(L, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(n)))


def test_c1_c3_fields_from_start_bit_exact():
    check(uniform_field(5), 3000, 20260818)       # C1: 5 x U(10,20), L = 2000
    check(uniform_field(20), 2000, 20260818)      # C3 / C5: 20 x U(10,20), L = 2000
    check(uniform_field(20), 1000, 7, sim_offset=10**9 - 1000)  # the last shard of C5


def test_c2_state_derby_lognormal_and_blocking():
    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    r = check(cfg, 4000, 11, state=st)
    assert r.blocked_steps > 0


def test_blocking_uniform_fields_bit_exact():
    rng = random.Random(64)
    for trial in range(12):
        n = rng.choice([3, 6, 10, 13, 20, 32, 40, 63])
        comps = tuple(Competitor(f"b{i}", UniformSteps(lo, lo + rng.uniform(0.0, 8.0)),
                                 preference=rng.random(), pref_sensitivity=rng.uniform(0.0, 0.9),
                                 theta=rng.choice([0.0, rng.uniform(0.5, 9.0)]),
                                 responsiveness=Responsiveness(rng.uniform(0.5, 1.5), rng.uniform(0.5, 1.5),
                                                               rng.random()))
                      for i, lo in enumerate(rng.uniform(2.0, 12.0) for _ in range(n)))
        cfg = RaceConfig(rng.choice([120.0, 500.0, 2000.0]), comps, conditions=rng.random())
        check(cfg, 300, rng.getrandbits(64))
        tick, pos, prev, fin, _ = oracle.advance_from_start(cfg, trial, rng.randint(2, 12))
        st = RaceState(tick, pos.tolist(), prev.tolist(), [None if f < 0 else int(f) for f in fin])
        if any(f is None for f in st.finish_ticks):
            check(cfg, 300, rng.getrandbits(64), state=st)


def test_reference_fuzz_corpus_configs():
    """The 400 configs of the reference's own generator (tests/test_acceptance.py:70-101), frozen in
    tests/golden/races.json.gz: 32 NATIVE64 sims each, from the start and from the recorded state."""
    seen = 0
    for case in race_corpus():
        cfg = config_from_dict(case["config"])
        check(cfg, 32, 1000 + seen)
        sf = case.get("simulate_from")
        if sf and any(f is None for f in sf["state"]["finish_ticks"]):
            check(cfg, 32, 5000 + seen, state=state_from_dict(sf["state"]))
        seen += 1
        if seen >= 200:
            break
    assert seen >= 100


def test_lane_layouts_and_shards_agree():
    g = c2()
    cfg = resize_race(config_from_dict(g["config"]), 20)
    base = sim.simulate_batch(None, cfg, 5000, 3, mode="native64", records=True)
    for k in (1, 2, 3, 4):
        r = sim.simulate_batch(None, cfg, 5000, 3, mode="native64", records=True, lanes_per_slot=k)
        assert (r.order == base.order).all() and (r.final_positions == base.final_positions).all()
    a = sim.simulate_batch(None, cfg, 2000, 3, mode="native64", records=True)
    b = sim.simulate_batch(None, cfg, 3000, 3, mode="native64", records=True, sim_offset=2000)
    assert (np.concatenate([a.order, b.order]) == base.order).all()


def test_degenerate_steps_equal_the_reference_race():
    # U(v, v) steps are RNG-independent: NATIVE64 must give the reference's (MT) race exactly
    cfg = RaceConfig(64.0, tuple(Competitor(f"d{i}", UniformSteps(v, v), theta=t)
                                 for i, (v, t) in enumerate([(1.5, 2.0), (2.0, 0.0), (1.0, 4.0), (2.5, 1.0)])))
    o = oracle.run_race(cfg, 1)
    r = sim.simulate_batch(None, cfg, 3, 9, mode="native64", records=True)
    for i in range(3):
        assert r.order[i].tolist() == o.order.tolist()
        assert r.final_positions[i].tolist() == o.final_positions.tolist()


def test_divergence_matches_oracle():
    cfg = RaceConfig(2000.0, tuple(Competitor(f"c{i}", UniformSteps(1.0, 2.0)) for i in range(4)), tick_limit=900)
    with pytest.raises(sim.SimDivergedError) as ei:
        sim.simulate_batch(None, cfg, 100, 5, mode="native64")
    o = oracle.batch_px(cfg, 100, 5)
    assert o["rc"] == 2
    assert ei.value.sim_index == 0


def test_rp_predict_native64_and_group_tallies():
    import random as pyrandom

    from paper_2108_02419_b200.agents import rp_predict

    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    agent = pyrandom.Random(11)
    probs = rp_predict(st, cfg, 20000, agent, mode="native64")
    ref = pyrandom.Random(11)
    key = ref.getrandbits(64)
    for _ in range(20000 - 1):
        ref.getrandbits(64)
    assert agent.getstate() == ref.getstate()
    o = oracle.batch_px(cfg, 20000, key, state=st, threads=8)
    assert probs == tuple((int(w) + 1) / (20000 + cfg.n_competitors) for w in o["wins"])
    r = sim.simulate_batch(st, cfg, 6000, 5, mode="native64", group_size=1000)
    assert (r.group_wins.sum(axis=0) == r.wins).all()


def test_device_launcher_native64_matches_host_call():
    import torch

    cfg = uniform_field(20)
    dl = sim.DeviceLauncher(None, cfg, native_mode="native64")
    t = torch.zeros(dl.tally_len, dtype=torch.int64, device="cuda")
    dl.launch(t.data_ptr(), 40_000, 123, mode="native64", stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    r = sim.simulate_batch(None, cfg, 40_000, 123, mode="native64")
    h = t.cpu().numpy().astype(np.uint64)
    n = 20
    assert (h[:n] == r.wins).all()
    assert int(h[dl.off["ct"]]) == r.competitor_steps
