"""Bit-exact parity of the FP64 inject kernel against the reference (draw-injection mode).

Fed the reference's own recorded step draws, the kernel must reproduce -- exactly -- the finish
order, finish ticks, final positions (bit patterns), blocked-step counts and draw consumption of
``run_race`` (race.py:373-390) and ``simulate_from`` (race.py:393-406).

Sources of expected values:
  * tests/golden/races.json.gz -- recorded by running the reference itself (make_golden.py);
  * the C oracle (pinned to those vectors in test_oracle_golden.py) for large seeded batches.
"""

import numpy as np
import pytest

import oracle
from golden_io import c2, config_from_dict, race_corpus, state_from_dict
from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.race import Competitor, RaceConfig, RaceState, UniformSteps

pytestmark = pytest.mark.gpu


def _inject_one(cfg, state, draws, **kw):
    draws = np.asarray(draws, np.float64)
    return sim.simulate_batch(state, cfg, 1, mode="inject", draws=draws,
                              draw_offsets=np.array([0, len(draws)], np.int64), records=True, perms=True, **kw)


def _assert_case(res, exp, i=0):
    assert res.order[i].tolist() == exp["order"]
    assert res.finish_ticks[i].tolist() == exp["finish_ticks"]
    assert res.final_positions[i].tolist() == exp["final_positions"]  # bit-exact doubles
    assert int(res.blocked[i]) == exp["blocked"]
    assert int(res.draws_used[i]) == len(exp["draws"])


@pytest.mark.parametrize("chunk", range(4))
def test_golden_corpus_bit_exact(chunk):
    for case in race_corpus()[chunk::4]:
        cfg = config_from_dict(case["config"])
        rr = case["run_race"]
        if rr["error"] is None:
            res = _inject_one(cfg, None, rr["draws"])
            _assert_case(res, rr)
            assert int(res.winner[0]) == rr["order"][0]
        else:
            with pytest.raises(sim.SimDivergedError):
                _inject_one(cfg, None, rr["draws"])
        sf = case["simulate_from"]
        st = state_from_dict(sf["state"])
        if sf["error"] is None:
            _assert_case(_inject_one(cfg, st, sf["draws"]), sf)
        else:
            with pytest.raises(sim.SimDivergedError):
                _inject_one(cfg, st, sf["draws"])


def _oracle_stream(cfg, state, seeds):
    """Record draws + expected outputs for each seed with the (pinned) C oracle."""
    draws, offs, exp = [], [0], []
    for s in seeds:
        r = oracle.run_race(cfg, int(s), record=True) if state is None else \
            oracle.simulate_from(state, cfg, int(s), record=True)
        assert r.rc == 0
        draws.append(r.draws)
        offs.append(offs[-1] + len(r.draws))
        exp.append(r)
    return np.concatenate(draws), np.array(offs, np.int64), exp


@pytest.mark.parametrize("k_hint", [0, 1, 2, 3, 4])
def test_c2_batch_bit_exact_all_lane_layouts(k_hint):
    g = c2()
    cfg = config_from_dict(g["config"])
    st = state_from_dict(g["state"])
    seeds = oracle.rp_seeds(g["agent_seed"], 600)
    draws, offs, exp = _oracle_stream(cfg, st, seeds)
    res = sim.simulate_batch(st, cfg, len(seeds), mode="inject", draws=draws, draw_offsets=offs, records=True,
                             lanes_per_slot=k_hint)
    for i, r in enumerate(exp):
        assert res.order[i].tolist() == r.order.tolist()
        assert res.finish_ticks[i].tolist() == r.finish_ticks.tolist()
        assert res.final_positions[i].tolist() == r.final_positions.tolist()
        assert int(res.blocked[i]) == r.blocked
        assert int(res.draws_used[i]) == r.draws_used
    # tallies agree with the per-sim records and with the oracle's batch tally
    ob = oracle.batch(cfg, len(seeds), state=st, seeds=seeds)
    assert res.wins.tolist() == ob["wins"].tolist()
    assert (res.ranks == ob["ranks"]).all()
    assert res.competitor_steps == ob["ct"]
    assert res.blocked_steps == ob["blocked"]
    # the reference's own rp_predict result for the first 64 seeds
    res64 = sim.simulate_batch(st, cfg, 64, mode="inject", draws=draws[: offs[64]], draw_offsets=offs[:65])
    n = cfg.n_competitors
    assert [(int(w) + 1) / (64 + n) for w in res64.wins] == g["probs"]


@pytest.mark.parametrize("n", [1, 2, 5, 7, 13, 20, 33, 40, 64, 100])
def test_from_start_batches_bit_exact_across_field_sizes(n):
    from paper_2108_02419_b200.race import LogNormalSteps, Responsiveness

    comps = []
    for i in range(n):
        steps = UniformSteps(2.0 + (i % 3), 6.0 + (i % 5)) if i % 4 else LogNormalSteps(0.8, 0.4, 1.5)
        comps.append(Competitor(f"c{i}", steps, preference=(i % 7) / 7.0, pref_sensitivity=0.3 * (i % 2),
                                theta=[0.0, 2.5, 6.0][i % 3],
                                responsiveness=Responsiveness(0.9 + 0.05 * (i % 4), 1.1, 0.4)))
    cfg = RaceConfig(120.0, tuple(comps), conditions=0.4)
    seeds = [oracle.derive_seed_run(99, i) for i in range(150)]
    draws, offs, exp = _oracle_stream(cfg, None, seeds)
    res = sim.simulate_batch(None, cfg, len(seeds), mode="inject", draws=draws, draw_offsets=offs, records=True,
                             perms=True)
    for i, r in enumerate(exp):
        assert res.order[i].tolist() == r.order.tolist()
        assert res.final_positions[i].tolist() == r.final_positions.tolist()
        assert res.finish_ticks[i].tolist() == r.finish_ticks.tolist()
        assert int(res.blocked[i]) == r.blocked
    if n <= 6:
        import itertools
        import math

        # perms histogram is the full finish-order PMF (batch.py:149-166) by Lehmer index
        perms = list(itertools.permutations(range(n)))
        counts = {p: 0 for p in perms}
        for r in exp:
            counts[tuple(r.order.tolist())] += 1
        assert res.perms.tolist() == [counts[p] for p in perms]
        assert len(res.perms) == math.factorial(n)


def test_stream_under_and_over_consumption_is_an_error():
    g = c2()
    cfg = config_from_dict(g["config"])
    st = state_from_dict(g["state"])
    draws, offs, _ = _oracle_stream(cfg, st, oracle.rp_seeds(5, 3))
    short = offs.copy()
    short[2:] -= 1
    with pytest.raises(sim.DrawStreamError) as e:
        sim.simulate_batch(st, cfg, 3, mode="inject", draws=draws, draw_offsets=short)
    assert e.value.sim_index == 1  # sim 1 is one draw short (sim 2 is misaligned too; the first is reported)
    longer = offs.copy()
    longer[2:] += 1
    d2 = np.insert(draws, offs[2], 15.0)
    with pytest.raises(sim.DrawStreamError) as e:
        sim.simulate_batch(st, cfg, 3, mode="inject", draws=d2, draw_offsets=longer)
    assert e.value.sim_index == 1


def test_degenerate_draw_semantics_exact():
    """tests/test_race.py:120-229 scenarios, driven through the kernel with injected draws."""
    def fixed(v):
        return UniformSteps(v, v)

    # blocked step copies min(prev) and skips the preference factor, keeps responsiveness
    slow = Competitor("c1", fixed(5.0), preference=0.0, pref_sensitivity=100.0, theta=5.0)
    front = Competitor("c2", fixed(3.0))
    cfg = RaceConfig(track_length=11.0, competitors=(slow, front), conditions=1.0)
    st = RaceState(0, [8.0, 10.0], [4.0, 3.0], [None, None])
    exp = oracle.simulate_from(st, cfg, 0, record=True)
    res = _inject_one(cfg, st, exp.draws)
    assert res.final_positions[0].tolist() == exp.final_positions.tolist()
    assert int(res.blocked[0]) == exp.blocked >= 1
    # overshoot tie-break then index (test_race.py:212-223)
    a, b = Competitor("c1", fixed(11.0)), Competitor("c2", fixed(12.0))
    cfg = RaceConfig(track_length=22.0, competitors=(a, b))
    res = _inject_one(cfg, None, [11.0, 12.0] * 3)
    assert res.order[0].tolist() == [1, 0] and res.finish_ticks[0].tolist() == [2, 2]
    cfg2 = RaceConfig(track_length=22.0, competitors=(Competitor("c1", fixed(11.0)), Competitor("c2", fixed(11.0))))
    res = _inject_one(cfg2, None, [11.0] * 6)
    assert res.order[0].tolist() == [0, 1]
    # finished rivals never block (test_race.py:152-155)
    cfg = RaceConfig(track_length=20.0, competitors=(Competitor("c1", fixed(5.0), theta=50.0),
                                                     Competitor("c2", fixed(3.0))))
    st = RaceState(3, [10.0, 21.0], [1.0, 1.0], [None, 3])
    res = _inject_one(cfg, st, [5.0, 5.0])
    assert res.finish_ticks[0].tolist() == [5, 3] and res.order[0].tolist() == [1, 0]
    assert int(res.blocked[0]) == 0
