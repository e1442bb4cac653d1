"""Pin the CPU oracle (oracle/bbe_oracle.c, oracle/pyref.py) to the reference's own outputs.

The golden vectors were produced by running the reference (tests/golden/make_golden.py).  Every
check here is bit-exact: floats are compared with ``==`` on values that round-trip through JSON.
"""

import numpy as np
import pytest

import oracle
from oracle import pyref
from golden_io import c2, config_from_dict, race_corpus, rng_vectors, state_from_dict


def test_mt_streams_match_cpython_reference():
    for p in rng_vectors()["probes"]:
        s = p["seed"]
        assert oracle.mt_random(s, 40).tolist() == p["random"]
        assert oracle.mt_uniform(s, 10.0, 20.0, 20).tolist() == p["uniform_10_20"]
        assert [int(v) for v in oracle.mt_getrandbits64(s, 20)] == [int(v) for v in p["getrandbits64"]]
        assert oracle.mt_lognormvariate(s, 2.67, 0.25, 30).tolist() == p["lognorm_2.67_0.25"]
        assert oracle.mt_lognormvariate(s, -0.3, 0.6, 30).tolist() == p["lognorm_-0.3_0.6"]


def test_derive_seed_matches_reference():
    for d in rng_vectors()["derive_seed_run"]:
        assert oracle.derive_seed_run(int(d["master"]), d["i"]) == int(d["seed"])
        assert pyref.derive_seed(int(d["master"]), "run", d["i"]) == int(d["seed"])


def test_preference_factor_matches_reference():
    lib = oracle.lib()
    for cond, p, k, f in rng_vectors()["preference_factor"]:
        assert lib.orc_preference_factor(cond, p, k) == f
        assert pyref.preference_factor(cond, p, k) == f


def _check(res, exp):
    assert res.rc == 0
    assert res.order.tolist() == exp["order"]
    assert res.finish_ticks.tolist() == exp["finish_ticks"]
    assert res.final_positions.tolist() == exp["final_positions"]
    assert res.blocked == exp["blocked"]
    assert res.draws_used == len(exp["draws"])


@pytest.mark.parametrize("chunk", range(4))
def test_oracle_run_race_and_simulate_from_bit_exact(chunk):
    corpus = race_corpus()
    for case in corpus[chunk::4]:
        cfg = config_from_dict(case["config"])
        rr = case["run_race"]
        if rr["error"] is None:
            # from the seed (MT19937 in the oracle) ...
            res = oracle.run_race(cfg, rr["seed"], record=True)
            _check(res, rr)
            assert res.draws.tolist() == rr["draws"]
            # ... and from the recorded draw stream (the kernel's injection contract)
            _check(oracle.run_race(cfg, 0, replay=np.array(rr["draws"])), rr)
        else:
            assert oracle.run_race(cfg, rr["seed"]).rc == oracle.ORC_EDIVERGED
        sf = case["simulate_from"]
        st = state_from_dict(sf["state"])
        if sf["error"] is None:
            res = oracle.simulate_from(st, cfg, sf["seed"], record=True)
            _check(res, sf)
            assert res.draws.tolist() == sf["draws"]
            _check(oracle.simulate_from(st, cfg, 0, replay=np.array(sf["draws"])), sf)
        else:
            assert oracle.simulate_from(st, cfg, sf["seed"]).rc == oracle.ORC_EDIVERGED


def test_replay_detects_draw_stream_mismatch():
    case = next(c for c in race_corpus() if c["run_race"]["error"] is None and len(c["run_race"]["draws"]) > 3)
    cfg = config_from_dict(case["config"])
    draws = np.array(case["run_race"]["draws"])
    assert oracle.run_race(cfg, 0, replay=draws[:-1]).rc == oracle.ORC_EDRAWS
    assert oracle.run_race(cfg, 0, replay=np.append(draws, 1.0)).rc == oracle.ORC_EDRAWS


def test_pyref_matches_reference_corpus():
    for case in race_corpus()[::7]:
        cfg = config_from_dict(case["config"])
        rr = case["run_race"]
        if rr["error"] is not None:
            with pytest.raises(pyref.Diverged):
                pyref.run_race(cfg, rr["seed"])
            continue
        out = pyref.run_race(cfg, rr["seed"])
        assert list(out["order"]) == rr["order"]
        assert list(out["finish_ticks"]) == rr["finish_ticks"]
        assert list(out["positions"]) == rr["final_positions"]
        sf = case["simulate_from"]
        if sf["error"] is None:
            st = state_from_dict(sf["state"])
            assert list(pyref.simulate_from(st, cfg, sf["seed"])["order"]) == sf["order"]


def test_c2_state_and_rp_predict_match_reference():
    g = c2()
    cfg = config_from_dict(g["config"])
    st = state_from_dict(g["state"])
    tick, pos, prev, fin, blocked = oracle.advance_from_start(cfg, 3, 65)
    assert tick == st.tick
    assert pos.tolist() == st.positions
    assert prev.tolist() == st.prev_steps
    assert [None if f < 0 else int(f) for f in fin] == st.finish_ticks
    seeds = oracle.rp_seeds(g["agent_seed"], g["d"])
    assert [int(s) for s in seeds] == [int(s) for s in g["seeds"]]
    out = oracle.batch(cfg, g["d"], state=st, seeds=seeds, winners=True)
    assert out["rc"] == 0
    assert out["winners"].tolist() == g["winners"]
    n = cfg.n_competitors
    probs = [(int(w) + 1) / (g["d"] + n) for w in out["wins"]]
    assert probs == g["probs"]
    import random

    agent = random.Random(g["agent_seed"])
    assert pyref.rp_predict(st, cfg, g["d"], agent) == tuple(g["probs"])
    assert agent.random() == g["agent_next_random"]


def test_batch_threads_do_not_change_tallies():
    g = c2()
    cfg = config_from_dict(g["config"])
    st = state_from_dict(g["state"])
    a = oracle.batch(cfg, 300, state=st, master=5, threads=1)
    b = oracle.batch(cfg, 300, state=st, master=5, threads=4)
    assert (a["wins"] == b["wins"]).all() and (a["ranks"] == b["ranks"]).all()
    assert a["ct"] == b["ct"] and a["blocked"] == b["blocked"]
    assert a["wins"].sum() == 300 and (a["ranks"].sum(axis=0) == 300).all()


def test_oracle_reproduces_reference_dry_run_criteria():
    """Criteria 7 and 8 of the reference's acceptance suite (tests/test_acceptance.py:301-355): the
    oracle rebuilds the mid-race states and the reference's rp_predict probabilities exactly."""
    from golden_io import acceptance, plain_race

    g = acceptance()
    cfg = plain_race(g["c07"]["race"])
    for case in g["c07"]["cases"]:
        st = state_from_dict(case["state"])
        seeds = oracle.rp_seeds(case["agent_seed"], case["d"])
        out = oracle.batch(cfg, case["d"], state=st, seeds=seeds)
        assert [(int(w) + 1) / (case["d"] + 2) for w in out["wins"]] == case["probs"]
    cfg = plain_race(g["c08"]["race"])
    from paper_2108_02419_b200.seeding import derive_seed

    for r, case in enumerate(g["c08"]["cases"][:150]):
        tick, pos, prev, fin, _ = oracle.advance_from_start(cfg, derive_seed(8, "run", r), 3)
        assert tick == case["state"]["tick"] and pos.tolist() == case["state"]["positions"]
        assert prev.tolist() == case["state"]["prev_steps"]
        st = state_from_dict(case["state"])
        for d in (5, 50):
            seeds = oracle.rp_seeds(derive_seed(8, "agent", r, d), d)
            out = oracle.batch(cfg, d, state=st, seeds=seeds)
            assert [(int(w) + 1) / (d + 3) for w in out["wins"]] == case["probs"][str(d)]


def test_bettor_predictions_via_oracle_match_reference():
    """RPBettor / RBBettor.predict (agents.py:345-362, 399-404): state reconstruction from the
    observation + dry runs (oracle) + rb weighting reproduce the reference's probabilities."""
    import random as _random
    from types import SimpleNamespace

    from golden_io import acceptance
    from paper_2108_02419_b200.agents import rb_weighted, reconstruct_state

    g = acceptance()["bettors"]
    cfg = config_from_dict(g["race"])
    n = cfg.n_competitors
    for case in g["cases"]:
        obs = SimpleNamespace(**case["obs"])
        st = reconstruct_state(obs)
        seeds = oracle.rp_seeds(case["agent_seed"], case["d"])
        out = oracle.batch(cfg, case["d"], state=st, seeds=seeds)
        probs = tuple((int(w) + 1) / (case["d"] + n) for w in out["wins"])
        if case["strategy"] == "rb":
            probs = rb_weighted(probs, case["gamma"])
        assert list(probs) == case["probs"]
        rng = _random.Random(case["agent_seed"])
        for _ in range(case["d"]):
            rng.getrandbits(64)
        assert rng.random() == case["next_random"]
