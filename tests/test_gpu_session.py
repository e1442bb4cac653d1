"""Batched dispatch of bettor dry runs, GPU run_batch / PMF / bench, and
trajectory recording (run_race(record=True)), all against the reference's semantics."""

import random

import numpy as np
import pytest

import oracle
from golden_io import c2, config_from_dict, race_corpus, state_from_dict
from paper_2108_02419_b200 import batch as B
from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.agents import rp_predict
from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps
from paper_2108_02419_b200.session import DryRunDispatcher, DryRunRequest, run_dry_run_session

pytestmark = pytest.mark.gpu


def test_dispatcher_equals_per_bettor_rp_predict():
    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    ds = [0, 1, 7, 64, 300, 1000] * 4
    a = [random.Random(1000 + i) for i in range(len(ds))]
    b = [random.Random(1000 + i) for i in range(len(ds))]
    got = DryRunDispatcher(cfg, "mt").predict_many(st, [DryRunRequest(r, d) for r, d in zip(a, ds)])
    want = [rp_predict(st, cfg, d, r, mode="mt") for r, d in zip(b, ds)]
    assert got == want
    assert all(x.getstate() == y.getstate() for x, y in zip(a, b))
    # and the first of them is the reference's own rp_predict value (golden)
    r = random.Random(g["agent_seed"])
    assert DryRunDispatcher(cfg, "mt").predict_many(st, [DryRunRequest(r, g["d"])])[0] == tuple(g["probs"])


def test_native_dispatcher_advances_streams_like_rp_predict():
    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    ds = [0, 5, 1000, 3, 20000]
    a = [random.Random(50 + i) for i in range(len(ds))]
    b = [random.Random(50 + i) for i in range(len(ds))]
    got = DryRunDispatcher(cfg, "native").predict_many(st, [DryRunRequest(r, d) for r, d in zip(a, ds)])
    for r, d in zip(b, ds):
        rp_predict(st, cfg, d, r, mode="native")
    assert all(x.getstate() == y.getstate() for x, y in zip(a, b))
    assert got[0] == tuple(1 / cfg.n_competitors for _ in range(cfg.n_competitors))
    assert all(abs(sum(p) - 1.0) < 1e-9 for p in got)
    # the 20000-run bettor's probabilities agree with the reference's golden rp_predict within binomial noise
    ref = np.array(g["probs"])
    assert np.abs(np.array(got[4]) - ref).max() < 5 * np.sqrt(0.25 / 20000) + 5 * np.sqrt(0.25 / g["d"])


def test_run_race_record_trajectory_matches_reference_stream():
    """race.py:373-390 with record=True; tests/test_race.py:226-242 trajectory properties."""
    case = next(c for c in race_corpus() if c["name"] == "derby5_0")
    cfg = config_from_dict(case["config"])
    seed = case["run_race"]["seed"]
    traj = sim.run_race(cfg, seed, record=True)
    assert traj.finish_ticks == tuple(case["run_race"]["finish_ticks"])
    assert len(traj.ticks) == traj.n_ticks + 1 and traj.ticks[0] == (0.0,) * cfg.n_competitors
    assert traj.final_positions == traj.ticks[-1] == tuple(case["run_race"]["final_positions"])
    for k in (1, 7, 40, traj.n_ticks // 2):
        _, pos, prev, fin, _ = oracle.advance_from_start(cfg, seed, k)
        assert list(traj.ticks[k]) == pos.tolist()
    for c in range(cfg.n_competitors):
        for t in range(1, len(traj.ticks)):
            if t <= traj.finish_ticks[c]:
                assert traj.ticks[t][c] > traj.ticks[t - 1][c]
            else:
                assert traj.ticks[t][c] == traj.ticks[t - 1][c]
    assert sim.run_race(cfg, seed, record=False).ticks is None


def test_run_batch_matches_reference_runs():
    cfg = RaceConfig(150.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(4)))
    res = B.run_batch(B.BatchConfig(cfg, 2000, master_seed=9))
    assert [r.run_index for r in res] == list(range(2000))
    for i in (0, 1, 999, 1999):
        o = oracle.run_race(cfg, oracle.derive_seed_run(9, i))
        assert res[i].finish_order == tuple(cfg.competitor_ids[c] for c in o.order)
        assert res[i].finish_ticks == tuple(int(t) for t in o.finish_ticks)
    assert res == B.run_batch(B.BatchConfig(cfg, 2000, master_seed=9, workers=8))  # workers never matter


def test_pmf_from_tally_equals_pmf_of_runs():
    cfg = RaceConfig(150.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0) if i != 2 else
                                             UniformSteps(1.0, 25.0)) for i in range(3)))
    runs = B.run_batch(B.BatchConfig(cfg, 3000, master_seed=4))
    a = B.pmf_from_results(runs)
    r = sim.simulate_batch(None, cfg, 3000, mode="mt", seed_master=4, perms=True)
    b = B.pmf_from_tally(r)
    assert a == b and B.compare_pmf(a, b).p_value == 1.0


def test_bench_columns():
    base = RaceConfig(500.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(5)))
    pts = B.bench(base, (5, 10, 20, 40), replications=2000, timing_reps=3, master_seed=99)
    assert [p.n_competitors for p in pts] == [5, 10, 20, 40]
    assert all(p.mean_s > 0 and p.reps == 6000 for p in pts)


def test_dry_run_session_c4_shape():
    base = RaceConfig(300.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(5)))
    out = run_dry_run_session(base, n_agents=20, d=50, master_seed=7, opening_period=3.0)
    assert out.launches >= 3 and out.sims == sum(50 for _ in out.predictions)
    assert all(abs(sum(p) - 1.0) < 1e-12 for _, _, p in out.predictions)
    # every prediction equals the bettor's own sequential rp_predict on the same live-race state, the
    # bettor's decision (its tie-break draw) made between its predictions as in the reference
    from paper_2108_02419_b200.seeding import spawn_rng
    from paper_2108_02419_b200.session import decide_draws, live_states

    states = live_states(base, 7)
    rngs = [spawn_rng(7, "agent", i) for i in range(20)]
    for t, i, p in out.predictions:
        tick = 0 if t <= 3.0 else int(np.ceil(t - 3.0 - 1e-9))
        assert rp_predict(states[tick], base, 50, rngs[i], mode="mt") == p
        decide_draws(rngs[i], p, None)


def test_cli_products(tmp_path):
    """python -m paper_2108_02419_b200 race|batch|bench|compare writes the reference's file formats."""
    import csv
    import json
    import os

    from golden_io import GOLDEN
    from paper_2108_02419_b200.__main__ import main
    from paper_2108_02419_b200.products import read_pmf_csv

    cfgp = os.path.join(GOLDEN, "derby_experiment.json")
    assert main(["race", "--config", cfgp, "--out", str(tmp_path / "r")]) == 0
    rows = list(csv.reader(open(tmp_path / "r" / "finish.csv")))
    assert rows[0] == ["competitor_id", "finish_tick", "finish_rank"] and len(rows) == 6
    # the reference's own race for derive_seed(20260818, "race") (cli.py:80-88)
    cfg = _race_from_doc(cfgp)
    o = oracle.run_race(cfg, oracle_seed_race())
    ticks = {r[0]: int(r[1]) for r in rows[1:]}
    assert [ticks[cid] for cid in cfg.competitor_ids] == [int(t) for t in o.finish_ticks]
    assert json.load(open(cfgp))["seed"] == 20260818
    assert main(["batch", "--config", cfgp, "--out", str(tmp_path / "b"), "--replications", "500"]) == 0
    assert main(["batch", "--config", cfgp, "--out", str(tmp_path / "b2"), "--replications", "500"]) == 0
    a, b = read_pmf_csv(tmp_path / "b" / "pmf.csv"), read_pmf_csv(tmp_path / "b2" / "pmf.csv")
    assert a == b and a.n_samples == 500
    assert main(["compare", str(tmp_path / "b" / "pmf.csv"), str(tmp_path / "b2" / "pmf.csv")]) == 0
    runs = list(csv.reader(open(tmp_path / "b" / "runs.csv")))
    assert runs[0] == ["run", "winner", "winner_ticks", "n_ticks", "finish_order"] and len(runs) == 501


def _race_from_doc(path):
    from paper_2108_02419_b200.products import load_experiment

    return load_experiment(path)[1]


def oracle_seed_race():
    from paper_2108_02419_b200.seeding import derive_seed

    return derive_seed(20260818, "race")


def test_session_on_batch_sees_every_batch_in_order():
    """on_batch (the host's use of a batch) reaches every batch exactly once, in order, and does not
    change the predictions."""
    base = RaceConfig(300.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(5)))
    ref = run_dry_run_session(base, n_agents=20, d=50, master_seed=7, opening_period=3.0)
    seen = []
    out = run_dry_run_session(base, n_agents=20, d=50, master_seed=7, opening_period=3.0,
                              on_batch=lambda batch: seen.extend(batch))
    assert out.predictions == ref.predictions == seen
