"""The reference's dry-run acceptance criteria (tests/test_acceptance.py) through the GPU path.

MT mode is the drop-in: its probabilities must EQUAL the reference's (golden, made by
tests/golden/make_acceptance_golden.py).  Native mode must satisfy the same criteria statistically.
Criterion 1 (random races terminate, positions strictly increase until the finish) runs on the
reference fuzz corpus with recorded trajectories.
"""

import math
import statistics

import numpy as np
import pytest
from golden_io import acceptance, config_from_dict, plain_race, race_corpus, state_from_dict

import oracle
from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.agents import rp_predict
from paper_2108_02419_b200.seeding import derive_seed, make_rng

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["mt", "native"])
def test_criterion_07_directional_dry_runs(mode):
    g = acceptance()["c07"]
    race = plain_race(g["race"])
    probs = []
    for case in g["cases"]:
        p = rp_predict(state_from_dict(case["state"]), race, case["d"], make_rng(case["agent_seed"]), mode=mode)
        if mode == "mt":
            assert list(p) == case["probs"]  # the reference's own estimate, bit for bit
        probs.append(p[0])
    # tests/test_acceptance.py:310-314
    assert abs(probs[0] - 0.5) < 0.12
    for a, b in zip(probs, probs[1:]):
        assert b >= a - 0.05
    assert probs[-1] > 0.95


@pytest.mark.parametrize("mode", ["mt", "native"])
def test_criterion_08_log_loss_non_increasing_in_dry_runs(mode):
    g = acceptance()["c08"]
    cfg = plain_race(g["race"])
    depths = g["depths"]
    losses = {d: [] for d in depths}
    for r, case in enumerate(g["cases"]):
        st = state_from_dict(case["state"])
        for d in depths:
            p = rp_predict(st, cfg, d, make_rng(derive_seed(8, "agent", r, d)), mode=mode)
            if mode == "mt":
                assert list(p) == case["probs"][str(d)]
            losses[d].append(-math.log(p[case["winner"]]))
    # tests/test_acceptance.py:347-353: paired differences, 2 standard errors
    for lo, hi in zip(depths, depths[1:]):
        diffs = [a - b for a, b in zip(losses[hi], losses[lo])]
        se = statistics.stdev(diffs) / math.sqrt(len(diffs))
        assert statistics.fmean(diffs) <= 2.0 * se


def test_criterion_01_fuzz_races_terminate_with_monotone_trajectories():
    """tests/test_acceptance.py:104-123 on the reference's own fuzz configs (golden corpus): every
    race finishes, every competitor strictly advances until it finishes, and the recorded trajectory
    is the reference's (finish ticks and final positions bit-exact)."""
    checked = 0
    for case in race_corpus():
        exp = case["run_race"]
        if exp["error"] is not None:
            continue
        cfg = config_from_dict(case["config"])
        traj = sim.run_race(cfg, exp["seed"], record=True)
        assert traj.finish_ticks == tuple(exp["finish_ticks"])
        assert traj.final_positions == tuple(exp["final_positions"])
        ticks = np.array(traj.ticks)
        for c in range(cfg.n_competitors):
            f = traj.finish_ticks[c]
            assert (np.diff(ticks[: f + 1, c]) > 0).all()
            assert (ticks[f:, c] == ticks[f, c]).all()
        checked += 1
        if checked == 300:
            break
    assert checked == 300


@pytest.mark.parametrize("mode", ["mt", "native"])
def test_rp_and_rb_bettor_predictions(mode):
    """RPBettor / RBBettor.predict from session observations: MT equals the reference bit for bit
    and leaves the bettor's stream where the reference leaves it."""
    from types import SimpleNamespace

    from paper_2108_02419_b200.agents import rb_bettor_predict, rp_bettor_predict

    g = acceptance()["bettors"]
    cfg = config_from_dict(g["race"])
    for case in g["cases"]:
        obs = SimpleNamespace(**case["obs"])
        rng = make_rng(case["agent_seed"])
        if case["strategy"] == "rp":
            p = rp_bettor_predict(obs, cfg, case["d"], rng, mode=mode)
        else:
            p = rb_bettor_predict(obs, cfg, case["d"], case["gamma"], rng, mode=mode)
        assert rng.random() == case["next_random"]
        assert abs(sum(p) - 1.0) < 1e-12
        if mode == "mt":
            assert list(p) == case["probs"]
