"""Host-side pieces of the drop-in API (no GPU): seeding, PMF bookkeeping, Lehmer indexing, the wake
schedule, and the reference-shaped types -- each checked against the reference's outputs."""

import itertools
import json
import os

import pytest

from golden_io import GOLDEN, rng_vectors
from paper_2108_02419_b200 import batch as B
from paper_2108_02419_b200 import race as R
from paper_2108_02419_b200.seeding import derive_seed, make_rng
from paper_2108_02419_b200.session import wake_schedule


def test_derive_seed_and_make_rng_match_reference():
    for d in rng_vectors()["derive_seed_run"]:
        assert derive_seed(int(d["master"]), "run", d["i"]) == int(d["seed"])
    for p in rng_vectors()["probes"]:
        r = make_rng(p["seed"])
        assert [r.random() for _ in range(40)] == p["random"]
    with pytest.raises(TypeError):
        derive_seed(1, True)


def test_preference_factor_matches_reference():
    for cond, p, k, f in rng_vectors()["preference_factor"]:
        assert R.preference_factor(cond, p, k) == f


def test_lehmer_index_is_itertools_order():
    for n in range(1, 7):
        for i, p in enumerate(itertools.permutations(range(n))):
            assert B.lehmer_index(p) == i


def test_estimate_pmf_spaces_and_compare():
    orders = [("a", "b", "c"), ("b", "a", "c"), ("a", "b", "c")]
    pmf = B.estimate_pmf(orders)
    assert pmf.space == B.ORDER_SPACE and pmf.counts == {"a-b-c": 2, "b-a-c": 1} and pmf.n_samples == 3
    wide = [tuple(f"c{i}" for i in range(7))] * 2
    assert B.estimate_pmf(wide).space == B.WINNER_SPACE
    assert B.compare_pmf(pmf, pmf).p_value == 1.0
    with pytest.raises(ValueError):
        B.estimate_pmf([])
    with pytest.raises(ValueError):
        B.compare_pmf(pmf, B.estimate_pmf(wide))
    other = B.OutcomePMF(B.ORDER_SPACE, 300, {"a-b-c": 10, "b-a-c": 290})
    assert B.compare_pmf(B.OutcomePMF(B.ORDER_SPACE, 300, {"a-b-c": 150, "b-a-c": 150}), other).p_value < 1e-6


def test_resize_race_cycles_templates():
    base = R.RaceConfig(100.0, (R.Competitor("x", R.UniformSteps(1, 2)), R.Competitor("y", R.UniformSteps(3, 4))))
    r5 = B.resize_race(base, 5)
    assert r5.competitor_ids == ("c1", "c2", "c3", "c4", "c5")
    assert [c.steps for c in r5.competitors] == [base.competitors[i % 2].steps for i in range(5)]
    assert B.resize_race(base, 2) is base


def test_wake_schedule_matches_reference():
    with open(os.path.join(GOLDEN, "sessions.json")) as fh:
        g = json.load(fh)
    for case in g["wake_schedules"]:
        got = wake_schedule(case["reevaluate_every"], case["wake_jitter"], case["horizon"], case["seed"])
        assert [list(w) for w in got] == case["wakes"]


def test_race_state_and_trajectory_types():
    st = R.RaceState(3, [1.0, 2.0], [0.5, 0.5], [None, 3])
    cl = st.clone()
    cl.positions[0] = 9.0
    assert st.positions[0] == 1.0 and st.finished_count() == 1 and not st.all_finished()
    t = R.Trajectory(("a", "b"), 1.0, None, (5, 4), ("b", "a"), (10.0, 11.0), 0)
    assert t.n_ticks == 5 and t.winner == "b"
    assert R.BettingClose.kth(2).close_rank(5) == 2 and R.BettingClose.last().close_rank(5) == 5
    with pytest.raises(R.RaceConfigError):
        R.Responsiveness(breakpoint=1.5).validate()
    assert R.Responsiveness(2.0, 0.5, 0.5).at(50.0, 100.0) == 0.5


def test_batch_config_validation():
    cfg = R.RaceConfig(100.0, (R.Competitor("a", R.UniformSteps(1, 2)),))
    with pytest.raises(ValueError):
        B.BatchConfig(cfg, 0, 1).validate()
    with pytest.raises(ValueError):
        B.BatchConfig(cfg, 1, 1, workers=0).validate()
    e = B.BatchRunError(7, "boom")
    import pickle

    assert pickle.loads(pickle.dumps(e)).run_index == 7


def test_race_section_parser_matches_reference_defaults():
    """products.parse_race applies the reference's defaults (config.py:93-178); derby.json parses."""
    from paper_2108_02419_b200.products import ConfigError, load_experiment, parse_race
    from golden_io import config_from_dict, c2

    # the reference's canonical form of configs/derby.json (config_to_dict(parse_config(...)), make_golden.py)
    doc, cfg, seed = load_experiment(os.path.join(GOLDEN, "derby_experiment.json"))
    assert seed == 20260818 and cfg.n_competitors == 5 and cfg.conditions == 0.35
    ref10 = config_from_dict(c2()["config"])  # the reference's parse of the same file, resized to 10
    for mine, ref in zip(cfg.competitors, ref10.competitors[:5]):
        assert (mine.steps, mine.preference, mine.pref_sensitivity, mine.theta, mine.responsiveness) == \
            (ref.steps, ref.preference, ref.pref_sensitivity, ref.theta, ref.responsiveness)
    with pytest.raises(ConfigError):
        parse_race({"competitors": [{"id": "a-b", "steps": {"family": "uniform", "lo": 1, "hi": 2}}]})
    with pytest.raises(ConfigError):
        parse_race({"competitors": [{"id": "a", "steps": {"family": "gamma"}}]})
    with pytest.raises(ConfigError):
        parse_race({"competitors": [], "track_length": 10})


def test_sim_errors_pickle_and_keep_the_sim_index():
    import pickle

    from paper_2108_02419_b200.race import RaceDivergedError
    from paper_2108_02419_b200.sim import DrawStreamError, SimDivergedError

    for cls in (SimDivergedError, DrawStreamError):
        e = pickle.loads(pickle.dumps(cls(7, "sim 7 failed")))
        assert type(e) is cls and e.sim_index == 7 and str(e) == "sim 7 failed"
    assert issubclass(SimDivergedError, RaceDivergedError) and issubclass(RaceDivergedError, RuntimeError)
