"""Generate golden vectors by running the REFERENCE itself (racemarket, /root/reference).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests python tests/golden/make_golden.py

Writes (all floats are JSON reprs, which round-trip bit-exactly):

* ``rng.json``      CPython MT19937 stream probes through the reference's ``make_rng``
                    (seeding.py:62-64): random(), uniform(), getrandbits(64), lognormvariate(), and
                    ``derive_seed`` (seeding.py:50-59).
* ``races.json.gz`` A corpus of races from the reference's own fuzz generator
                    (tests/test_acceptance.py:70-101) plus derby.json: for each, ``run_race`` from the
                    start line and ``simulate_from`` a mid-race state, with every step draw recorded in
                    consumption order (the draw-injection stream) and the outputs the kernel must match
                    bit-exactly (finish order, finish ticks, final positions, blocked steps, draw count).
* ``c2.json``       The SURVEY C2 workload: derby resized to 10 runners (batch.py:228-238), mid-race state
                    make_rng(3) + initial_state + 65 advance_race ticks, and a reference rp_predict
                    (agents.py:153-166) with d=64 from make_rng(11): seeds, per-sim winners, probabilities.

Draws are recorded by wrapping UniformSteps.draw / LogNormalSteps.draw (race.py:46-47, 68-69); the
wrapped methods return the reference's own values unchanged.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

from racemarket import race as R
from racemarket.agents import rp_predict
from racemarket.batch import resize_race
from racemarket.config import emit_default_config, parse_config
from racemarket.seeding import derive_seed, make_rng

from test_acceptance import random_race_config  # reference fuzz generator

HERE = os.path.dirname(os.path.abspath(__file__))
DERBY = "/root/reference/pkg/configs/derby.json"

_rec: list[float] | None = None
_u_draw = R.UniformSteps.draw
_l_draw = R.LogNormalSteps.draw


def _wrap(orig):
    def draw(self, rng):
        v = orig(self, rng)
        if _rec is not None:
            _rec.append(v)
        return v

    return draw


R.UniformSteps.draw = _wrap(_u_draw)
R.LogNormalSteps.draw = _wrap(_l_draw)


def cfg_to_dict(cfg: R.RaceConfig) -> dict:
    comps = []
    for c in cfg.competitors:
        s = c.steps
        d = {"id": c.cid}
        if isinstance(s, R.UniformSteps):
            d.update(family="uniform", lo=s.lo, hi=s.hi)
        else:
            d.update(family="lognormal", mu=s.mu, sigma=s.sigma, scale=s.scale)
        r = c.responsiveness
        d.update(preference=c.preference, pref_sensitivity=c.pref_sensitivity, theta=c.theta,
                 early_mult=r.early_mult, late_mult=r.late_mult, breakpoint=r.breakpoint)
        comps.append(d)
    return {"track_length": cfg.track_length, "conditions": cfg.conditions, "dt": cfg.dt,
            "tick_limit": cfg.tick_limit, "competitors": comps}


def state_to_dict(st: R.RaceState) -> dict:
    return {"tick": st.tick, "positions": list(st.positions), "prev_steps": list(st.prev_steps),
            "finish_ticks": list(st.finish_ticks), "blocked_steps": st.blocked_steps}


def record_run_race(cfg, seed):
    global _rec
    _rec = []
    try:
        traj = R.run_race(cfg, seed, record=False)
        err = None
    except R.RaceDivergedError as e:
        traj, err = None, str(e)
    draws, _rec = _rec, None
    out = {"seed": seed, "draws": draws, "error": err}
    if traj is not None:
        idx = {cid: i for i, cid in enumerate(cfg.competitor_ids)}
        out.update(order=[idx[c] for c in traj.finish_order], finish_ticks=list(traj.finish_ticks),
                   final_positions=list(traj.final_positions), blocked=traj.blocked_steps)
    return out


def record_simulate_from(state, cfg, seed):
    """simulate_from's order, plus the full final state from the same loop (race.py:399-405)."""
    global _rec
    _rec = []
    try:
        order_ids = R.simulate_from(state, cfg, seed)
        err = None
    except R.RaceDivergedError as e:
        order_ids, err = None, str(e)
    draws, _rec = _rec, None
    out = {"seed": seed, "draws": draws, "error": err}
    if order_ids is not None:
        st = state.clone()
        rng = make_rng(seed)
        while not st.all_finished():
            R.advance_race(st, cfg, rng)
        idx = {cid: i for i, cid in enumerate(cfg.competitor_ids)}
        order = [idx[c] for c in order_ids]
        assert order == list(R._finish_order(st, cfg))
        out.update(order=order, finish_ticks=list(st.finish_ticks), final_positions=list(st.positions),
                   blocked=st.blocked_steps - state.blocked_steps, end_tick=st.tick)
    return out


def mid_state(cfg, seed, k):
    rng = make_rng(seed)
    st = R.initial_state(cfg, rng)
    for _ in range(k):
        if st.all_finished():
            break
        R.advance_race(st, cfg, rng)
    return st


def make_rng_json():
    seeds = [0, 1, 3, 11, 12345, 2**32 - 1, 2**32, 2**63 + 12345, 2**64 - 1]
    probes = []
    for s in seeds:
        r = make_rng(s)
        rand = [r.random() for _ in range(40)]
        r = make_rng(s)
        unif = [r.uniform(10.0, 20.0) for _ in range(20)]
        r = make_rng(s)
        bits = [r.getrandbits(64) for _ in range(20)]
        r = make_rng(s)
        ln1 = [r.lognormvariate(2.67, 0.25) for _ in range(30)]
        r = make_rng(s)
        ln2 = [r.lognormvariate(-0.3, 0.6) for _ in range(30)]
        probes.append({"seed": s, "random": rand, "uniform_10_20": unif, "getrandbits64": [str(b) for b in bits],
                       "lognorm_2.67_0.25": ln1, "lognorm_-0.3_0.6": ln2})
    derived = []
    for m in [0, 1, 20260818, 2**64 - 1]:
        for i in [0, 1, 2, 999, 2**40 + 7]:
            derived.append({"master": str(m), "i": i, "seed": str(derive_seed(m, "run", i))})
    pref = []
    for cond, p, k in [(0.5, 0.5, 3.0), (0.7, 0.2, 0.0), (0.3, 0.5, 1.0), (1.0, 0.0, 2.0), (0.35, 0.3, 0.5),
                       (0.123, 0.987, 0.77)]:
        pref.append([cond, p, k, R.preference_factor(cond, p, k)])
    with open(os.path.join(HERE, "rng.json"), "w") as fh:
        json.dump({"python": sys.version.split()[0], "probes": probes, "derive_seed_run": derived,
                   "preference_factor": pref}, fh, indent=0)


def make_races_json():
    gen = random.Random(20_240_001)  # the reference's own fuzz stream (test_acceptance.py:106)
    corpus = []
    for i in range(400):
        cfg = random_race_config(gen)
        seed = derive_seed(1, "run", i)
        rr = record_run_race(cfg, seed)
        n_ticks = max(rr["finish_ticks"]) if rr.get("finish_ticks") else 1
        k = random.Random(i).randrange(0, max(1, n_ticks))
        st = mid_state(cfg, derive_seed(2, "mid", i), k)
        sf = record_simulate_from(st, cfg, derive_seed(3, "sim", i))
        corpus.append({"name": f"fuzz{i}", "config": cfg_to_dict(cfg), "run_race": rr,
                       "simulate_from": {"state": state_to_dict(st), **sf}})
    with open(DERBY) as fh:
        doc = json.load(fh)
    derby = parse_config({"race": doc["race"]}).race
    for n in (5, 10, 20, 40):
        cfg = resize_race(derby, n)
        for j in range(3):
            seed = derive_seed(20260818, "run", j)
            rr = record_run_race(cfg, seed)
            st = mid_state(cfg, 3, 40 + 10 * j)
            sf = record_simulate_from(st, cfg, derive_seed(20260818, "sim", n, j))
            corpus.append({"name": f"derby{n}_{j}", "config": cfg_to_dict(cfg), "run_race": rr,
                           "simulate_from": {"state": state_to_dict(st), **sf}})
    default = parse_config(emit_default_config()).race
    for j in range(4):
        seed = derive_seed(20260818, "run", j)
        rr = record_run_race(default, seed)
        st = mid_state(default, 7, 60)
        sf = record_simulate_from(st, default, derive_seed(7, "sim", j))
        corpus.append({"name": f"default5_{j}", "config": cfg_to_dict(default), "run_race": rr,
                       "simulate_from": {"state": state_to_dict(st), **sf}})
    # a divergence case (test_race.py:251-254)
    comps = tuple(R.Competitor(f"c{i + 1}", R.UniformSteps(1.0, 1.0)) for i in range(2))
    cfg = R.RaceConfig(track_length=100.0, competitors=comps, tick_limit=10)
    rr = record_run_race(cfg, 0)
    st = mid_state(cfg, 0, 3)
    sf = record_simulate_from(st, cfg, 5)
    corpus.append({"name": "diverge", "config": cfg_to_dict(cfg), "run_race": rr,
                   "simulate_from": {"state": state_to_dict(st), **sf}})
    with gzip.open(os.path.join(HERE, "races.json.gz"), "wt") as fh:
        json.dump({"python": sys.version.split()[0], "corpus": corpus}, fh)


def make_c2_json():
    with open(DERBY) as fh:
        doc = json.load(fh)
    derby = parse_config({"race": doc["race"]}).race
    cfg = resize_race(derby, 10)
    st = mid_state(cfg, 3, 65)
    d = 64
    agent = make_rng(11)
    probs = rp_predict(st, cfg, d, agent)
    seeds_rng = make_rng(11)
    seeds = [seeds_rng.getrandbits(64) for _ in range(d)]
    winners = []
    idx = {cid: i for i, cid in enumerate(cfg.competitor_ids)}
    for s in seeds:
        winners.append(idx[R.simulate_from(st, cfg, s)[0]])
    after = agent.random()  # agent stream position after rp_predict
    with open(os.path.join(HERE, "c2.json"), "w") as fh:
        json.dump({"config": cfg_to_dict(cfg), "state": state_to_dict(st), "agent_seed": 11, "d": d,
                   "seeds": [str(s) for s in seeds], "winners": winners, "probs": list(probs),
                   "agent_next_random": after}, fh, indent=0)


def make_sessions_json():
    """wake_schedule (session.py:104-121) for a few agent populations."""
    from racemarket.agents import AgentParams
    from racemarket.session import wake_schedule

    cases = []
    for seed, periods, jitters, horizon in [(7, [1.0] * 5, [1.0] * 5, 12.0),
                                            (20260818, [1.0, 2.5, 0.5], [1.0, 0.0, 3.0], 30.0),
                                            (3, [1.0] * 100, [1.0] * 100, 5.0)]:
        params = [AgentParams("rp", reevaluate_every=p, wake_jitter=j) for p, j in zip(periods, jitters)]
        wakes = wake_schedule(params, horizon, seed)
        cases.append({"seed": seed, "reevaluate_every": periods, "wake_jitter": jitters, "horizon": horizon,
                      "wakes": [list(w) for w in wakes]})
    with open(os.path.join(HERE, "sessions.json"), "w") as fh:
        json.dump({"wake_schedules": cases}, fh)


def make_derby_experiment():
    """The reference's canonical (defaults-applied) form of configs/derby.json, minus the session."""
    from racemarket.config import config_to_dict

    with open(DERBY) as fh:
        canon = config_to_dict(parse_config(json.load(fh)))
    canon.pop("session", None)
    with open(os.path.join(HERE, "derby_experiment.json"), "w") as fh:
        json.dump(canon, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    make_derby_experiment()
    make_rng_json()
    make_c2_json()
    make_races_json()
    make_sessions_json()
    print("golden vectors written to", HERE)
