"""Golden values for the reference's dry-run acceptance criteria, computed by the REFERENCE itself.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests python tests/golden/make_acceptance_golden.py

Writes ``acceptance.json.gz``:

* ``c07`` -- tests/test_acceptance.py:301-314: rp_predict(d=200) of a 2-runner race (conftest.make_race,
  L = 2000) for leader gaps 0..400, agent streams make_rng(500 + gap): the reference's probabilities.
* ``bettors`` -- RPBettor.predict / RBBettor.predict (agents.py:345-362, 399-404) on observations of a
  derby race (the session's view: positions, finish ticks, step histories), with the bettor's rng
  state after the call (its next random()) -- the reference's values.
* ``c08`` -- tests/test_acceptance.py:325-355: 1000 races of make_race(n=3, L=120); per race the
  mid-race state after initial_state + 3 advance_race ticks, the eventual winner, and the reference's
  rp_predict probabilities for d = 0, 5, 50 from make_rng(derive_seed(8, "agent", r, d)).
"""

from __future__ import annotations

import gzip
import json
import os

from conftest import make_race  # reference test helper (tests/conftest.py:6-8)
from racemarket.agents import AgentParams, Observation, RBBettor, RPBettor, rp_predict
from racemarket.batch import resize_race
from racemarket.config import parse_config
from racemarket.race import RaceState, advance_race, initial_state
from racemarket.seeding import derive_seed, make_rng

HERE = os.path.dirname(os.path.abspath(__file__))


def state_dict(st):
    return {"tick": st.tick, "positions": list(st.positions), "prev_steps": list(st.prev_steps),
            "finish_ticks": list(st.finish_ticks)}


def derby_dict(cfg):
    comps = []
    for c in cfg.competitors:
        s = c.steps
        fam = "uniform" if hasattr(s, "lo") else "lognormal"
        comps.append({"id": c.cid, "family": fam, "lo": getattr(s, "lo", 0.0), "hi": getattr(s, "hi", 0.0),
                      "mu": getattr(s, "mu", 0.0), "sigma": getattr(s, "sigma", 0.0), "scale": getattr(s, "scale", 1.0),
                      "preference": c.preference, "pref_sensitivity": c.pref_sensitivity, "theta": c.theta,
                      "early_mult": c.responsiveness.early_mult, "late_mult": c.responsiveness.late_mult,
                      "breakpoint": c.responsiveness.breakpoint})
    return {"track_length": cfg.track_length, "dt": cfg.dt, "conditions": cfg.conditions,
            "tick_limit": cfg.tick_limit, "competitors": comps}


def main():
    race = make_race(n=2, length=2000.0)
    c07 = []
    for gap in (0.0, 50.0, 100.0, 200.0, 400.0):
        st = RaceState(tick=70, positions=[1000.0, 1000.0 - gap], prev_steps=[15.0, 15.0], finish_ticks=[None, None])
        c07.append({"gap": gap, "state": state_dict(st), "agent_seed": 500 + int(gap), "d": 200,
                    "probs": list(rp_predict(st, race, 200, make_rng(500 + int(gap))))})
    cfg = make_race(n=3, length=120.0)
    c08 = []
    for r in range(1000):
        rng = make_rng(derive_seed(8, "run", r))
        state = initial_state(cfg, rng)
        for _ in range(3):
            advance_race(state, cfg, rng)
        mid = state.clone()
        while not state.all_finished():
            advance_race(state, cfg, rng)
        winner = min(range(cfg.n_competitors),
                     key=lambda c: (state.finish_ticks[c], cfg.track_length - state.positions[c], c))
        probs = {str(d): list(rp_predict(mid, cfg, d, make_rng(derive_seed(8, "agent", r, d)))) for d in (0, 5, 50)}
        c08.append({"state": state_dict(mid), "winner": winner, "probs": probs})
    with open("/root/reference/pkg/configs/derby.json") as fh:
        derby = resize_race(parse_config(json.load(fh)).race, 6)
    bettors = []
    rng = make_rng(99)
    st = initial_state(derby, rng)
    hist = [[] for _ in range(derby.n_competitors)]
    for tick in range(1, 400):
        if st.all_finished():
            break
        before = list(st.positions)
        advance_race(st, derby, rng)
        for c in range(derby.n_competitors):
            if st.positions[c] != before[c]:
                hist[c].append(st.positions[c] - before[c])
        some_done = any(f is not None for f in st.finish_ticks)
        if st.all_finished() or not (tick % 20 == 0 or (some_done and tick % 2 == 0)):
            continue
        obs = Observation(time=float(tick), race_tick=st.tick, positions=tuple(st.positions),
                          finish_ticks=tuple(st.finish_ticks), step_history=tuple(tuple(h) for h in hist),
                          grid={}, my_bets=(), balance=100_000)
        for strategy, cls in (("rp", RPBettor), ("rb", RBBettor)):
            params = AgentParams(strategy, d=40, gamma=0.61)
            b = cls(f"{strategy}{tick}", params, derby, make_rng(1000 + tick))
            probs = b.predict(obs)
            bettors.append({"strategy": strategy, "tick": tick, "d": 40, "gamma": 0.61, "agent_seed": 1000 + tick,
                            "obs": {"race_tick": obs.race_tick, "positions": list(obs.positions),
                                    "finish_ticks": list(obs.finish_ticks),
                                    "step_history": [list(h) for h in obs.step_history]},
                            "probs": list(probs), "next_random": b.rng.random()})
    doc = {"bettors": {"race": derby_dict(derby), "cases": bettors},
           "c07": {"race": {"n": 2, "lo": 10.0, "hi": 20.0, "length": 2000.0}, "cases": c07},
           "c08": {"race": {"n": 3, "lo": 10.0, "hi": 20.0, "length": 120.0}, "depths": [0, 5, 50], "cases": c08}}
    with gzip.open(os.path.join(HERE, "acceptance.json.gz"), "wt") as fh:
        json.dump(doc, fh)


if __name__ == "__main__":
    main()
