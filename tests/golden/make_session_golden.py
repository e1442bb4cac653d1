"""Record full BBE sessions by running the REFERENCE itself (racemarket's run_session).

Run in the build container (the reference sources are not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_session_golden.py

Writes ``session_c4.json.gz``: for each session config (100 RP/RB bettors on a derby field, the
SURVEY C4 shape at a small d so the reference finishes in seconds),

* the config (race fields, agent groups, master seed, opening period),
* the reference's complete event log (session.py:152-153) -- every race tick, submit, match, cancel,
  reject, expire, close and settle event, JSON floats round-trip exactly,
* every RP/RB prediction in processing order: (time, agent index, race tick, MT19937 stream position
  before the dry-run seeds, probabilities), recorded by wrapping RPBettor.predict / RBBettor.predict
  (agents.py:360-362, 402-404) -- the wrapped methods return the reference's own values unchanged,
* the settlement and final balances.

tests/test_session_exchange.py replays these sessions through paper_2108_02419_b200.session
(one batched launch per wake round, the exchange loop the reference's own) and requires the
identical event log.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import time
from dataclasses import replace

from racemarket import agents as A
from racemarket.agents import AgentParams
from racemarket.batch import resize_race
from racemarket.config import parse_config
from racemarket.race import BettingClose, RaceConfig
from racemarket.session import SessionConfig, run_session

HERE = os.path.dirname(os.path.abspath(__file__))
DERBY = "/root/reference/pkg/configs/derby.json"

_log: list | None = None
_depth = 0


def _wrap(cls):
    orig = cls.predict

    def predict(self, obs):
        # RBBettor.predict calls RPBettor.predict: only the outermost call is logged
        global _depth
        st = self.rng.getstate()[1]
        _depth += 1
        try:
            p = orig(self, obs)
        finally:
            _depth -= 1
        if _log is not None and _depth == 0:
            _log.append([obs.time, int(self.bettor_id[1:4]), obs.race_tick, st[624], hashlib.sha256(
                repr(st[:624]).encode()).hexdigest()[:16], list(p)])
        return p

    cls.predict = predict


_wrap(A.RPBettor)
_wrap(A.RBBettor)


def race_dict(rc: RaceConfig) -> dict:
    comps = []
    for c in rc.competitors:
        s = c.steps
        steps = ({"family": "uniform", "lo": s.lo, "hi": s.hi} if hasattr(s, "lo")
                 else {"family": "lognormal", "mu": s.mu, "sigma": s.sigma, "scale": s.scale})
        comps.append({"id": c.cid, "steps": steps, "preference": c.preference,
                      "pref_sensitivity": c.pref_sensitivity, "theta": c.theta,
                      "responsiveness": {"early_mult": c.responsiveness.early_mult,
                                         "late_mult": c.responsiveness.late_mult,
                                         "breakpoint": c.responsiveness.breakpoint}})
    bc = rc.betting_close
    return {"track_length": rc.track_length, "dt": rc.dt, "conditions": rc.conditions,
            "tick_limit": rc.tick_limit, "betting_close": {"rule": bc.rule, "k": bc.k}, "competitors": comps}


def agent_dict(g: AgentParams) -> dict:
    return {"strategy": g.strategy, "count": g.count, "d": g.d, "gamma": g.gamma,
            "stake_multiples": list(g.stake_multiples), "base_stake": g.base_stake, "max_stake": g.max_stake,
            "reevaluate_every": g.reevaluate_every, "wake_jitter": g.wake_jitter,
            "starting_balance": g.starting_balance}


def main():
    global _log
    with open(DERBY) as fh:
        derby = parse_config(json.load(fh)).race
    derby5 = resize_race(derby, 5)
    short = replace(derby5, track_length=600.0)
    cases = [
        # C4 shape: 100 bettors (RP and RB), 1 s re-evaluation with 1 s jitter, 5 s opening period
        ("c4_rp_rb_derby5_L600", short, (AgentParams("rp", count=50, d=12, reevaluate_every=1.0, wake_jitter=1.0),
                                          AgentParams("rb", count=50, d=12, reevaluate_every=1.0, wake_jitter=1.0)),
         20260818, 5.0),
        # small d makes exact probability ties (the _pick randrange draw) frequent; betting closes at the
        # 2nd finisher; a mixed population (linex/zi agents act between the RP/RB wakes)
        ("ties_kth2_mixed", replace(derby5, track_length=300.0, betting_close=BettingClose.kth(2)),
         (AgentParams("rp", count=20, d=3, reevaluate_every=0.5, wake_jitter=2.0),
          AgentParams("rb", count=20, d=2, reevaluate_every=1.5, wake_jitter=0.5, max_stake=7),
          AgentParams("linex", count=5, reevaluate_every=1.0, wake_jitter=1.0),
          AgentParams("zi", count=5, reevaluate_every=1.0, wake_jitter=1.0)),
         7, 3.0),
    ]
    out = []
    for name, race, groups, master, opening in cases:
        cfg = SessionConfig(race=race, agent_groups=groups, master_seed=master, opening_period=opening)
        _log = []
        t0 = time.perf_counter()
        res = run_session(cfg)
        dt = time.perf_counter() - t0
        preds, _log = _log, None
        ev = json.dumps(res.events, sort_keys=True)
        print(f"{name}: {len(res.events)} events, {len(preds)} predictions, {dt:.1f} s", flush=True)
        out.append({
            "name": name, "race": race_dict(race), "agent_groups": [agent_dict(g) for g in groups],
            "master_seed": master, "opening_period": opening, "reference_seconds": dt,
            "events": res.events, "events_sha256": hashlib.sha256(ev.encode()).hexdigest(),
            "predictions": preds,
            "winner": res.trajectory.winner,
            "final_balances": res.final_balances,
        })
    with gzip.open(os.path.join(HERE, "session_c4.json.gz"), "wt") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
