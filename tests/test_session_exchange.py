"""The full BBE session (C4) with batched predictions against sessions recorded from the reference.

tests/golden/session_c4.json.gz holds complete ``racemarket.session.run_session`` event logs (every
race tick, submit, match, cancel, reject, expire, close and settle event) plus every RP/RB
prediction with the bettor's MT19937 stream position before it (make_session_golden.py).  The
session here is the reference's own loop and exchange (racemarket from baseline/_ref, the offline
install of /root/reference) with paper_2108_02419_b200.session batching every wake round's
predictions into one launch.  Exact equality of the event log proves the batched rounds consume
every bettor's stream exactly as the reference does -- dry-run seeds, the tie-break ``randrange``
and the RB stake ``randint`` (agents.py:304-310, 334-342, 406-408) -- and return the reference's
probabilities.

CPU: the rounds are served by the C oracle (test infrastructure standing in for the GPU batch).
GPU: the rounds are served by the MT kernel through DryRunDispatcher -- the product path.
"""

from __future__ import annotations

import functools
import gzip
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2108_02419_b200 import session as S

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "session_c4.json.gz")

try:
    S.import_racemarket()
    HAVE_RM = True
except ImportError:
    HAVE_RM = False

pytestmark = pytest.mark.skipif(not HAVE_RM, reason="racemarket (baseline/_ref) not installed")


@functools.lru_cache(None)
def golden():
    with gzip.open(GOLDEN, "rt") as fh:
        return json.load(fh)


def session_config(g):
    from racemarket.agents import AgentParams
    from racemarket.race import BettingClose, Competitor, LogNormalSteps, RaceConfig, Responsiveness, UniformSteps
    from racemarket.session import SessionConfig

    r = g["race"]
    comps = []
    for c in r["competitors"]:
        s = c["steps"]
        steps = (UniformSteps(s["lo"], s["hi"]) if s["family"] == "uniform"
                 else LogNormalSteps(s["mu"], s["sigma"], s["scale"]))
        rs = c["responsiveness"]
        comps.append(Competitor(c["id"], steps, c["preference"], c["pref_sensitivity"], c["theta"],
                                Responsiveness(rs["early_mult"], rs["late_mult"], rs["breakpoint"])))
    bc = r["betting_close"]
    race = RaceConfig(r["track_length"], tuple(comps), dt=r["dt"], conditions=r["conditions"],
                      betting_close=BettingClose(bc["rule"], bc["k"]), tick_limit=r["tick_limit"])
    groups = tuple(AgentParams(a["strategy"], count=a["count"], d=a["d"], gamma=a["gamma"],
                               stake_multiples=tuple(a["stake_multiples"]), base_stake=a["base_stake"],
                               max_stake=a["max_stake"], reevaluate_every=a["reevaluate_every"],
                               wake_jitter=a["wake_jitter"], starting_balance=a["starting_balance"])
                   for a in g["agent_groups"])
    return SessionConfig(race=race, agent_groups=groups, master_seed=g["master_seed"],
                         opening_period=g["opening_period"])


class OraclePredictor:
    """Serves a wake round on the CPU oracle: the requests' seeds drawn with getrandbits(64) as
    rp_predict draws them (agents.py:164), simulated by oracle.batch, winners split per request."""

    def __init__(self, race):
        self.race = race
        self.launches = 0
        self.sims = 0

    def prepare(self, requests):
        ds = [r.d for r in requests]
        return {"ds": ds, "seeds": [r.rng.getrandbits(64) for r, d in zip(requests, ds) for _ in range(d)]}

    def launch(self, state, prep):
        """Runs the batch at once; the 'pending' handle is the result (the GPU's is asynchronous)."""
        import oracle

        n = len(self.race.competitors)
        ds, seeds = prep["ds"], prep["seeds"]
        total = len(seeds)
        if total == 0:
            return [tuple(1 / (d + n) for _ in range(n)) for d in ds]
        self.launches += 1
        self.sims += total
        out = oracle.batch(self.race, total, state=state, seeds=np.array(seeds, np.uint64), winners=True)
        assert out["rc"] == 0
        w = out["winners"]
        res, at = [], 0
        for d in ds:
            wins = np.bincount(w[at:at + d], minlength=n)
            at += d
            res.append(tuple((int(x) + 1) / (d + n) for x in wins))
        return res

    def finish(self, pending, prep):
        return pending

    def predict_many(self, state, requests):
        prep = self.prepare(requests)
        return self.finish(self.launch(state, prep), prep)


def record_predictions(sess):
    """Wrap each batched bettor's predict hook to log what the golden file records."""
    log = []
    for i, a in sess._batched.items():
        hook = a.predict

        def predict(obs, _hook=hook, _a=a, _i=i):
            st = _a.rng.getstate()[1]
            p = _hook(obs)
            log.append([obs.time, _i, obs.race_tick, st[624], hashlib.sha256(repr(st[:624]).encode()).hexdigest()[:16],
                        list(p)])
            return p

        a.predict = predict
    return log


def run_and_compare(g, predictor=None, mode="mt", look_ahead=True):
    cfg = session_config(g)
    sess = S.make_gpu_session(cfg, mode=mode, predictor=predictor, look_ahead=look_ahead)
    log = record_predictions(sess)
    res = sess.run()
    assert sess.stats.fallbacks == 0, "every prediction should come from its planned round"
    assert len(log) == len(g["predictions"])
    for k, (mine, ref) in enumerate(zip(log, g["predictions"])):
        assert mine == ref, f"prediction {k}: {mine} != {ref}"
    events = json.loads(json.dumps(res.events))
    assert len(events) == len(g["events"])
    for k, (mine, ref) in enumerate(zip(events, g["events"])):
        assert mine == ref, f"event {k}: {mine} != {ref}"
    assert hashlib.sha256(json.dumps(res.events, sort_keys=True).encode()).hexdigest() == g["events_sha256"]
    assert res.trajectory.winner == g["winner"]
    assert dict(res.final_balances) == g["final_balances"]
    return sess


@pytest.mark.parametrize("look_ahead", [False, True])
@pytest.mark.parametrize("case", [0, 1])
def test_session_rounds_on_oracle_equal_reference_event_log(case, look_ahead):
    g = golden()[case]
    sess = run_and_compare(g, predictor=OraclePredictor(session_config(g).race), look_ahead=look_ahead)
    st = sess.stats
    # one launch per wake round (plus discarded look-aheads), far fewer than one rp_predict per wake
    assert st.launches - st.ahead_misses <= st.rounds < st.predictions
    if look_ahead:
        # the first round of every call after the opening one was launched during the previous
        # call's exchange (later rounds of a call depend on its earlier decisions), none wasted
        assert st.ahead_hits > 0 and st.ahead_misses == 0
    else:
        assert st.ahead_hits == st.ahead_misses == 0


def test_decide_draws_match_reference_decide():
    """decide_draws advances a stream exactly as Bettor.decide does for RP and RB bettors (ties and
    no ties), whatever the book holds."""
    import random

    from racemarket.agents import AgentParams, RBBettor, RPBettor

    cfg = session_config(golden()[0])
    for cls, strat in ((RPBettor, "rp"), (RBBettor, "rb")):
        for probs in ((0.25, 0.25, 0.5), (0.4, 0.4, 0.2), (0.2, 0.3, 0.5), (1 / 3, 1 / 3, 1 / 3)):
            a = cls("a000." + strat, AgentParams(strat, d=0, max_stake=9), cfg.race, random.Random(5))
            a.predict = lambda obs, p=probs: p
            twin = random.Random(5)
            from racemarket.agents import Observation
            from racemarket.exchange import MarketBook

            book = MarketBook(cfg.race.competitor_ids, 0.05)
            obs = Observation(time=0.0, race_tick=0, positions=(0.0,) * 5, finish_ticks=(None,) * 5,
                              step_history=((),) * 5, grid=book.market_grid(3), my_bets=(), balance=10 ** 6)
            a.decide(obs)
            S.decide_draws(twin, probs, 9 if strat == "rb" else None)
            assert a.rng.getstate() == twin.getstate()


@pytest.mark.gpu
@pytest.mark.parametrize("case", [0, 1])
def test_gpu_session_mt_equals_reference_event_log(case):
    """The product path: every wake round one MT launch (DryRunDispatcher), the reference's exchange
    loop unchanged -- the event log, predictions, winner and balances equal the reference's."""
    g = golden()[case]
    sess = run_and_compare(g, mode="mt")
    assert sess.stats.launches - sess.stats.ahead_misses <= sess.stats.rounds and sess.stats.ahead_hits > 0


@pytest.mark.gpu
def test_gpu_session_native_modes_run():
    """NATIVE64 / NATIVE sessions run end to end through the same hooks (statistically equal
    predictions, so the log differs from the reference's) and keep every planned prediction."""
    g = golden()[0]
    for mode in ("native64", "native"):
        res, st = S.run_session_with_stats(session_config(g), mode=mode)
        assert st.fallbacks == 0 and st.predictions == len(g["predictions"])
        assert res.events[-1]["kind"] == "settle"
