"""Simulation dispatch for the bettor-agent loop: batch every due RP/RB dry run.

In the reference every RP/RB wake runs ``rp_predict`` on its own: d sequential ``simulate_from``
calls (session.py:240-267 -> agents.py:345-362 -> agents.py:153-166).  Predictions depend only on
the live race state (never on the order book), and each bettor's dry-run seeds come from its own
private stream.  So all predictions a wake round needs can run as ONE launch:
concatenate every requesting bettor's d seeds -- drawn from each bettor's stream in its own order,
exactly as ``rp_predict`` would -- simulate them together, and split the per-sim winners back per
bettor.  In MT mode every bettor then gets exactly the probabilities (and the stream position) the
reference would have produced.

``run_session`` / ``GpuSession`` is the full BBE session (C4): the reference's own session loop,
exchange, matching and settlement (racemarket.session._Session, session.py:124-340) with the
RP/RB predictions of every ``_process_wakes`` call served from batched launches.  The event log is
the reference's, byte for byte, in MT mode (tests/test_session_exchange.py).

``run_dry_run_session`` drives the prediction side of C4 alone (no exchange): the live race, the
jittered wake schedule of session.py:104-121, and one batched prediction launch per wake round.
"""

from __future__ import annotations

import ctypes
import os
import random
import sys
import time
from collections import deque
from dataclasses import dataclass

import numpy as np

from .agents import (_IDX_OFF, _inplace_ok, dry_run_seeds, dry_run_seeds_many, rb_bettor_predict, rb_weighted,
                     rp_bettor_predict)
from .race import RaceState
from .seeding import derive_seed, spawn_rng
from .sim import run_race, simulate_batch_begin


@dataclass
class DryRunRequest:
    """One bettor's prediction request: its private stream and its number of dry runs."""

    rng: object
    d: int


class DryRunDispatcher:
    """Batch the dry runs of every bettor that predicts from the same race state into one launch.

    ``predict_many`` = ``prepare`` (host: advance every bettor's stream, collect the seeds) ->
    ``launch`` (enqueue one batch) -> ``finish`` (wait, split the winners per bettor).  A caller
    with a queue of batches prepares batch i+1 while batch i runs on the GPU
    (``run_dry_run_session`` does).
    """

    def __init__(self, config, mode: str = "mt"):
        self.config = config
        self.mode = mode
        self.launches = 0
        self.sims = 0
        self._n = len(config.competitors)

    def prepare(self, requests: list[DryRunRequest]) -> dict:
        """Advance each bettor's stream exactly as its own ``rp_predict`` call would, in request
        order (bettors own disjoint streams, so the order across bettors does not matter)."""
        ds = [max(int(r.d), 0) for r in requests]
        total = sum(ds)
        prep = {"ds": ds, "total": total, "seeds": None, "key": 0}
        rngs = [r.rng for r in requests]
        if self.mode == "mt":
            seeds = dry_run_seeds_many(rngs, ds, ds)
            if total:
                prep["seeds"] = np.concatenate([s for s in seeds if s is not None and len(s)])
        else:
            # native: the batch's Philox stream is keyed by the first dry-run seed; every other draw
            # only advances its bettor's stream
            first = next((i for i, d in enumerate(ds) if d > 0), None)
            seeds = dry_run_seeds_many(rngs, ds, [1 if i == first else 0 for i in range(len(ds))])
            if first is not None:
                prep["key"] = int(seeds[first][0])
        return prep

    def launch(self, state, prep: dict):
        """Enqueue one batch for a prepared request list (None if it has no dry runs)."""
        if prep["total"] == 0:
            return None
        self.launches += 1
        self.sims += prep["total"]
        # equal d for every bettor (the session's case): per-bettor winner counts come from the
        # kernel (group_size = d); otherwise the per-sim winners are split on the host
        ds = [d for d in prep["ds"] if d > 0]
        g = ds[0] if len(set(ds)) == 1 else 0
        kw = dict(group_size=g) if g else dict(winners=True)
        if self.mode == "mt":
            return simulate_batch_begin(state, self.config, prep["total"], mode="mt", seeds=prep["seeds"],
                                        ranks=False, **kw)
        return simulate_batch_begin(state, self.config, prep["total"], prep["key"], mode=self.mode, ranks=False, **kw)

    def finish(self, pending, prep: dict) -> list[tuple[float, ...]]:
        """Laplace-smoothed win probabilities per request (agents.py:153-166), in request order."""
        n, ds = self._n, prep["ds"]
        if pending is None:
            return [tuple(1 / (d + n) for _ in range(n)) for d in ds]
        res = pending.end()
        if res.group_wins is not None:
            rows = iter(res.group_wins.tolist())
            wins = [next(rows) if d > 0 else [0] * n for d in ds]
        else:
            group = np.repeat(np.arange(len(ds)), ds)
            wins = np.bincount(group * n + res.winner, minlength=len(ds) * n).reshape(len(ds), n).tolist()
        return [tuple((w + 1) / (d + n) for w in row) for d, row in zip(ds, wins)]

    def predict_many(self, state, requests: list[DryRunRequest]) -> list[tuple[float, ...]]:
        """One batched prediction for every request, in request order."""
        prep = self.prepare(requests)
        return self.finish(self.launch(state, prep), prep)


def wake_schedule(reevaluate_every: list[float], wake_jitter: list[float], horizon: float, master_seed: int):
    """All (wake time, agent index) pairs with jitter + k * period <= horizon (session.py:104-121)."""
    wakes = []
    for i, (period, jit) in enumerate(zip(reevaluate_every, wake_jitter)):
        jitter = spawn_rng(master_seed, "jitter", i).uniform(0.0, jit)
        k = 0
        while k * period <= horizon:
            wakes.append((jitter + k * period, i))
            k += 1
    wakes.sort()
    return wakes


@dataclass
class DryRunSessionResult:
    predictions: list          # (time, agent index, probabilities) in processing order
    launches: int
    sims: int
    seconds: float
    ticks: int

    @property
    def sims_per_second(self) -> float:
        return self.sims / self.seconds if self.seconds > 0 else 0.0


def live_states(config, master_seed: int):
    """Per-tick RaceState an RP bettor reconstructs (agents.py:348-358) along the session's live race.

    The session races on spawn_rng(master, "race") (session.py:130, 143): the same stream as
    run_race(config, derive_seed(master, "race")).  Before the first tick the bettor sees empty step
    histories, i.e. previous steps 0.0.
    """
    traj, prevs = run_race(config, derive_seed(master_seed, "race"), record=True, mode="mt", with_prev_steps=True)
    fin = traj.finish_ticks
    states = []
    for t, row in enumerate(traj.ticks):
        prev = [0.0] * len(row) if t == 0 else [float(x) for x in prevs[t]]
        states.append(RaceState(t, list(row), prev, [f if f <= t else None for f in fin]))
    return states


def run_dry_run_session(config, n_agents: int, d: int, master_seed: int, *, opening_period: float = 5.0,
                        reevaluate_every: float = 1.0, wake_jitter: float = 1.0, mode: str = "mt",
                        agent_rngs=None, on_batch=None) -> DryRunSessionResult:
    """C4 without the exchange: n_agents RP bettors, each predicting with d dry runs at every wake.

    Time runs as in session.py:271-311: wakes up to the opening period see the pre-race state; then
    each race tick advances the clock by dt and processes the wakes due by then (one launch per
    batch of wakes that share a race state).  Returns every prediction and the end-to-end rate.

    Every bettor is an RP bettor whose decision draws from its stream only on an exact probability
    tie (``_pick``'s randrange, agents.py:304-310); that draw is made after each batch, so every
    stream stays where the reference's session leaves it.  ``on_batch(predictions)`` is called after
    each batch (it must not draw from the bettors' streams).  ``run_session`` is the full session
    with the exchange.
    """
    states = live_states(config, master_seed)
    n_ticks = len(states) - 1
    rngs = agent_rngs or [spawn_rng(master_seed, "agent", i) for i in range(n_agents)]
    next_wake = [spawn_rng(master_seed, "jitter", i).uniform(0.0, wake_jitter) for i in range(n_agents)]
    disp = DryRunDispatcher(config, mode)
    preds = []

    def batches(until: float, state):
        due = []
        for i in range(n_agents):
            while next_wake[i] <= until:
                due.append((next_wake[i], i))
                next_wake[i] += reevaluate_every
        due.sort()
        # a bettor waking k times in one batch needs its k-th prediction after its (k-1)-th decision,
        # so rounds are batched: round r = every bettor's r-th due wake.
        rounds: list[list[tuple[float, int]]] = []
        seen: dict[int, int] = {}
        for t, i in due:
            r = seen.get(i, 0)
            seen[i] = r + 1
            if r == len(rounds):
                rounds.append([])
            rounds[r].append((t, i))
        return [(state, rnd) for rnd in rounds]

    # the live race is fixed in advance (session.py:282 uses only rng_race), so the whole sequence of
    # (race state, wake round) batches is known up front.  Wakes stop once betting closes: at
    # close_rank finishers (session.py:294-311).
    close_rank = config.betting_close.close_rank(len(config.competitors))
    work = batches(opening_period, states[0])
    for tick in range(1, n_ticks + 1):
        if sum(f is not None for f in states[tick].finish_ticks) >= close_rank:
            break
        work.extend(batches(opening_period + tick * config.dt, states[tick]))

    t0 = time.perf_counter()
    for state, rnd in work:
        # a bettor's next seeds are drawn only after its previous decision's draws (the RP tie-break
        # randrange, agents.py:304-310), so a batch is prepared once the one before it is decided
        prep = disp.prepare([DryRunRequest(rngs[i], d) for _, i in rnd])
        done = [(t, i, p) for (t, i), p in zip(rnd, disp.finish(disp.launch(state, prep), prep))]
        for _, i, p in done:
            decide_draws(rngs[i], p, None)
        preds.extend(done)
        if on_batch is not None:
            on_batch(done)
    seconds = time.perf_counter() - t0
    return DryRunSessionResult(preds, disp.launches, disp.sims, seconds, n_ticks)


def decide_draws(rng, probs, max_stake: int | None) -> None:
    """The draws ``Bettor.decide`` makes from the bettor's stream after its prediction
    (agents.py:334-342): ``_pick``'s ``randrange`` over exactly tied maxima (agents.py:304-310), then
    for an RB bettor the stake ``randint(1, max_stake)`` (agents.py:406-408).  Neither depends on
    the order book, so the stream position after a decision is a function of the prediction alone.
    """
    best = max(probs)
    k = sum(1 for p in probs if p == best)
    if k > 1:
        rng.randrange(k)
    if max_stake is not None:
        rng.randint(1, max_stake)


# -- the full session: the reference's exchange loop with batched GPU predictions --------------------


def import_racemarket():
    """The reference package, whose session loop, exchange and agents run on the host unchanged.

    Imported as installed; else from ``$RACEMARKET_PATH`` or this checkout's ``baseline/_ref`` (the
    offline install of /root/reference)."""
    try:
        import racemarket.session  # noqa: F401
    except ImportError:
        here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        for p in (os.environ.get("RACEMARKET_PATH"), os.path.join(here, "baseline", "_ref")):
            if p and os.path.isdir(os.path.join(p, "racemarket")) and p not in sys.path:
                sys.path.append(p)
        import racemarket.session  # noqa: F401
    import racemarket

    return racemarket


def to_reference_race(config):
    """This package's RaceConfig as a ``racemarket.race.RaceConfig`` (same fields; race.py:99-189).
    A racemarket config is returned unchanged."""
    rm = import_racemarket()
    R = rm.race
    if isinstance(config, R.RaceConfig):
        return config
    comps = []
    for c in config.competitors:
        s = c.steps
        steps = (R.LogNormalSteps(s.mu, s.sigma, s.scale) if hasattr(s, "mu") else R.UniformSteps(s.lo, s.hi))
        r = c.responsiveness
        comps.append(R.Competitor(c.cid, steps, c.preference, c.pref_sensitivity, c.theta,
                                  R.Responsiveness(r.early_mult, r.late_mult, r.breakpoint)))
    bc = config.betting_close
    return R.RaceConfig(config.track_length, tuple(comps), dt=config.dt, conditions=config.conditions,
                        betting_close=R.BettingClose(bc.rule, bc.k), tick_limit=config.tick_limit)


def c4_session_config(race, *, n_agents: int = 100, d: int = 1000, master_seed: int = 20260818,
                      opening_period: float = 5.0, strategy: str = "rp"):
    """``SessionConfig(race, (AgentParams(strategy, count=n_agents, d=d,
    reevaluate_every=1.0, wake_jitter=1.0),), master_seed, opening_period=5.0)``."""
    rm = import_racemarket()
    group = rm.agents.AgentParams(strategy, count=n_agents, d=d, reevaluate_every=1.0, wake_jitter=1.0)
    return rm.session.SessionConfig(race=to_reference_race(race), agent_groups=(group,), master_seed=master_seed,
                                    opening_period=opening_period)


_MT_BYTES = 4 + 624 * 4  # RandomObject: int index, then uint32_t state[624] (agents.py layout)


def stream_fingerprint(rng):
    """The exact position of a bettor's MT19937 stream: the 2,500 bytes of index + state inside a
    CPython random.Random (layout verified once by agents._inplace_ok), else its getstate()."""
    if type(rng) is random.Random and _inplace_ok():
        return ctypes.string_at(id(rng) + _IDX_OFF, _MT_BYTES)
    return rng.getstate()


def clone_stream(rng, into: random.Random | None = None) -> random.Random:
    """A random.Random at the same stream position as ``rng`` (``into``, reused, or a new one): a
    memmove of the MT19937 fields when the layout is verified, else setstate(getstate())."""
    v = into if into is not None else random.Random(0)
    if type(rng) is random.Random and type(v) is random.Random and _inplace_ok():
        ctypes.memmove(id(v) + _IDX_OFF, id(rng) + _IDX_OFF, _MT_BYTES)
    else:
        v.setstate(rng.getstate())
    return v


@dataclass
class SessionStats:
    launches: int = 0          # batched prediction launches (look-ahead launches included)
    sims: int = 0              # dry runs simulated
    predictions: int = 0       # RP/RB predictions served from a batch
    fallbacks: int = 0         # predictions computed on their own (stream not where planned)
    rounds: int = 0            # wake rounds
    ahead_hits: int = 0        # rounds served by the launch made during the previous call's exchange
    ahead_misses: int = 0      # look-ahead launches discarded (their inputs did not come true)
    predict_seconds: float = 0.0  # host wall time inside the prediction planning (seeds + waits + tally)
    seconds: float = 0.0          # wall time of the whole session run


def make_gpu_session(config, *, mode: str = "mt", predictor=None, look_ahead: bool = True):
    """A ``racemarket.session._Session`` whose RP/RB bettors' predictions come from batched launches.

    ``predictor.predict_many(state, requests)`` serves a round (default: ``DryRunDispatcher(race,
    mode)``).  Everything else -- wake schedule, observations, ``decide``, the exchange, matching,
    close, settlement, the event log -- is the reference's own code (session.py:124-340).
    ``look_ahead`` (predictors with ``prepare``/``launch``/``finish``): the next call's first round
    is launched before this call's exchange runs, so the GPU works while the host matches orders.
    """
    rm = import_racemarket()
    from racemarket.agents import RBBettor, RPBettor
    from racemarket.race import advance_race

    class GpuSession(rm.session._Session):
        """session.py:_Session with ``_process_wakes`` (session.py:258-267) prefetching predictions.

        For one ``_process_wakes(until)`` call the due wakes are computed exactly as the reference
        computes them (on a copy of ``next_wake``).  RP/RB wakes are grouped into rounds -- round r
        holds every bettor's r-th due wake -- and each round is ONE batched launch from the race state
        of this call (the race does not move inside a call).  Round r's seeds come from a clone of
        the bettor's stream advanced past its earlier predictions and decisions (``decide_draws``).
        Then the reference's own loop runs the wakes in (time, index) order; each RP/RB ``predict``
        pops its planned probabilities after checking that the bettor's real stream is exactly
        where the plan drew the seeds, and advances it by d ``getrandbits(64)`` as ``rp_predict``
        does (agents.py:164).  A stream found anywhere else is predicted on its own (GPU, same
        mode), so the result never depends on the plan being right.

        Look-ahead (§8f-1): the live race never depends on the market (session.py:282 advances it
        with ``rng_race`` alone) and a bettor's stream after its decision depends only on its
        prediction, so once a call's rounds are planned, the next call's first round is fully
        determined: its race state (one ``advance_race`` of a clone of the state and of
        ``rng_race``), its due wakes (the schedule) and every member's stream position.  It is
        launched right away and runs on the GPU while the reference processes this call's wakes; the
        next call uses it only if its until, members, race state and stream positions all match.
        """

        def __init__(self, cfg):
            super().__init__(cfg)
            self.bbe_mode = mode
            self.predictor = predictor if predictor is not None else DryRunDispatcher(cfg.race, mode)
            self.stats = SessionStats()
            self._plans: dict[int, deque] = {}
            self._batched: dict[int, object] = {}
            self._virt: dict[int, random.Random] = {}   # per bettor: the planning clone of its stream
            self._avirt: dict[int, random.Random] = {}  # per bettor: the look-ahead clone
            for i, a in enumerate(self.agents):
                if type(a) in (RPBettor, RBBettor) and type(a.rng) is random.Random:
                    self._batched[i] = a
                    self._plans[i] = deque()
                    self._virt[i] = random.Random(0)
                    self._avirt[i] = random.Random(0)
                    a.predict = self._hook(i, a)  # instance attribute: shadows the class method
            self._look_ahead = look_ahead and all(hasattr(self.predictor, f) for f in ("prepare", "launch", "finish"))
            self._ahead = None
            self._race_clone = random.Random(0)
            self._close_rank = cfg.race.betting_close.close_rank(self.n)

        def _hook(self, i, agent):
            rb = isinstance(agent, RBBettor)
            d = agent.params.d

            def predict(obs):
                q = self._plans[i]
                if q:
                    expect, probs = q.popleft()
                    if stream_fingerprint(agent.rng) == expect:
                        dry_run_seeds(agent.rng, d, want=False)
                        return probs
                    q.clear()  # the stream moved off the plan: later planned wakes are void too
                self.stats.fallbacks += 1
                if rb:
                    return rb_bettor_predict(obs, self.race_cfg, d, agent.params.gamma, agent.rng, mode=self.bbe_mode)
                return rp_bettor_predict(obs, self.race_cfg, d, agent.rng, mode=self.bbe_mode)

            return predict

        def _due(self, until: float, nw: list) -> list:
            """session.py:259-264 on the wake times ``nw`` (advanced in place)."""
            due = []
            for i, agent in enumerate(self.agents):
                period = agent.params.reevaluate_every
                while nw[i] <= until:
                    due.append((nw[i], i))
                    nw[i] += period
            due.sort()
            return due

        def _process_wakes(self, until: float) -> None:
            nw = list(self.next_wake)
            due = self._due(until, nw)
            positions, finish_ticks, history = self._race_view()
            state = RaceState(self.state.tick, list(positions), [h[-1] if h else 0.0 for h in history],
                              list(finish_ticks))
            t0 = time.perf_counter()
            count = self._prefetch(due, state, until)
            if self._look_ahead:
                self._launch_ahead(nw, count)
            self.stats.predict_seconds += time.perf_counter() - t0
            super()._process_wakes(until)

        def _members(self, due, r: int) -> list:
            """The batched bettors of round r of a due list (their r-th wake), in due order."""
            seen: dict[int, int] = {}
            out = []
            for _, i in due:
                if i in self._batched:
                    k = seen.get(i, 0)
                    seen[i] = k + 1
                    if k == r:
                        out.append(i)
            return out

        def _prefetch(self, due, state, until) -> dict:
            count: dict[int, int] = {}
            for _, i in due:
                if i in self._batched:
                    count[i] = count.get(i, 0) + 1
            ahead, self._ahead = self._ahead, None
            if not count:
                if ahead is not None:
                    self._drop(ahead)
                return count
            virt = {i: clone_stream(self._batched[i].rng, self._virt[i]) for i in count}
            for r in range(max(count.values())):
                members = [i for i in count if count[i] > r]
                expects = [stream_fingerprint(virt[i]) for i in members]
                probs = None
                if r == 0 and ahead is not None:
                    if (ahead["until"] == until and ahead["members"] == members and ahead["state"] == _sig(state)
                            and ahead["expects"] == expects):
                        probs = self.predictor.finish(ahead["pending"], ahead["prep"])
                        for i in members:
                            clone_stream(self._avirt[i], virt[i])  # advanced past its d seeds by prepare
                        self.stats.ahead_hits += 1
                    else:
                        self._drop(ahead)
                    ahead = None
                if probs is None:
                    reqs = [DryRunRequest(virt[i], self._batched[i].params.d) for i in members]
                    probs = self.predictor.predict_many(state, reqs)
                self.stats.rounds += 1
                for i, e, p in zip(members, expects, probs):
                    a = self._batched[i]
                    rb = isinstance(a, RBBettor)
                    out = rb_weighted(p, a.params.gamma) if rb else tuple(p)
                    self._plans[i].append((e, out))
                    decide_draws(virt[i], out, a.params.max_stake if rb else None)
                self.stats.predictions += len(members)
            if ahead is not None:
                self._drop(ahead)
            self._sync_counts()
            return count

        def _launch_ahead(self, nw: list, count: dict) -> None:
            """Launch the next call's first round now (see the class docstring)."""
            if self.state.all_finished() or self.state.tick >= self.race_cfg.tick_limit:
                return
            st = self.state.clone()
            rng = clone_stream(self.rng_race, self._race_clone)
            racing_before = [t is None for t in st.finish_ticks]
            advance_race(st, self.race_cfg, rng)
            if st.finished_count() >= self._close_rank:
                return  # betting closes on that tick: no wakes (session.py:294-311)
            until = self.config.opening_period + st.tick * self.race_cfg.dt
            due = self._due(until, list(nw))
            members = self._members(due, 0)
            if not members:
                return
            hist = self.histories
            prev = [st.prev_steps[c] if racing_before[c] else (hist[c][-1] if hist[c] else 0.0) for c in range(self.n)]
            state = RaceState(st.tick, list(st.positions), prev, list(st.finish_ticks))
            # member streams now: the planned clone for bettors of this call, the real stream otherwise
            src = {i: (self._virt[i] if i in count else self._batched[i].rng) for i in members}
            expects = [stream_fingerprint(src[i]) for i in members]
            la = [clone_stream(src[i], self._avirt[i]) for i in members]
            prep = self.predictor.prepare([DryRunRequest(v, self._batched[i].params.d) for v, i in zip(la, members)])
            pending = self.predictor.launch(state, prep)
            self._ahead = {"until": until, "members": members, "state": _sig(state), "expects": expects,
                           "prep": prep, "pending": pending}

        def _drop(self, ahead) -> None:
            """Discard a look-ahead launch whose inputs did not come true: wait for it (releasing its
            launch context) and ignore its outcome -- the reference never runs that prediction, so
            not even its failure (e.g. a diverged dry run) may surface."""
            self.stats.ahead_misses += 1
            try:
                self.predictor.finish(ahead["pending"], ahead["prep"])
            except Exception:  # noqa: BLE001 -- an unused prediction's error is not the session's
                pass

        def _sync_counts(self) -> None:
            self.stats.launches = getattr(self.predictor, "launches", 0)
            self.stats.sims = getattr(self.predictor, "sims", 0)

        def run(self):
            try:
                return super().run()
            finally:
                if self._ahead is not None:
                    self._drop(self._ahead)
                    self._ahead = None
                self._sync_counts()

    return GpuSession(config)


def _sig(state) -> tuple:
    """Exact identity of a RaceState as a bettor reconstructs it."""
    return (state.tick, tuple(state.positions), tuple(state.prev_steps), tuple(state.finish_ticks))


def run_session(config, *, mode: str = "mt", predictor=None, look_ahead: bool = True):
    """``racemarket.session.run_session`` (session.py:345-347) with batched GPU predictions.

    mode="mt": every prediction, and so the whole event log, settlement and balances, equals the
    reference's; "native64"/"native": Philox dry runs (statistically equal predictions).  Returns
    the reference's ``SessionResult``."""
    return run_session_with_stats(config, mode=mode, predictor=predictor, look_ahead=look_ahead)[0]


def run_session_with_stats(config, *, mode: str = "mt", predictor=None, look_ahead: bool = True):
    """``run_session`` plus the dispatch counters (``SessionStats``) and the wall time of ``run``."""
    s = make_gpu_session(config, mode=mode, predictor=predictor, look_ahead=look_ahead)
    t0 = time.perf_counter()
    res = s.run()
    s.stats.seconds = time.perf_counter() - t0
    return res, s.stats
