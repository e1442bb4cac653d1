"""Simulation dispatch for the bettor-agent loop: batch every due RP/RB dry run.

In the reference every RP/RB wake runs ``rp_predict`` on its own: d sequential ``simulate_from``
calls (session.py:240-267 -> agents.py:345-362 -> agents.py:153-166).  Predictions depend only on
the live race state (never on the order book), and each bettor's dry-run seeds come from its own
private stream.  So all predictions a tick needs can run as ONE launch:
concatenate every requesting bettor's d seeds -- drawn from each bettor's stream in its own order,
exactly as ``rp_predict`` would -- simulate them together, and split the per-sim winners back per
bettor.  In MT mode every bettor then gets exactly the probabilities (and the stream position) the
reference would have produced; the exchange loop stays on the host and unchanged.

``run_dry_run_session`` drives the C4 workload without the exchange: the live race (the reference's
own race for ``derive_seed(master, "race")``, recorded tick by tick on the GPU in MT mode), the
jittered wake schedule of session.py:104-121, and one batched prediction launch per tick.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .agents import dry_run_seeds_many
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

    ``on_batch(predictions)`` -- the host's use of a batch (the exchange loop's decisions and order
    book in a full session) -- runs while the NEXT batch is already on the GPU: the race never depends
    on the market (session.py:282), so predictions run one batch ahead of the host.
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
        # a bettor waking k times in one batch needs its k-th prediction after its (k-1)-th decision;
        # RP decisions draw from the stream only on ties (agents.py:304-310), which this driver does
        # not model, so rounds are batched: round r = every bettor's r-th due wake.
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
    # (race state, wake round) batches is known: prepare batch i+1 on the host while batch i runs
    work = batches(opening_period, states[0])
    for tick in range(1, n_ticks + 1):
        if all(f is not None for f in states[tick].finish_ticks):
            break  # betting closes when the last runner finishes (BettingClose.last, session.py:294-311)
        work.extend(batches(opening_period + tick * config.dt, states[tick]))

    t0 = time.perf_counter()
    prev = None  # (batch, prepared, pending) in flight
    for state, rnd in work:
        prep = disp.prepare([DryRunRequest(rngs[i], d) for _, i in rnd])
        done = None
        if prev is not None:
            done = [(t, i, p) for (t, i), p in zip(prev[0], disp.finish(prev[2], prev[1]))]
            preds.extend(done)
        prev = (rnd, prep, disp.launch(state, prep))
        if done is not None and on_batch is not None:
            on_batch(done)  # overlaps the batch just launched
    if prev is not None:
        done = [(t, i, p) for (t, i), p in zip(prev[0], disp.finish(prev[2], prev[1]))]
        preds.extend(done)
        if on_batch is not None:
            on_batch(done)
    seconds = time.perf_counter() - t0
    return DryRunSessionResult(preds, disp.launches, disp.sims, seconds, n_ticks)
