"""Pure-Python restatement of the reference hot path -- TEST INFRASTRUCTURE / CPU BASELINE ONLY.

Same language and same RNG (CPython ``random.Random``, MT19937) as the reference, so it produces
the reference's exact outputs; it runs about 1.35x faster than ``racemarket`` itself (measured on C2:
692 vs 512 races/s on one core -- it hoists the per-step constants the reference recomputes).
``bench.py`` times the reference itself (``racemarket`` from ``baseline/_ref``) and falls back to
this restatement, labelled kind "port", only where that install is missing.  Pinned against the
reference by tests/test_oracle_golden.py.

Follows /root/reference/pkg/src/racemarket/:
  race.py:192-199 preference_factor, :93-96 responsiveness, :233-241 initial_state,
  :244-274 front runner + step resolution, :287-320 advance, :323-332 finish order,
  :373-390 run_race, :393-406 simulate_from; agents.py:153-166 rp_predict;
  seeding.py:24-64 derive_seed / make_rng; batch.py:110-124 run_batch fan-out.
"""

from __future__ import annotations

import math
import os
import random
from concurrent.futures import ProcessPoolExecutor

M64 = (1 << 64) - 1


class Diverged(RuntimeError):
    pass


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def _fnv(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & M64
    return h


def derive_seed(master: int, *path) -> int:
    h = splitmix64(master & M64)
    for part in path:
        enc = b"s:" + part.encode() if isinstance(part, str) else b"i:" + (part & M64).to_bytes(8, "big")
        h = splitmix64(h ^ _fnv(enc))
    return h


def preference_factor(conditions: float, preference: float, sensitivity: float) -> float:
    f = 1.0 - sensitivity * abs(conditions - preference)
    return 0.01 if f < 0.01 else (1.0 if f > 1.0 else f)


class _Field:
    """Flattened per-competitor parameters of a (duck-typed) race config."""

    def __init__(self, cfg):
        self.n = len(cfg.competitors)
        self.L = float(cfg.track_length)
        self.limit = int(cfg.tick_limit)
        self.pref = []
        self.bp = []
        self.early = []
        self.late = []
        self.theta = []
        self.draw = []
        for c in cfg.competitors:
            self.pref.append(preference_factor(cfg.conditions, c.preference, c.pref_sensitivity))
            r = c.responsiveness
            self.bp.append(r.breakpoint * self.L)
            self.early.append(r.early_mult)
            self.late.append(r.late_mult)
            self.theta.append(c.theta)
            s = c.steps
            if hasattr(s, "lo"):
                lo, hi = s.lo, s.hi
                self.draw.append(lambda rng, lo=lo, hi=hi: rng.uniform(lo, hi))
            else:
                mu, sg, sc = s.mu, s.sigma, s.scale
                self.draw.append(lambda rng, mu=mu, sg=sg, sc=sc: sc * rng.lognormvariate(mu, sg))


def _tick(f: _Field, pos, prev, fin, tick, rng):
    n = f.n
    steps = [0.0] * n
    blocked = 0
    for c in range(n):
        if fin[c] is not None:
            continue
        pc = pos[c]
        resp = f.early[c] if pc < f.bp[c] else f.late[c]
        bi, bg = -1, 0.0
        for i in range(n):
            if i != c and fin[i] is None and pos[i] > pc:
                g = pos[i] - pc
                if bi < 0 or g < bg:
                    bi, bg = i, g
        if bi < 0 or bg > f.theta[c]:
            steps[c] = resp * f.pref[c] * f.draw[c](rng)
        else:
            steps[c] = resp * min(prev[c], prev[bi])
            blocked += 1
    t = tick + 1
    for c in range(n):
        if fin[c] is None:
            p = pos[c] + steps[c]
            if p == pos[c]:
                p = math.nextafter(p, math.inf)
            pos[c] = p
            prev[c] = steps[c]
            if p >= f.L:
                fin[c] = t
    return t, blocked


def _order(f: _Field, pos, fin):
    return tuple(sorted(range(f.n), key=lambda c: (fin[c], f.L - pos[c], c)))


def run_race(cfg, seed: int, f: _Field | None = None) -> dict:
    f = f or _Field(cfg)
    rng = random.Random(seed & M64)
    prev = [(f.early[c] if 0.0 < f.bp[c] else f.late[c]) * f.pref[c] * f.draw[c](rng) for c in range(f.n)]
    pos = [0.0] * f.n
    fin = [None] * f.n
    tick, blocked, ct = 0, 0, 0
    while any(t is None for t in fin):
        if tick >= f.limit:
            raise Diverged(f"race exceeded tick_limit={f.limit}")
        ct += sum(t is None for t in fin)
        tick, b = _tick(f, pos, prev, fin, tick, rng)
        blocked += b
    return {"order": _order(f, pos, fin), "finish_ticks": fin, "positions": pos, "blocked": blocked, "ct": ct}


def simulate_from(state, cfg, seed: int, f: _Field | None = None) -> dict:
    f = f or _Field(cfg)
    rng = random.Random(seed & M64)
    pos, prev, fin = list(state.positions), list(state.prev_steps), list(state.finish_ticks)
    tick = start = state.tick
    blocked, ct = 0, 0
    while any(t is None for t in fin):
        if tick - start >= f.limit:
            raise Diverged(f"continuation exceeded tick_limit={f.limit}")
        ct += sum(t is None for t in fin)
        tick, b = _tick(f, pos, prev, fin, tick, rng)
        blocked += b
    return {"order": _order(f, pos, fin), "finish_ticks": fin, "positions": pos, "blocked": blocked, "ct": ct}


def rp_predict(state, cfg, d: int, rng) -> tuple[float, ...]:
    f = _Field(cfg)
    wins = [0] * f.n
    for _ in range(d):
        wins[simulate_from(state, cfg, rng.getrandbits(64), f)["order"][0]] += 1
    return tuple((w + 1) / (d + f.n) for w in wins)


# -- multi-process fan-out (batch.py:120-124 style) for the CPU baseline ---------------------------

_G: dict = {}


def _init(cfg, state):
    _G["cfg"], _G["state"], _G["f"] = cfg, state, _Field(cfg)


def _chunk(args):
    seeds = args
    cfg, state, f = _G["cfg"], _G["state"], _G["f"]
    wins = [0] * f.n
    ct = 0
    for s in seeds:
        out = run_race(cfg, s, f) if state is None else simulate_from(state, cfg, s, f)
        wins[out["order"][0]] += 1
        ct += out["ct"]
    return wins, ct


def batch_tally(cfg, seeds, state=None, workers: int = 1):
    """Winner tallies and competitor-timesteps over explicit seeds; workers > 1 uses processes."""
    seeds = [int(s) for s in seeds]
    if workers <= 1:
        _init(cfg, state)
        return _chunk(seeds)
    k = max(1, len(seeds) // (workers * 8))
    chunks = [seeds[i:i + k] for i in range(0, len(seeds), k)]
    n = len(cfg.competitors)
    wins, ct = [0] * n, 0
    with ProcessPoolExecutor(max_workers=workers, initializer=_init, initargs=(cfg, state)) as pool:
        for w, c in pool.map(_chunk, chunks):
            wins = [a + b for a, b in zip(wins, w)]
            ct += c
    return wins, ct


class TallyPool:
    """A persistent process pool over (cfg, state) for repeated timed batches."""

    def __init__(self, cfg, state=None, workers: int = 1):
        self.cfg, self.state, self.workers = cfg, state, workers
        self.pool = ProcessPoolExecutor(max_workers=workers, initializer=_init, initargs=(cfg, state))
        list(self.pool.map(_chunk, [[1]] * workers))  # start every worker before timing

    def run(self, seeds):
        seeds = [int(s) for s in seeds]
        k = max(1, len(seeds) // (self.workers * 4))
        chunks = [seeds[i:i + k] for i in range(0, len(seeds), k)]
        n = len(self.cfg.competitors)
        wins, ct = [0] * n, 0
        for w, c in self.pool.map(_chunk, chunks):
            wins = [a + b for a, b in zip(wins, w)]
            ct += c
        return wins, ct

    def close(self):
        self.pool.shutdown()


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
