"""CPU oracle for the race-simulation hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package, and only as the checker / CPU baseline.  The
product package ``paper_2108_02419_b200`` never imports it and has no CPU fallback.

Two restatements live here:

* ``bbe_oracle.c`` (loaded through ctypes below): MT19937/CPython ``random`` + the race engine of
  ``/root/reference/pkg/src/racemarket/race.py:192-406``.  It can generate the reference's draws
  from seeds, replay recorded draws, and run multi-threaded batches (the C CPU baseline).
* ``pyref.py``: a pure-Python restatement on ``random.Random`` (the reference's own language and
  RNG), used as the reference-speed CPU baseline.

Parity pin: ``tests/test_oracle_golden.py`` checks both against vectors produced by running the
reference itself (``tests/golden/make_golden.py``, fixtures committed under ``tests/golden/``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libbbe_oracle.so")

ORC_OK, ORC_EINVAL, ORC_EDIVERGED, ORC_EDRAWS = 0, 1, 2, 3


class OrcComp(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("lo", ctypes.c_double),
        ("hi", ctypes.c_double),
        ("mu", ctypes.c_double),
        ("sigma", ctypes.c_double),
        ("scale", ctypes.c_double),
        ("preference", ctypes.c_double),
        ("pref_sensitivity", ctypes.c_double),
        ("theta", ctypes.c_double),
        ("early_mult", ctypes.c_double),
        ("late_mult", ctypes.c_double),
        ("breakpoint", ctypes.c_double),
    ]


class OrcRace(ctypes.Structure):
    _fields_ = [
        ("track_length", ctypes.c_double),
        ("conditions", ctypes.c_double),
        ("tick_limit", ctypes.c_int64),
        ("n", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
    ]


class OrcOut(ctypes.Structure):
    _fields_ = [
        ("finish_ticks", ctypes.POINTER(ctypes.c_int64)),
        ("order", ctypes.POINTER(ctypes.c_int32)),
        ("final_pos", ctypes.POINTER(ctypes.c_double)),
        ("blocked", ctypes.c_int64),
        ("draws_used", ctypes.c_int64),
        ("n_ticks_run", ctypes.c_int64),
        ("ct", ctypes.c_int64),
    ]


_lib = None


def build() -> str:
    """Compile libbbe_oracle.so with the committed Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "bbe_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER
        d, i64, u64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32
        L.orc_run_race.argtypes = [P(OrcRace), P(OrcComp), u64, P(d), i64, P(d), i64, P(OrcOut)]
        L.orc_simulate_from.argtypes = [P(OrcRace), P(OrcComp), i64, P(d), P(d), P(i64), u64, P(d), i64,
                                        P(d), i64, P(OrcOut)]
        L.orc_advance_from_start.argtypes = [P(OrcRace), P(OrcComp), u64, i64, P(i64), P(d), P(d), P(i64),
                                             P(i64)]
        L.orc_batch.argtypes = [P(OrcRace), P(OrcComp), i32, i64, P(d), P(d), P(i64), i64, P(u64), u64,
                                i32, P(u64), P(u64), P(i32), P(i64), P(i64), P(i64)]
        L.orc_batch_px.argtypes = [P(OrcRace), P(OrcComp), i32, i64, P(d), P(d), P(i64), i64, i64, u64, i32,
                                   P(u64), P(u64), P(i32), P(i64), P(d), P(i64), P(i64), P(i64), P(i64)]
        L.orc_philox4x32_10.argtypes = [P(ctypes.c_uint32), u64, P(ctypes.c_uint32)]
        L.orc_mt_random.argtypes = [u64, i64, P(d)]
        L.orc_mt_uniform.argtypes = [u64, d, d, i64, P(d)]
        L.orc_mt_getrandbits64.argtypes = [u64, i64, P(u64)]
        L.orc_mt_lognormvariate.argtypes = [u64, d, d, i64, P(d)]
        L.orc_derive_seed_run.argtypes = [u64, u64]
        L.orc_derive_seed_run.restype = u64
        L.orc_splitmix64.argtypes = [u64]
        L.orc_splitmix64.restype = u64
        L.orc_preference_factor.argtypes = [d, d, d]
        L.orc_preference_factor.restype = d
        _lib = L
    return _lib


def _ptr(a, ct):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ct))


# -- config conversion (duck-typed: works for racemarket and paper_2108_02419_b200 types) --------


def pack_race(cfg):
    n = len(cfg.competitors)
    race = OrcRace(float(cfg.track_length), float(cfg.conditions), int(cfg.tick_limit), n, 0)
    comps = (OrcComp * n)()
    for k, c in enumerate(cfg.competitors):
        s = c.steps
        r = c.responsiveness
        o = comps[k]
        if hasattr(s, "lo"):
            o.family, o.lo, o.hi = 0, float(s.lo), float(s.hi)
        else:
            o.family, o.mu, o.sigma, o.scale = 1, float(s.mu), float(s.sigma), float(s.scale)
        o.preference, o.pref_sensitivity, o.theta = float(c.preference), float(c.pref_sensitivity), float(c.theta)
        o.early_mult, o.late_mult, o.breakpoint = float(r.early_mult), float(r.late_mult), float(r.breakpoint)
    return race, comps


def _fin_array(finish_ticks):
    return np.array([-1 if t is None else int(t) for t in finish_ticks], dtype=np.int64)


class RaceOut:
    def __init__(self, rc, n, draws=None):
        self.rc = rc
        self.finish_ticks = np.zeros(n, np.int64)
        self.order = np.zeros(n, np.int32)
        self.final_positions = np.zeros(n, np.float64)
        self.blocked = 0
        self.draws_used = 0
        self.n_ticks_run = 0
        self.ct = 0
        self.draws = draws

    def _out(self):
        return OrcOut(_ptr(self.finish_ticks, ctypes.c_int64), _ptr(self.order, ctypes.c_int32),
                      _ptr(self.final_positions, ctypes.c_double), 0, 0, 0, 0)

    def _take(self, o, rc):
        self.rc = rc
        self.blocked, self.draws_used, self.n_ticks_run, self.ct = o.blocked, o.draws_used, o.n_ticks_run, o.ct
        if self.draws is not None:
            self.draws = self.draws[: self.draws_used].copy()
        return self


def run_race(cfg, seed: int, replay=None, record: bool = False, rec_cap: int = 1 << 20) -> RaceOut:
    """Oracle run_race (race.py:373-390): MT(seed) draws, or a replay of recorded draws."""
    race, comps = pack_race(cfg)
    n = race.n
    rec = np.zeros(rec_cap, np.float64) if record else None
    res = RaceOut(0, n, rec)
    o = res._out()
    rp = None if replay is None else np.ascontiguousarray(replay, np.float64)
    rc = lib().orc_run_race(ctypes.byref(race), comps, seed & 0xFFFFFFFFFFFFFFFF, _ptr(rp, ctypes.c_double),
                            0 if rp is None else len(rp), _ptr(rec, ctypes.c_double), 0 if rec is None else rec_cap,
                            ctypes.byref(o))
    return res._take(o, rc)


def simulate_from(state, cfg, seed: int, replay=None, record: bool = False, rec_cap: int = 1 << 20) -> RaceOut:
    """Oracle simulate_from (race.py:393-406)."""
    race, comps = pack_race(cfg)
    n = race.n
    pos = np.array(state.positions, np.float64)
    prev = np.array(state.prev_steps, np.float64)
    fin = _fin_array(state.finish_ticks)
    rec = np.zeros(rec_cap, np.float64) if record else None
    res = RaceOut(0, n, rec)
    o = res._out()
    rp = None if replay is None else np.ascontiguousarray(replay, np.float64)
    rc = lib().orc_simulate_from(ctypes.byref(race), comps, int(state.tick), _ptr(pos, ctypes.c_double),
                                 _ptr(prev, ctypes.c_double), _ptr(fin, ctypes.c_int64),
                                 seed & 0xFFFFFFFFFFFFFFFF, _ptr(rp, ctypes.c_double),
                                 0 if rp is None else len(rp), _ptr(rec, ctypes.c_double),
                                 0 if rec is None else rec_cap, ctypes.byref(o))
    return res._take(o, rc)


def advance_from_start(cfg, seed: int, k: int):
    """initial_state + k advance_race ticks on make_rng(seed); returns (tick, pos, prev, fin, blocked)."""
    race, comps = pack_race(cfg)
    n = race.n
    tick = ctypes.c_int64(0)
    blocked = ctypes.c_int64(0)
    pos, prev, fin = np.zeros(n), np.zeros(n), np.zeros(n, np.int64)
    lib().orc_advance_from_start(ctypes.byref(race), comps, seed, k, ctypes.byref(tick), _ptr(pos, ctypes.c_double),
                                 _ptr(prev, ctypes.c_double), _ptr(fin, ctypes.c_int64), ctypes.byref(blocked))
    return tick.value, pos, prev, fin, blocked.value


def batch(cfg, n_sims: int, *, state=None, seeds=None, master: int = 0, threads: int = 1, winners=False):
    """Tallies over n_sims oracle sims: from the start line (state None, run_race) or simulate_from.

    seeds: per-sim seeds (u64 array); default derive_seed(master, "run", i) as batch.py:117-119.
    Returns dict(wins, ranks, winners, ct, blocked, rc, first_diverged).
    """
    race, comps = pack_race(cfg)
    n = race.n
    wins = np.zeros(n, np.uint64)
    ranks = np.zeros(n * n, np.uint64)
    win_arr = np.zeros(n_sims, np.int32) if winners else None
    ct, blk, fd = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    sd = None if seeds is None else np.ascontiguousarray(seeds, np.uint64)
    if state is None:
        rc = lib().orc_batch(ctypes.byref(race), comps, 1, 0, None, None, None, n_sims, _ptr(sd, ctypes.c_uint64),
                             master, threads, _ptr(wins, ctypes.c_uint64), _ptr(ranks, ctypes.c_uint64),
                             _ptr(win_arr, ctypes.c_int32), ctypes.byref(ct), ctypes.byref(blk), ctypes.byref(fd))
    else:
        pos = np.array(state.positions, np.float64)
        prev = np.array(state.prev_steps, np.float64)
        fin = _fin_array(state.finish_ticks)
        rc = lib().orc_batch(ctypes.byref(race), comps, 0, int(state.tick), _ptr(pos, ctypes.c_double),
                             _ptr(prev, ctypes.c_double), _ptr(fin, ctypes.c_int64), n_sims,
                             _ptr(sd, ctypes.c_uint64), master, threads, _ptr(wins, ctypes.c_uint64),
                             _ptr(ranks, ctypes.c_uint64), _ptr(win_arr, ctypes.c_int32), ctypes.byref(ct),
                             ctypes.byref(blk), ctypes.byref(fd))
    return dict(wins=wins, ranks=ranks.reshape(n, n), winners=win_arr, ct=ct.value, blocked=blk.value, rc=rc,
                first_diverged=fd.value)


def batch_px(cfg, n_sims: int, key: int, *, state=None, sim_offset: int = 0, threads: int = 1,
             records: bool = False):
    """The NATIVE64 stream (native64_kernel.cuh) on the CPU: sims sim_offset .. sim_offset + n_sims - 1 of
    the Philox4x32-10 stream keyed by ``key``, the reference's race engine in FP64.  Returns dict(wins,
    ranks, ct, blocked, rc, first_diverged) and, with records=True, order / finish_ticks /
    final_positions / blocked_per_sim arrays."""
    race, comps = pack_race(cfg)
    n = race.n
    wins = np.zeros(n, np.uint64)
    ranks = np.zeros(n * n, np.uint64)
    order = fin = fpos = blk = None
    if records:
        order = np.zeros((n_sims, n), np.int32)
        fin = np.zeros((n_sims, n), np.int64)
        fpos = np.zeros((n_sims, n), np.float64)
        blk = np.zeros(n_sims, np.int64)
    ct, bl, fd = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    if state is None:
        args = (1, 0, None, None, None)
    else:
        pos = np.array(state.positions, np.float64)
        prev = np.array(state.prev_steps, np.float64)
        f0 = _fin_array(state.finish_ticks)
        args = (0, int(state.tick), _ptr(pos, ctypes.c_double), _ptr(prev, ctypes.c_double), _ptr(f0, ctypes.c_int64))
    rc = lib().orc_batch_px(ctypes.byref(race), comps, *args, int(n_sims), int(sim_offset), key & 0xFFFFFFFFFFFFFFFF,
                            threads, _ptr(wins, ctypes.c_uint64), _ptr(ranks, ctypes.c_uint64),
                            _ptr(order, ctypes.c_int32), _ptr(fin, ctypes.c_int64), _ptr(fpos, ctypes.c_double),
                            _ptr(blk, ctypes.c_int64), ctypes.byref(ct), ctypes.byref(bl), ctypes.byref(fd))
    out = dict(wins=wins, ranks=ranks.reshape(n, n), ct=ct.value, blocked=bl.value, rc=rc, first_diverged=fd.value)
    if records:
        out.update(order=order, finish_ticks=fin, final_positions=fpos, blocked_per_sim=blk)
    return out


def philox4x32_10(counter, key: int) -> list:
    """One Philox4x32-10 block: four counter words and a 64-bit key -> four output words."""
    c = np.array(counter, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_ptr(c, ctypes.c_uint32), key & 0xFFFFFFFFFFFFFFFF, _ptr(out, ctypes.c_uint32))
    return [int(x) for x in out]


def rp_seeds(agent_seed: int, d: int) -> np.ndarray:
    """The d dry-run seeds rp_predict draws from make_rng(agent_seed) (agents.py:164)."""
    out = np.zeros(d, np.uint64)
    lib().orc_mt_getrandbits64(agent_seed, d, _ptr(out, ctypes.c_uint64))
    return out


def mt_random(seed: int, k: int) -> np.ndarray:
    out = np.zeros(k)
    lib().orc_mt_random(seed, k, _ptr(out, ctypes.c_double))
    return out


def mt_uniform(seed: int, a: float, b: float, k: int) -> np.ndarray:
    out = np.zeros(k)
    lib().orc_mt_uniform(seed, a, b, k, _ptr(out, ctypes.c_double))
    return out


def mt_getrandbits64(seed: int, k: int) -> np.ndarray:
    out = np.zeros(k, np.uint64)
    lib().orc_mt_getrandbits64(seed, k, _ptr(out, ctypes.c_uint64))
    return out


def mt_lognormvariate(seed: int, mu: float, sigma: float, k: int) -> np.ndarray:
    out = np.zeros(k)
    lib().orc_mt_lognormvariate(seed, mu, sigma, k, _ptr(out, ctypes.c_double))
    return out


def derive_seed_run(master: int, i: int) -> int:
    return int(lib().orc_derive_seed_run(master & 0xFFFFFFFFFFFFFFFF, i & 0xFFFFFFFFFFFFFFFF))
