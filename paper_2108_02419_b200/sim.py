"""ctypes binding of the C-ABI (include/bbe_sim.h) and the batched simulation API.

``simulate_batch`` is the one call everything else goes through: it packs a race (reference
``RaceConfig`` / ``RaceState`` or this package's mirrors, duck-typed) into the POD structs of the
header, hoists the two per-competitor constants the reference recomputes every step
(``preference_factor``, race.py:192-199, and ``breakpoint * track_length``, race.py:94) in Python
double exactly as the reference evaluates them, and calls ``bbe_simulate``.

There is no CPU path: if ``_lib/libbbe_sim.so`` is missing or no GPU is visible, calls raise
``BackendUnavailable``.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
from dataclasses import dataclass

import numpy as np

from .race import (
    RaceConfigError,
    RaceDivergedError,
    Trajectory,
    preference_factor,
    validate_config,
)

_LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
LIB_PATH = os.environ.get("BBE_LIB") or os.path.join(_LIB_DIR, "libbbe_sim.so")  # BBE_LIB: A/B builds

BBE_OK, BBE_EINVAL, BBE_EDIVERGED, BBE_EDRAWS, BBE_ECUDA, BBE_ENODEV, BBE_ENCCL = range(7)
MODES = {"native": 0, "inject": 1, "mt": 2, "native64": 3}
MAX_COMPETITORS = 128
MAX_PERM_COMPETITORS = 6
M64 = (1 << 64) - 1

ABI_VERSION = 5  # include/bbe_sim.h BBE_ABI_VERSION

EXPORTED_SYMBOLS = (
    "bbe_simulate",
    "bbe_simulate_begin",
    "bbe_simulate_end",
    "bbe_simulate_async",
    "bbe_simulate_multi",
    "bbe_tally_len",
    "bbe_tally_offset",
    "bbe_derive_seeds",
    "bbe_last_error",
    "bbe_version",
    "bbe_device_count",
    "bbe_device_info",
    "bbe_last_kernel_ms",
    "bbe_param_bytes",
    "bbe_mt_getrandbits64",
    "bbe_mt_exp_exact",
    "bbe_mt_advance64",
    "bbe_mt_advance64_many",
    "bbe_rp_predict",
    "bbe_prepare",
    "bbe_launch_prepared",
    "bbe_prepared_kernel_ms",
    "bbe_release_prepared",
)


class BackendUnavailable(RuntimeError):
    """The CUDA library is not built or no GPU is visible (there is deliberately no CPU fallback)."""


class DrawStreamError(RuntimeError):
    """Inject mode: a sim consumed fewer or more recorded draws than it was given."""

    def __init__(self, sim_index: int, message: str):
        super().__init__(message)
        self.sim_index = sim_index

    def __reduce__(self):  # picklable across process pools, like batch.BatchRunError
        return (type(self), (self.sim_index, self.args[0] if self.args else ""))


class SimDivergedError(RaceDivergedError):
    """A dry run exceeded tick_limit; ``sim_index`` is the first failing sim (the reference raises
    RaceDivergedError from that sim's simulate_from, race.py:402-404)."""

    def __init__(self, sim_index: int, message: str):
        super().__init__(message)
        self.sim_index = sim_index

    def __reduce__(self):
        return (type(self), (self.sim_index, self.args[0] if self.args else ""))


# -- ctypes mirrors of the header structs -------------------------------------------------------


class BbeRace(ctypes.Structure):
    _fields_ = [("track_length", ctypes.c_double), ("tick_limit", ctypes.c_int64), ("n", ctypes.c_int32),
                ("_pad", ctypes.c_int32)]


class BbeCompetitor(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("_pad", ctypes.c_int32), ("lo", ctypes.c_double),
                ("hi", ctypes.c_double), ("mu", ctypes.c_double), ("sigma", ctypes.c_double),
                ("scale", ctypes.c_double), ("pref_factor", ctypes.c_double), ("theta", ctypes.c_double),
                ("early_mult", ctypes.c_double), ("late_mult", ctypes.c_double), ("bp_abs", ctypes.c_double)]


_P = ctypes.POINTER


# Pointer members are declared c_void_p (ABI-identical to the header's typed pointers) and set from
# integer addresses: ndarray.ctypes.data is about half the cost of ctypes.data_as per call.
_VP = ctypes.c_void_p


class BbeState(ctypes.Structure):
    _fields_ = [("tick", ctypes.c_int64), ("positions", _VP), ("prev_steps", _VP),
                ("finish_ticks", _VP), ("from_start", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class BbeRequest(ctypes.Structure):
    _fields_ = [("n_sims", ctypes.c_int64), ("sim_offset", ctypes.c_int64), ("seed", ctypes.c_uint64),
                ("mode", ctypes.c_int32), ("lanes_per_slot_hint", ctypes.c_int32),
                ("draws", _VP), ("draw_offsets", _VP), ("seeds", _VP), ("seed_master", ctypes.c_uint64),
                ("group_size", ctypes.c_int64)]


class BbeResult(ctypes.Structure):
    _fields_ = [("wins", _VP), ("ranks", _VP), ("perms", _VP), ("winner", _VP), ("order", _VP),
                ("finish_ticks", _VP), ("final_positions", _VP), ("blocked", _VP), ("draws_used", _VP),
                ("competitor_steps", ctypes.c_uint64), ("blocked_steps", ctypes.c_uint64),
                ("first_diverged", ctypes.c_int64), ("first_bad_draws", ctypes.c_int64),
                ("kernel_ms", ctypes.c_float), ("lanes_per_slot", ctypes.c_int32),
                ("traj_positions", _VP), ("traj_prev_steps", _VP),
                ("traj_cap", ctypes.c_int32), ("_pad", ctypes.c_int32), ("group_wins", _VP)]


_lib = None


def lib():
    """Load the sm_100a library (built in-tree by ``__graft_entry__.build()`` / ``make``)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BackendUnavailable(f"{LIB_PATH} is not built; run `make` or __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.bbe_simulate.argtypes = [_P(BbeRace), _P(BbeCompetitor), _P(BbeState), _P(BbeRequest), _P(BbeResult)]
        L.bbe_simulate.restype = ctypes.c_int
        L.bbe_simulate_begin.argtypes = L.bbe_simulate.argtypes
        L.bbe_simulate_begin.restype = ctypes.c_int
        L.bbe_simulate_multi.argtypes = [ctypes.c_int32] + L.bbe_simulate.argtypes
        L.bbe_simulate_multi.restype = ctypes.c_int
        L.bbe_simulate_end.argtypes = [_P(BbeResult)]
        L.bbe_simulate_end.restype = ctypes.c_int
        L.bbe_simulate_async.argtypes = [_P(BbeRace), _P(BbeCompetitor), _P(BbeState), _P(BbeRequest),
                                         _P(BbeResult), ctypes.c_void_p, ctypes.c_void_p]
        L.bbe_simulate_async.restype = ctypes.c_int
        L.bbe_tally_len.argtypes = [ctypes.c_int32]
        L.bbe_tally_len.restype = ctypes.c_int64
        L.bbe_tally_offset.argtypes = [ctypes.c_int32, ctypes.c_int32]
        L.bbe_tally_offset.restype = ctypes.c_int64
        L.bbe_derive_seeds.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, _P(ctypes.c_uint64)]
        L.bbe_derive_seeds.restype = ctypes.c_int
        L.bbe_last_kernel_ms.restype = ctypes.c_float
        L.bbe_mt_getrandbits64.argtypes = [_P(ctypes.c_uint32), ctypes.c_int64, _P(ctypes.c_uint64)]
        L.bbe_mt_getrandbits64.restype = ctypes.c_int
        L.bbe_mt_exp_exact.restype = ctypes.c_int
        L.bbe_mt_advance64_many.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
        L.bbe_mt_advance64_many.restype = ctypes.c_int
        L.bbe_mt_advance64.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_int64]
        L.bbe_mt_advance64.restype = ctypes.c_int
        L.bbe_rp_predict.argtypes = [_P(BbeRace), _P(BbeCompetitor), _P(BbeState), ctypes.c_int64, ctypes.c_int32,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.bbe_rp_predict.restype = ctypes.c_int
        L.bbe_prepare.argtypes = [_P(BbeRace), _P(BbeCompetitor), _P(BbeState), ctypes.c_int32, ctypes.c_int32,
                                  _P(ctypes.c_void_p)]
        L.bbe_prepare.restype = ctypes.c_int
        L.bbe_launch_prepared.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                          ctypes.c_void_p, ctypes.c_void_p]
        L.bbe_launch_prepared.restype = ctypes.c_int
        L.bbe_prepared_kernel_ms.argtypes = [ctypes.c_void_p]
        L.bbe_prepared_kernel_ms.restype = ctypes.c_float
        L.bbe_release_prepared.argtypes = [ctypes.c_void_p]
        L.bbe_release_prepared.restype = None
        L.bbe_param_bytes.argtypes = [ctypes.c_int32]
        L.bbe_param_bytes.restype = ctypes.c_int64
        L.bbe_last_error.restype = ctypes.c_char_p
        L.bbe_version.restype = ctypes.c_int
        L.bbe_device_count.restype = ctypes.c_int
        L.bbe_device_info.argtypes = [ctypes.c_int, ctypes.c_char_p, _P(ctypes.c_int32), _P(ctypes.c_int32)]
        L.bbe_device_info.restype = ctypes.c_int
        # The entry points that write a CPython random.Random in place (bbe_rp_predict,
        # bbe_mt_advance64, bbe_mt_advance64_many) go through a PyDLL handle: they run with the GIL
        # held, so no other thread can use the generator mid-write (bbe_rp_predict drops the GIL in C
        # for its GPU wait once all its writes are done).
        G = ctypes.PyDLL(LIB_PATH)
        for name in ("bbe_rp_predict", "bbe_mt_advance64", "bbe_mt_advance64_many"):
            f = getattr(G, name)
            f.argtypes, f.restype = getattr(L, name).argtypes, getattr(L, name).restype
            setattr(L, name, f)
        if L.bbe_version() != ABI_VERSION:
            raise BackendUnavailable(f"{LIB_PATH} has ABI {L.bbe_version()}, expected {ABI_VERSION}: rebuild (make)")
        _lib = L
    return _lib


_EXP_EXACT: bool | None = None


def mt_exp_exact() -> bool:
    """Whether MT mode reproduces the host libm's exp() bit for bit (bbe_mt_exp_exact): the library
    found glibc's exp table in the loaded libm and verified it.  When False, lognormal steps in MT
    mode may differ from the reference's in the last bit."""
    global _EXP_EXACT
    if _EXP_EXACT is None:
        _EXP_EXACT = bool(lib().bbe_mt_exp_exact())
    return _EXP_EXACT


def check_mt_exact(config) -> None:
    """Warn (once per config object) when an MT-mode call on a field with a lognormal runner cannot
    be bit-exact because the libm exp table was not found."""
    if mt_exp_exact() or not any(not hasattr(c.steps, "lo") for c in config.competitors):
        return
    if id(config) in _warned:
        return
    _warned.add(id(config))
    import warnings

    warnings.warn("mode='mt': glibc's exp table was not found in this process's libm, so lognormal steps "
                  "use CUDA's exp and may differ from the reference in the last bit (bbe_mt_exp_exact() == 0)",
                  RuntimeWarning, stacklevel=3)


_warned: set = set()


def last_error() -> str:
    return lib().bbe_last_error().decode(errors="replace")


def device_count() -> int:
    return int(lib().bbe_device_count())


# -- packing ------------------------------------------------------------------------------------


@dataclass
class Packed:
    race: BbeRace
    comps: ctypes.Array
    n: int
    ids: tuple


_last_packed: tuple = (None, None)  # (config object, Packed): bettors re-predict on one frozen config


def pack_config(config) -> Packed:
    """RaceConfig -> (bbe_race, bbe_competitor[n]).  Validates like RaceConfig.validate.

    Race configs are frozen dataclasses, so the last packed config is reused when the same object
    comes back (every bettor of a session predicts on the session's one config)."""
    global _last_packed
    cached = _last_packed  # one read: another thread may replace the cache meanwhile
    if cached[0] is config:
        return cached[1]
    pk = _pack_config(config)
    _last_packed = (config, pk)
    return pk


def _pack_config(config) -> Packed:
    validate_config(config)
    n = len(config.competitors)
    if n > MAX_COMPETITORS:
        raise RaceConfigError(f"at most {MAX_COMPETITORS} competitors are supported, got {n}")
    L = float(config.track_length)
    race = BbeRace(L, int(config.tick_limit), n, 0)
    comps = (BbeCompetitor * n)()
    for k, c in enumerate(config.competitors):
        o = comps[k]
        s = c.steps
        if hasattr(s, "lo"):
            o.family, o.lo, o.hi = 0, float(s.lo), float(s.hi)
            o.scale = 1.0
        else:
            o.family, o.mu, o.sigma, o.scale = 1, float(s.mu), float(s.sigma), float(s.scale)
        o.pref_factor = preference_factor(config.conditions, c.preference, c.pref_sensitivity)
        o.theta = float(c.theta)
        r = c.responsiveness
        o.early_mult, o.late_mult = float(r.early_mult), float(r.late_mult)
        o.bp_abs = r.breakpoint * L  # race.py:94 evaluates breakpoint * track_length in double
    return Packed(race, comps, n, tuple(c.cid for c in config.competitors))


def _ptr(a, ct=None):
    """Address of an ndarray's data for a c_void_p member (None stays NULL)."""
    return None if a is None else a.ctypes.data


_last_state = (None, None, None)  # (key, BbeState, arrays): a session predicts many times per state


def pack_state(state, n: int):
    global _last_state
    if state is None:
        return BbeState(0, None, None, None, 1, 0), ()
    if len(state.positions) != n or len(state.prev_steps) != n or len(state.finish_ticks) != n:
        raise RaceConfigError("state vectors must have one entry per competitor")
    key = (state.tick, tuple(state.positions), tuple(state.prev_steps), tuple(state.finish_ticks))
    cached = _last_state
    if cached[0] == key:
        return cached[1], cached[2]
    pos = np.ascontiguousarray(state.positions, np.float64)
    prev = np.ascontiguousarray(state.prev_steps, np.float64)
    fin = np.array([-1 if t is None else int(t) for t in state.finish_ticks], np.int64)
    st = BbeState(int(state.tick), pos.ctypes.data, prev.ctypes.data, fin.ctypes.data, 0, 0)
    _last_state = (key, st, (pos, prev, fin))
    return st, (pos, prev, fin)  # keep arrays alive


# -- results ------------------------------------------------------------------------------------


@dataclass
class SimResult:
    """Tallies (always) and optional per-sim records of one batched call."""

    ids: tuple
    n_sims: int
    wins: np.ndarray
    ranks: np.ndarray | None
    perms: np.ndarray | None
    winner: np.ndarray | None
    order: np.ndarray | None
    finish_ticks: np.ndarray | None
    final_positions: np.ndarray | None
    blocked: np.ndarray | None
    draws_used: np.ndarray | None
    competitor_steps: int
    blocked_steps: int
    kernel_ms: float
    lanes_per_slot: int
    traj_positions: np.ndarray | None = None
    traj_prev_steps: np.ndarray | None = None
    group_wins: np.ndarray | None = None  # [groups, n] winner counts per group_size consecutive sims

    def win_probabilities(self, laplace: bool = True) -> tuple[float, ...]:
        """(w + 1) / (d + n) as agents.py:166, or plain frequencies."""
        n, d = len(self.ids), self.n_sims
        if laplace:
            return tuple((int(w) + 1) / (d + n) for w in self.wins)
        return tuple(int(w) / d for w in self.wins)


def _raise(rc: int, res: BbeResult):
    msg = last_error()
    if rc == BBE_EINVAL:
        raise RaceConfigError(msg)
    if rc == BBE_EDIVERGED:
        raise SimDivergedError(int(res.first_diverged), msg)
    if rc == BBE_EDRAWS:
        raise DrawStreamError(int(res.first_bad_draws), msg)
    if rc == BBE_ENODEV:
        raise BackendUnavailable(msg)
    raise RuntimeError(f"bbe_simulate failed ({rc}): {msg}")


def simulate_batch(
    state,
    config,
    n_sims: int,
    seed: int = 0,
    *,
    mode: str = "native",
    draws=None,
    draw_offsets=None,
    seeds=None,
    seed_master: int = 0,
    sim_offset: int = 0,
    ranks: bool = True,
    perms: bool = False,
    records: bool = False,
    winners: bool = False,
    trajectory_ticks: int = 0,
    lanes_per_slot: int = 0,
    parts: int | None = None,
    group_size: int = 0,
    _defer: bool = False,
) -> SimResult:
    """Run ``n_sims`` independent continuations of ``state`` (or races from the start line when
    ``state is None``) and return tallies.

    mode="native": Philox stream keyed by ``seed``; sim i uses counter (tick block, competitor,
    sim_offset + i), so any sharding of the index range reproduces the same per-sim outcomes.
    mode="mt": sim i replays random.Random(seeds[i]) (or derive_seed(seed_master, "run",
    sim_offset + i) when ``seeds`` is None) -- the reference's own result.
    mode="inject": replay recorded reference draws (``draws`` / CSR ``draw_offsets``) -- bit-exact.
    records=True also returns per-sim winner, order, finish ticks, final positions, blocked counts;
    winners=True only the per-sim winner; trajectory_ticks=T (exact modes) positions and previous
    steps after each of the first T ticks of every sim.
    group_size=g also counts winners per group of g consecutive sims (``group_wins``, [groups, n]):
    one bettor's dry runs in a batched dispatch.
    parts=P splits the sims over the visible GPUs (``bbe_simulate_multi``: P contiguous shards, part p
    on device p % device_count, 0 = one per device) -- run_batch(workers=...) -- with identical results.
    """
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    pk = pack_config(config)
    if mode == "mt":
        check_mt_exact(config)
    n = pk.n
    st, keep = pack_state(state, n)
    n_sims = int(n_sims)
    req = BbeRequest(n_sims, int(sim_offset), int(seed) & M64, MODES[mode], int(lanes_per_slot), None, None, None,
                     int(seed_master) & M64, int(group_size))
    if mode == "inject":
        draws = np.ascontiguousarray(draws, np.float64)
        draw_offsets = np.ascontiguousarray(draw_offsets, np.int64)
        if len(draw_offsets) != n_sims + 1:
            raise ValueError("draw_offsets needs n_sims + 1 entries")
        if draw_offsets[-1] > len(draws):
            raise ValueError("draw_offsets point past the end of draws")
        req.draws = _ptr(draws, ctypes.c_double)
        req.draw_offsets = _ptr(draw_offsets, ctypes.c_int64)
    if seeds is not None:
        seeds = np.ascontiguousarray(seeds, np.uint64)
        if len(seeds) != n_sims:
            raise ValueError("seeds needs one entry per sim")
        req.seeds = _ptr(seeds, ctypes.c_uint64)
    wins = np.zeros(n, np.uint64)
    rk = np.zeros((n, n), np.uint64) if ranks else None
    pm = np.zeros(math.factorial(n), np.uint64) if (perms and n <= MAX_PERM_COMPETITORS) else None
    winner = order = fin = fpos = blk = used = tpos = tprev = None
    if records or winners:
        winner = np.zeros(n_sims, np.int32)
    if records:
        order = np.zeros((n_sims, n), np.int32)
        fin = np.zeros((n_sims, n), np.int64)
        fpos = np.zeros((n_sims, n), np.float64)
        blk = np.zeros(n_sims, np.int64)
        used = np.zeros(n_sims, np.int64) if mode == "inject" else None
    gw = None
    if group_size > 0:
        gw = np.zeros(((n_sims + int(group_size) - 1) // int(group_size), n), np.uint64)
    cap = int(trajectory_ticks)
    if cap > 0:
        tpos = np.zeros((n_sims, cap + 1, n), np.float64)
        tprev = np.zeros((n_sims, cap + 1, n), np.float64)
    res = BbeResult(_ptr(wins, ctypes.c_uint64), _ptr(rk, ctypes.c_uint64), _ptr(pm, ctypes.c_uint64),
                    _ptr(winner, ctypes.c_int32), _ptr(order, ctypes.c_int32), _ptr(fin, ctypes.c_int64),
                    _ptr(fpos, ctypes.c_double), _ptr(blk, ctypes.c_int64), _ptr(used, ctypes.c_int64),
                    0, 0, -1, -1, 0.0, 0, _ptr(tpos, ctypes.c_double), _ptr(tprev, ctypes.c_double), cap, 0,
                    _ptr(gw))
    build = (lambda r: SimResult(pk.ids, n_sims, wins, rk, pm, winner, order, fin, fpos, blk, used,
                                 int(r.competitor_steps), int(r.blocked_steps), float(r.kernel_ms),
                                 int(r.lanes_per_slot), tpos, tprev, gw))
    if parts is not None:
        if _defer:
            raise ValueError("parts= runs synchronously (one host thread per device)")
        rc = lib().bbe_simulate_multi(int(parts), ctypes.byref(pk.race), pk.comps, ctypes.byref(st),
                                      ctypes.byref(req), ctypes.byref(res))
        if rc != BBE_OK:
            _raise(rc, res)
        return build(res)
    rc = lib().bbe_simulate_begin(ctypes.byref(pk.race), pk.comps, ctypes.byref(st), ctypes.byref(req),
                                  ctypes.byref(res))
    if rc != BBE_OK:
        _raise(rc, res)
    pending = PendingSim(res, (pk, st, keep, req, draws, draw_offsets, seeds), build)
    return pending if _defer else pending.end()


class PendingSim:
    """A batch enqueued on the GPU (``bbe_simulate_begin``); ``end()`` waits and returns the result.
    Host work done before ``end()`` overlaps the kernel."""

    def __init__(self, res, keep, build):
        self._res, self._keep, self._build = res, keep, build
        self._done = None

    def end(self) -> SimResult:
        if self._done is None:
            rc = lib().bbe_simulate_end(ctypes.byref(self._res))
            self._keep = None
            if rc != BBE_OK:
                _raise(rc, self._res)
            self._done = self._build(self._res)
        return self._done


class _PredictBufs(threading.local):
    """Per-thread output buffers of bbe_rp_predict (reused: one call at a time per thread)."""

    def __init__(self):
        self.wins = np.zeros(MAX_COMPETITORS, np.uint64)
        self.first = np.zeros(1, np.int64)


_pbufs = _PredictBufs()


def rp_predict_counts(state, config, d: int, state624_addr: int, pos_addr: int, *, mode: str = "mt") -> list:
    """``bbe_rp_predict``: winner counts of d dry runs whose seeds are d getrandbits(64) of the MT19937
    state at ``state624_addr`` (624 uint32) / ``pos_addr`` (int32), advanced in place (a CPython
    random.Random's own fields, agents.py); returns the counts as a list of ints."""
    pk = pack_config(config)
    if mode == "mt":
        check_mt_exact(config)
    st, keep = pack_state(state, pk.n)
    b = _pbufs
    rc = lib().bbe_rp_predict(ctypes.byref(pk.race), pk.comps, ctypes.byref(st), int(d), MODES[mode], state624_addr,
                              pos_addr, b.wins.ctypes.data, b.first.ctypes.data)
    if rc != BBE_OK:
        if rc == BBE_EDIVERGED:
            raise SimDivergedError(int(b.first[0]), last_error())
        if rc == BBE_EINVAL:
            raise RaceConfigError(last_error())
        if rc == BBE_ENODEV:
            raise BackendUnavailable(last_error())
        raise RuntimeError(f"bbe_rp_predict failed ({rc}): {last_error()}")
    return b.wins[:pk.n].tolist()


def simulate_batch_begin(*args, **kwargs) -> PendingSim:
    """``simulate_batch`` that returns as soon as the work is enqueued (see PendingSim)."""
    return simulate_batch(*args, _defer=True, **kwargs)


# -- reference-shaped single-race entry points ---------------------------------------------------


def simulate_from(state, config, seed: int, *, mode: str = "mt") -> tuple[str, ...]:
    """One continuation (race.py:393-406) on the GPU; returns the finish order as ids.

    mode="mt" (default): the reference's MT19937 stream from ``seed`` -- the reference's own result."""
    r = simulate_batch(state, config, 1, seed, mode=mode, records=True, ranks=False,
                       seeds=np.array([seed & M64], np.uint64) if mode == "mt" else None)
    return tuple(r.ids[c] for c in r.order[0])


def run_race(config, seed: int, record: bool = True, *, mode: str = "mt", with_prev_steps: bool = False):
    """One race from the start line (race.py:373-390) on the GPU.

    record=True returns the per-tick position snapshots (``Trajectory.ticks``) recorded by the exact
    kernel (mode "mt" or "inject"); with_prev_steps=True also returns the per-tick previous steps as
    a second value (the state an in-play bettor reconstructs, agents.py:348-358).
    """
    seeds = np.array([seed & M64], np.uint64) if mode == "mt" else None
    cap = 0
    if record:
        if mode == "native":
            raise ValueError("record=True needs an exact mode (mt)")
        cap = int(min(config.tick_limit, 4096))
    while True:
        r = simulate_batch(None, config, 1, seed, mode=mode, records=True, ranks=False, seeds=seeds,
                           trajectory_ticks=cap)
        n_ticks = int(r.finish_ticks[0].max())
        if not record or n_ticks <= cap:
            break
        cap = n_ticks  # the race outlived the first guess: record again with room for every tick
    ticks = prevs = None
    if record:
        ticks = tuple(tuple(float(p) for p in row) for row in r.traj_positions[0, : n_ticks + 1])
        prevs = r.traj_prev_steps[0, : n_ticks + 1].copy()
    traj = Trajectory(
        competitor_ids=r.ids,
        dt=config.dt,
        ticks=ticks,
        finish_ticks=tuple(int(t) for t in r.finish_ticks[0]),
        finish_order=tuple(r.ids[c] for c in r.order[0]),
        final_positions=tuple(float(p) for p in r.final_positions[0]),
        blocked_steps=int(r.blocked[0]),
    )
    return (traj, prevs) if with_prev_steps else traj


# -- device-resident path (bench `value`, multi-GPU shards) --------------------------------------


class DeviceLauncher:
    """Pre-packed race for repeated device-resident launches.

    Tallies are added into a caller-owned device buffer (e.g. a torch int64 CUDA tensor, passed by
    ``data_ptr()``) on a caller stream (``torch.cuda.current_stream().cuda_stream``).  NATIVE and
    NATIVE64 launches use a prepared race (``bbe_prepare``: parameters uploaded once, nothing copied
    per launch; ``native_mode`` picks which); MT launches go through ``bbe_simulate_async``.
    """

    def __init__(self, state, config, *, lanes_per_slot: int = 0, native_mode: str = "native"):
        if native_mode not in ("native", "native64"):
            raise ValueError("native_mode: 'native' (FP32 state) or 'native64' (FP64 state)")
        self.native_mode = native_mode
        self.pk = pack_config(config)
        self.st, self._keep = pack_state(state, self.pk.n)
        self.lanes_per_slot = int(lanes_per_slot)
        self.tally_len = int(lib().bbe_tally_len(self.pk.n))
        off = lambda f: int(lib().bbe_tally_offset(self.pk.n, f))  # noqa: E731
        self.off = {name: off(i) for i, name in enumerate(
            ["wins", "ranks", "perms", "ct", "blocked", "n_div", "n_bad", "first_div", "first_bad"])}
        self._prep = None
        self._last_prepared = False

    def _prepared(self):
        if self._prep is None:
            h = ctypes.c_void_p()
            rc = lib().bbe_prepare(ctypes.byref(self.pk.race), self.pk.comps, ctypes.byref(self.st),
                                   MODES[self.native_mode], self.lanes_per_slot, ctypes.byref(h))
            if rc != BBE_OK:
                _raise(rc, BbeResult())
            self._prep = h
        return self._prep

    def __del__(self):
        if getattr(self, "_prep", None) is not None and _lib is not None:
            _lib.bbe_release_prepared(self._prep)
            self._prep = None

    def launch(self, d_tally_ptr: int, n_sims: int, seed: int, *, sim_offset: int = 0, stream: int = 0,
               mode: str = "native") -> None:
        if mode in ("native", "native64"):
            if mode != self.native_mode:
                raise ValueError(f"this launcher was prepared for {self.native_mode!r}")
            rc = lib().bbe_launch_prepared(self._prepared(), int(n_sims), int(sim_offset), int(seed) & M64,
                                           d_tally_ptr, stream)
            if rc != BBE_OK:
                _raise(rc, BbeResult())
            self._last_prepared = True
            return
        # mode "mt": sim i replays random.Random(derive_seed(seed, "run", sim_offset + i)), derived on the GPU
        req = BbeRequest(int(n_sims), int(sim_offset), int(seed) & M64, MODES[mode], self.lanes_per_slot, None,
                         None, None, int(seed) & M64)
        rc = lib().bbe_simulate_async(ctypes.byref(self.pk.race), self.pk.comps, ctypes.byref(self.st),
                                      ctypes.byref(req), None, ctypes.c_void_p(d_tally_ptr),
                                      ctypes.c_void_p(stream))
        if rc != BBE_OK:
            _raise(rc, BbeResult())
        self._last_prepared = False

    def last_kernel_ms(self) -> float:
        """Device time of this launcher's last launch (waits for it)."""
        if self._last_prepared:
            return float(lib().bbe_prepared_kernel_ms(self._prep))
        return float(lib().bbe_last_kernel_ms())

