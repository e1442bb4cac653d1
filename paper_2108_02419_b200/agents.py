"""GPU dry-run predictor: drop-in for ``racemarket.agents.rp_predict`` (agents.py:153-166).

The reference runs d sequential ``simulate_from`` calls, each seeded with ``rng.getrandbits(64)``,
tallies winners and returns Laplace-smoothed probabilities ``(w + 1) / (d + n)``.  Here the d
continuations are one batched launch.  The bettor's stream is advanced exactly as the reference
advances it -- d ``getrandbits(64)`` calls, 2d MT19937 words -- by ``bbe_mt_getrandbits64`` on the
generator's own state (``getstate``/``setstate``), so everything the bettor draws afterwards
(tie-break ``randrange``, RB stake ``randint``: agents.py:304-310, 406-408) is unchanged.
"""

from __future__ import annotations

import ctypes
import random

import numpy as np

from .race import RaceState
from .sim import _P, lib, rp_predict_counts, simulate_batch, simulate_batch_begin

M64 = (1 << 64) - 1


_INPLACE_OK: bool | None = None
_MT_SPLIT_MIN = 16384  # rp_predict(mode="mt") splits d >= 2x this into two overlapped launches
_IDX_OFF, _STATE_OFF = 16, 20  # CPython RandomObject: PyObject_HEAD (16 B), int index, uint32_t state[624]


def _inplace_ok() -> bool:
    """Whether this interpreter lays out random.Random as CPython's _randommodule.c RandomObject
    (checked once against getstate(); the in-place path is used only if it matches exactly)."""
    global _INPLACE_OK
    if _INPLACE_OK is None:
        try:
            r = random.Random(12345)
            r.random()
            st = r.getstate()[1]
            base = id(r)
            idx = ctypes.c_int.from_address(base + _IDX_OFF).value
            words = list((ctypes.c_uint32 * 624).from_address(base + _STATE_OFF))
            _INPLACE_OK = idx == st[624] and words == list(st[:624])
        except Exception:  # pragma: no cover - non-CPython
            _INPLACE_OK = False
    return _INPLACE_OK


def _advance(rng, d: int, out: np.ndarray | None, out_len: int) -> bool:
    """Advance a random.Random by d getrandbits(64) in place in C; False if not possible here."""
    if type(rng) is not random.Random or not _inplace_ok():
        return False
    base = id(rng)
    rc = lib().bbe_mt_advance64(base + _STATE_OFF, base + _IDX_OFF, d, None if out is None else out.ctypes.data,
                                out_len)
    if rc != 0:
        raise RuntimeError("bbe_mt_advance64 failed")
    return True


def dry_run_seeds(rng, d: int, *, want: bool = True, first_only: bool = False) -> np.ndarray | None:
    """Advance ``rng`` by d ``getrandbits(64)`` calls (agents.py:164); return the d seeds if ``want``
    (only the first one if ``first_only``).

    A ``random.Random`` is advanced in C on its own MT19937 state -- in place when the interpreter's
    object layout is the verified CPython one, else through getstate()/setstate(); any other
    generator object falls back to its own ``getrandbits`` (host bookkeeping only).
    """
    if d <= 0:
        return np.zeros(0, np.uint64) if want else None
    if want:
        out = np.zeros(1 if first_only else d, np.uint64)
        if _advance(rng, d, out, len(out)):
            return out
    elif _advance(rng, d, None, 0):
        return None
    if type(rng) is random.Random:
        version, internal, gauss = rng.getstate()
        st = np.array(internal, dtype=np.uint32)
        out = np.zeros(d, np.uint64) if want else None
        rc = lib().bbe_mt_getrandbits64(st.ctypes.data_as(_P(ctypes.c_uint32)), d,
                                        None if out is None else out.ctypes.data_as(_P(ctypes.c_uint64)))
        if rc != 0:
            raise RuntimeError("bbe_mt_getrandbits64 failed")
        rng.setstate((version, tuple(st.tolist()), gauss))
        return out
    bits = rng.getrandbits(64 * d)
    return np.frombuffer(bits.to_bytes(8 * d, "little"), dtype="<u8").astype(np.uint64) if want else None


def dry_run_seeds_many(rngs, ds, out_lens) -> list:
    """dry_run_seeds for many bettors in one C call (threads over generators): advance rngs[i] by
    ds[i] getrandbits(64) and return its first out_lens[i] values (None where out_lens[i] == 0).

    Falls back to per-generator calls unless every generator is a plain random.Random with the
    verified in-place layout."""
    outs = [np.zeros(int(k), np.uint64) if k else None for k in out_lens]
    if not all(type(r) is random.Random for r in rngs) or not _inplace_ok():
        res = []
        for r, d, k in zip(rngs, ds, out_lens):
            if k:
                v = dry_run_seeds(r, d, first_only=(k == 1 and d > 1))
                res.append(v[:k])
            else:
                dry_run_seeds(r, d, want=False)
                res.append(None)
        return res
    m = len(rngs)
    if m == 0:
        return []
    base = np.array([id(r) for r in rngs], np.uint64)
    states = base + np.uint64(_STATE_OFF)
    pos = base + np.uint64(_IDX_OFF)
    counts = np.array([max(int(d), 0) for d in ds], np.int64)
    optr = np.array([o.ctypes.data if o is not None else 0 for o in outs], np.uint64)
    olen = np.array([int(k) for k in out_lens], np.int64)
    rc = lib().bbe_mt_advance64_many(m, states.ctypes.data, pos.ctypes.data, counts.ctypes.data,
                                     optr.ctypes.data, olen.ctypes.data, 0)
    if rc != 0:
        raise RuntimeError("bbe_mt_advance64_many failed")
    return outs


def _end_both(first, second):
    """Wait for two pending batches; both are always ended (their contexts released), and the first
    batch's error, if any, wins -- it holds the lower sim indices."""
    out, err = [], None
    for p in (first, second):
        try:
            out.append(p.end())
        except Exception as e:  # noqa: BLE001 -- re-raised below
            err = err or e
    if err is not None:
        raise err
    return out


def rp_predict(state, config, d: int, rng, *, mode: str = "mt") -> tuple[float, ...]:
    """Laplace-smoothed win probabilities from d dry-run continuations, computed on the GPU.

    mode="mt" (default): every continuation replays the reference's own MT19937 stream from its
    dry-run seed, so the probabilities equal the reference's exactly (a true drop-in).
    mode="native64": Philox stream keyed by the first dry-run seed with the reference's FP64 race
    arithmetic (only the word generator differs; tests/test_gpu_native64.py) -- statistically equal.
    mode="native": the same stream with FP32 race state -- the fastest path (binomial bounds,
    tests/test_gpu_native.py).
    """
    n = len(config.competitors)
    if d <= 0:
        dry_run_seeds(rng, d, want=False)
        return tuple(1 / (d + n) for _ in range(n))
    if type(rng) is random.Random and _inplace_ok():
        # one C call: the d seeds drawn from the bettor's own MT19937 fields (advanced in place), the
        # dry runs on the GPU (bbe_rp_predict; MT: two overlapped halves when d is large)
        base = id(rng)
        wins = rp_predict_counts(state, config, d, base + _STATE_OFF, base + _IDX_OFF, mode=mode)
        dn = d + n
        return tuple((w + 1) / dn for w in wins)
    if mode == "mt":
        if d < 2 * _MT_SPLIT_MIN:
            res = simulate_batch(state, config, d, mode="mt", seeds=dry_run_seeds(rng, d), ranks=False)
        else:
            # two halves, each enqueued as soon as its seeds exist: the host draws the second half's
            # seeds while the GPU seeds and races the first, and the second launch (its own stream)
            # fills the first one's tail.  Same seeds, same sims: the summed tallies are unchanged.
            h = d // 2
            first = simulate_batch_begin(state, config, h, mode="mt", seeds=dry_run_seeds(rng, h), ranks=False)
            second = simulate_batch_begin(state, config, d - h, mode="mt", seeds=dry_run_seeds(rng, d - h),
                                          sim_offset=h, ranks=False)
            r0, r1 = _end_both(first, second)
            return tuple((int(a) + int(b) + 1) / (d + n) for a, b in zip(r0.wins, r1.wins))
    else:
        # the first dry-run seed keys the Philox stream; the other d-1 draws only advance the
        # bettor's stream, which the host does while the kernel runs
        key = int(dry_run_seeds(rng, 1)[0])
        pending = simulate_batch_begin(state, config, d, key, mode=mode, ranks=False)
        dry_run_seeds(rng, d - 1, want=False)
        res = pending.end()
    return tuple((int(w) + 1) / (d + n) for w in res.wins)


# -- the RP / RB bettors' prediction step (agents.py:345-362, 399-404) ----------------------------


def reconstruct_state(obs) -> RaceState:
    """RPBettor._reconstruct_state (agents.py:348-358): the bettor's view of the race from an
    observation -- previous steps are the last entry of each step history (0.0 before the race)."""
    prev = [h[-1] if h else 0.0 for h in obs.step_history]
    return RaceState(obs.race_tick, list(obs.positions), prev, list(obs.finish_ticks))


def rb_weight(p: float, gamma: float) -> float:
    """Inverse-S probability weighting p^g / (p^g + (1-p)^g)^(1/g) (agents.py:234-245)."""
    if not 0.0 <= p <= 1.0:
        raise ValueError(f"probability must be in [0, 1], got {p}")
    if p in (0.0, 1.0) or gamma == 1.0:
        return p
    num = p**gamma
    return num / (num + (1.0 - p) ** gamma) ** (1.0 / gamma)


def rb_weighted(probs, gamma: float) -> tuple[float, ...]:
    """Elementwise rb_weight, renormalised to sum to 1 (agents.py:248-252)."""
    w = [rb_weight(p, gamma) for p in probs]
    total = sum(w)
    return tuple(x / total for x in w)


def rp_bettor_predict(obs, config, d: int, rng, *, mode: str = "mt") -> tuple[float, ...]:
    """RPBettor.predict (agents.py:360-362) with the dry runs on the GPU."""
    return rp_predict(reconstruct_state(obs), config, d, rng, mode=mode)


def rb_bettor_predict(obs, config, d: int, gamma: float, rng, *, mode: str = "mt") -> tuple[float, ...]:
    """RBBettor.predict (agents.py:402-404): the RP estimate through the inverse-S weighting."""
    return rb_weighted(rp_bettor_predict(obs, config, d, rng, mode=mode), gamma)
