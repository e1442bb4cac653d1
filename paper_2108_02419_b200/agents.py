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

from .sim import _P, lib, simulate_batch

M64 = (1 << 64) - 1


def dry_run_seeds(rng, d: int, *, want: bool = True) -> np.ndarray | None:
    """Advance ``rng`` by d ``getrandbits(64)`` calls (agents.py:164); return the d seeds if ``want``.

    A ``random.Random`` is advanced in C on its MT19937 state; any other generator object falls back
    to calling its own ``getrandbits`` (host bookkeeping only -- no simulation happens here).
    """
    if d <= 0:
        return np.zeros(0, np.uint64) if want else None
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


def rp_predict(state, config, d: int, rng, *, mode: str = "mt") -> tuple[float, ...]:
    """Laplace-smoothed win probabilities from d dry-run continuations, computed on the GPU.

    mode="mt" (default): every continuation replays the reference's own MT19937 stream from its
    dry-run seed, so the probabilities equal the reference's exactly (a true drop-in).
    mode="native": Philox stream keyed by the first dry-run seed -- statistically equal to the
    reference (binomial bounds, tests/test_gpu_native.py) and the fastest path.
    """
    n = len(config.competitors)
    if d <= 0:
        dry_run_seeds(rng, d, want=False)
        return tuple(1 / (d + n) for _ in range(n))
    if mode == "mt":
        res = simulate_batch(state, config, d, mode="mt", seeds=dry_run_seeds(rng, d), ranks=False)
    else:
        key = int(dry_run_seeds(rng, 1)[0])  # the first dry-run seed keys the Philox stream
        dry_run_seeds(rng, d - 1, want=False)  # the other d-1 draws only advance the stream
        res = simulate_batch(state, config, d, key, mode=mode, ranks=False)
    return tuple((int(w) + 1) / (d + n) for w in res.wins)
