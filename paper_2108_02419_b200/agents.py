"""GPU dry-run predictor: drop-in for ``racemarket.agents.rp_predict`` (agents.py:153-166).

The reference runs d sequential ``simulate_from`` calls, each seeded with ``rng.getrandbits(64)``,
tallies winners and returns Laplace-smoothed probabilities ``(w + 1) / (d + n)``.  Here the d
continuations are one batched launch.  The agent stream is advanced exactly as the reference does
(one ``getrandbits(64 * d)`` call yields the same 2d MT words, least-significant first, as d calls of
``getrandbits(64)``), so everything the agent draws afterwards (tie-break ``randrange``, RB stake
``randint``: agents.py:304-310, 406-408) is unchanged.
"""

from __future__ import annotations

import numpy as np

from .sim import simulate_batch

M64 = (1 << 64) - 1


def dry_run_seeds(rng, d: int) -> np.ndarray:
    """The d per-dry-run seeds the reference would draw (agents.py:164), advancing ``rng`` by 2d words."""
    if d <= 0:
        return np.zeros(0, np.uint64)
    bits = rng.getrandbits(64 * d)
    return np.frombuffer(bits.to_bytes(8 * d, "little"), dtype="<u8").astype(np.uint64)


def rp_predict(state, config, d: int, rng, *, mode: str = "native") -> tuple[float, ...]:
    """Laplace-smoothed win probabilities from d dry-run continuations, computed on the GPU.

    mode="native": the d continuations use the Philox stream keyed by the first dry-run seed.
    """
    n = len(config.competitors)
    if d <= 0:
        return tuple(1 / (d + n) for _ in range(n))
    seeds = dry_run_seeds(rng, d)
    if mode == "mt":
        res = simulate_batch(state, config, d, mode="mt", seeds=seeds, ranks=False)
    else:
        res = simulate_batch(state, config, d, int(seeds[0]), mode=mode, ranks=False)
    return tuple((int(w) + 1) / (d + n) for w in res.wins)
