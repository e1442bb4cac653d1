"""Race model types and the GPU-backed race entry points (drop-in for ``racemarket.race``).

The records here carry the same names, fields, defaults and validation errors as the reference
(``/root/reference/pkg/src/racemarket/race.py``) so configurations, states and call sites move over
unchanged; objects from the reference package are also accepted anywhere (duck-typed by field).

What differs is where the work runs: ``simulate_from`` / ``run_race`` / ``simulate_batch`` launch the
sm_100a kernels in ``csrc/`` through the C-ABI (``include/bbe_sim.h``).  There is no CPU
fallback: without the built library every entry point raises ``BackendUnavailable``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

DEFAULT_TICK_LIMIT = 1_000_000  # race.py:21
MIN_PREFERENCE_FACTOR = 0.01  # race.py:24


# When the reference package is installed, the errors here also subclass its own, so reference code
# (and callers) catching ``racemarket.race.RaceConfigError`` / ``RaceDivergedError`` catch ours too.
try:  # pragma: no cover - depends on the environment
    from racemarket.race import RaceConfigError as _RefConfigError
    from racemarket.race import RaceDivergedError as _RefDivergedError
except ImportError:
    _RefConfigError, _RefDivergedError = ValueError, RuntimeError


class RaceConfigError(_RefConfigError):
    """Invalid race configuration (race.py:27-28); a ValueError, and racemarket's when installed."""


class RaceDivergedError(_RefDivergedError):
    """A simulated race exceeded its tick limit (race.py:31-32); a RuntimeError, and racemarket's when
    installed."""


@dataclass(frozen=True)
class UniformSteps:
    """Step law U[lo, hi] drawn as ``lo + (hi - lo) * u`` (race.py:35-51)."""

    lo: float
    hi: float

    def validate(self) -> None:
        if not (0.0 < self.lo <= self.hi):
            raise RaceConfigError(f"uniform steps need 0 < lo <= hi, got ({self.lo}, {self.hi})")

    @property
    def mean(self) -> float:
        return 0.5 * (self.lo + self.hi)


@dataclass(frozen=True)
class LogNormalSteps:
    """Step law ``scale * exp(N(mu, sigma))`` (race.py:54-73)."""

    mu: float
    sigma: float
    scale: float = 1.0

    def validate(self) -> None:
        if self.sigma < 0.0:
            raise RaceConfigError(f"lognormal sigma must be >= 0, got {self.sigma}")
        if self.scale <= 0.0:
            raise RaceConfigError(f"lognormal scale must be > 0, got {self.scale}")

    @property
    def mean(self) -> float:
        import math

        return self.scale * math.exp(self.mu + 0.5 * self.sigma * self.sigma)


@dataclass(frozen=True)
class Responsiveness:
    """``early_mult`` while position < breakpoint * L, else ``late_mult`` (race.py:79-96)."""

    early_mult: float = 1.0
    late_mult: float = 1.0
    breakpoint: float = 0.5

    def validate(self) -> None:
        if self.early_mult <= 0.0 or self.late_mult <= 0.0:
            raise RaceConfigError("responsiveness multipliers must be > 0")
        if not (0.0 <= self.breakpoint <= 1.0):
            raise RaceConfigError(f"breakpoint must be in [0, 1], got {self.breakpoint}")

    def at(self, position: float, track_length: float) -> float:
        return self.early_mult if position < self.breakpoint * track_length else self.late_mult


@dataclass(frozen=True)
class Competitor:
    """One runner (race.py:99-116)."""

    cid: str
    steps: UniformSteps | LogNormalSteps
    preference: float = 0.5
    pref_sensitivity: float = 0.0
    theta: float = 0.0
    responsiveness: Responsiveness = field(default_factory=Responsiveness)

    def validate(self) -> None:
        if not self.cid:
            raise RaceConfigError("competitor id must be non-empty")
        self.steps.validate()
        if self.pref_sensitivity < 0.0:
            raise RaceConfigError(f"pref_sensitivity must be >= 0, got {self.pref_sensitivity}")
        if self.theta < 0.0:
            raise RaceConfigError(f"theta must be >= 0, got {self.theta}")
        self.responsiveness.validate()


@dataclass(frozen=True)
class BettingClose:
    """When in-play betting closes (race.py:119-155).  Not used by the simulation itself."""

    rule: str
    k: int | None = None

    @staticmethod
    def first() -> "BettingClose":
        return BettingClose("first")

    @staticmethod
    def kth(k: int) -> "BettingClose":
        return BettingClose("kth", k)

    @staticmethod
    def last() -> "BettingClose":
        return BettingClose("last")

    def close_rank(self, n_competitors: int) -> int:
        return {"first": 1, "kth": self.k}.get(self.rule, n_competitors)  # type: ignore[return-value]

    def validate(self, n_competitors: int) -> None:
        if self.rule not in ("first", "kth", "last"):
            raise RaceConfigError(f"unknown betting_close rule: {self.rule!r}")
        if self.rule == "kth":
            if self.k is None or not (1 <= self.k <= n_competitors):
                raise RaceConfigError(f"betting_close kth needs 1 <= k <= {n_competitors}, got {self.k}")
        elif self.k is not None:
            raise RaceConfigError(f"betting_close {self.rule!r} takes no k")


@dataclass(frozen=True)
class RaceConfig:
    """Race parameters (race.py:158-189).  ``dt`` and ``betting_close`` do not enter a step."""

    track_length: float
    competitors: tuple[Competitor, ...]
    dt: float = 1.0
    conditions: float = 0.5
    betting_close: BettingClose = field(default_factory=BettingClose.last)
    tick_limit: int = DEFAULT_TICK_LIMIT

    @property
    def n_competitors(self) -> int:
        return len(self.competitors)

    @property
    def competitor_ids(self) -> tuple[str, ...]:
        return tuple(c.cid for c in self.competitors)

    def validate(self) -> None:
        validate_config(self)


def validate_config(cfg) -> None:
    """RaceConfig.validate (race.py:175-189), usable on reference config objects too."""
    if cfg.track_length <= 0.0:
        raise RaceConfigError(f"track_length must be > 0, got {cfg.track_length}")
    if cfg.dt <= 0.0:
        raise RaceConfigError(f"dt must be > 0, got {cfg.dt}")
    if cfg.tick_limit < 1:
        raise RaceConfigError(f"tick_limit must be >= 1, got {cfg.tick_limit}")
    if not cfg.competitors:
        raise RaceConfigError("a race needs at least one competitor")
    ids = [c.cid for c in cfg.competitors]
    if len(set(ids)) != len(ids):
        raise RaceConfigError(f"competitor ids must be unique, got {ids}")
    for c in cfg.competitors:
        c.validate()
    cfg.betting_close.validate(len(cfg.competitors))


def preference_factor(conditions: float, preference: float, sensitivity: float) -> float:
    """Conditions multiplier clamped to [0.01, 1] (race.py:192-199).

    Evaluated once per competitor per launch on the host in Python double -- the exact value the
    reference recomputes on every free step -- and shipped to the kernel as ``pref_factor``.
    """
    f = 1.0 - sensitivity * abs(conditions - preference)
    return MIN_PREFERENCE_FACTOR if f < MIN_PREFERENCE_FACTOR else (1.0 if f > 1.0 else f)


@dataclass
class RaceState:
    """Mid-race state (race.py:207-230); ``finish_ticks[c] is None`` while c is racing."""

    tick: int
    positions: list[float]
    prev_steps: list[float]
    finish_ticks: list[int | None]
    blocked_steps: int = 0

    def clone(self) -> "RaceState":
        return RaceState(self.tick, list(self.positions), list(self.prev_steps), list(self.finish_ticks),
                         self.blocked_steps)

    def finished_count(self) -> int:
        return sum(t is not None for t in self.finish_ticks)

    def all_finished(self) -> bool:
        return all(t is not None for t in self.finish_ticks)


@dataclass(frozen=True)
class Trajectory:
    """Completed race record (race.py:335-353)."""

    competitor_ids: tuple[str, ...]
    dt: float
    ticks: tuple[tuple[float, ...], ...] | None
    finish_ticks: tuple[int, ...]
    finish_order: tuple[str, ...]
    final_positions: tuple[float, ...]
    blocked_steps: int

    @property
    def n_ticks(self) -> int:
        return max(self.finish_ticks)

    @property
    def winner(self) -> str:
        return self.finish_order[0]


# -- GPU-backed entry points (thin wrappers over sim.py) ----------------------------------------


def simulate_from(state, config, seed: int, *, mode: str = "mt") -> tuple[str, ...]:
    """Finish order of one continuation of ``state`` (race.py:393-406) computed on the GPU.

    ``mode="mt"`` (default) reproduces the reference's CPython MT19937 stream from ``seed`` in-kernel,
    so the result equals the reference's for the same seed.  ``mode="native"`` uses the Philox stream.
    """
    from .sim import simulate_from as _sf

    return _sf(state, config, seed, mode=mode)


def run_race(config, seed: int, record: bool = True, *, mode: str = "mt") -> Trajectory:
    """One race from the start line (race.py:373-390) on the GPU (``mode="mt"``: the reference's
    result for the same seed)."""
    from .sim import run_race as _rr

    return _rr(config, seed, record=record, mode=mode)
