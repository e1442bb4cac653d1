"""B200-native batched Monte Carlo race simulator (the BBE dry-run hot path).

Drop-in for the simulation entry points of the reference ``racemarket`` package
(arXiv 2108.02419, /root/reference/pkg/src/racemarket): the race types, ``simulate_from``,
``run_race``, ``rp_predict`` and ``run_batch`` keep their signatures; the work runs in hand-written
sm_100a kernels behind the C-ABI declared in ``include/bbe_sim.h``.
"""

__version__ = "0.1.0"

from .race import (  # noqa: F401
    DEFAULT_TICK_LIMIT,
    BettingClose,
    Competitor,
    LogNormalSteps,
    RaceConfig,
    RaceConfigError,
    RaceDivergedError,
    RaceState,
    Responsiveness,
    Trajectory,
    UniformSteps,
    preference_factor,
    run_race,
    simulate_from,
)
