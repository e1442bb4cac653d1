"""File products of GPU runs, in the reference's formats (racemarket/writers.py), plus the race
section of its JSON config (config.py:93-178) so the GPU CLI reads the same experiment files.

Only the simulation products are here: runs.csv / pmf.csv (batch), bench.csv, trajectory.csv and
finish.csv (race).  Session products (events, settlement, sentiment) belong to the host exchange
loop and stay out of scope.  Numbers are written with repr precision, as the reference does.
"""

from __future__ import annotations

import csv
import json
from pathlib import Path

from .batch import BenchPoint, OutcomePMF, RaceResult
from .race import (
    BettingClose,
    Competitor,
    LogNormalSteps,
    RaceConfig,
    RaceConfigError,
    Responsiveness,
    Trajectory,
    UniformSteps,
)

_RACE_KEYS = ("track_length", "dt", "conditions", "betting_close", "tick_limit", "competitors")
_COMP_KEYS = ("id", "steps", "preference", "pref_sensitivity", "theta", "responsiveness")


class ConfigError(RaceConfigError):
    pass


def _check(obj, allowed, path):
    if not isinstance(obj, dict):
        raise ConfigError(f"{path}: must be an object")
    extra = sorted(set(obj) - set(allowed))
    if extra:
        raise ConfigError(f"{path}: unknown keys {extra}")


def _steps(obj, path):
    family = obj.get("family")
    if family == "uniform":
        if "lo" not in obj or "hi" not in obj:
            raise ConfigError(f"{path}: uniform steps need lo and hi")
        return UniformSteps(float(obj["lo"]), float(obj["hi"]))
    if family == "lognormal":
        if "mu" not in obj or "sigma" not in obj:
            raise ConfigError(f"{path}: lognormal steps need mu and sigma")
        return LogNormalSteps(float(obj["mu"]), float(obj["sigma"]), float(obj.get("scale", 1.0)))
    raise ConfigError(f"{path}.family: must be 'uniform' or 'lognormal', got {family!r}")


def parse_race(obj, path: str = "race") -> RaceConfig:
    """The race section with the reference's defaults (config.py:160-178)."""
    _check(obj, _RACE_KEYS, path)
    comps = obj.get("competitors")
    if not isinstance(comps, list) or not comps:
        raise ConfigError(f"{path}.competitors: must be a non-empty list")
    parsed = []
    for i, c in enumerate(comps):
        p = f"{path}.competitors[{i}]"
        _check(c, _COMP_KEYS, p)
        cid = c.get("id", "")
        if not cid or "-" in cid or "," in cid:
            raise ConfigError(f"{p}.id: required, without '-' or ','")
        r = c.get("responsiveness", {})
        parsed.append(Competitor(cid, _steps(c.get("steps", {}), f"{p}.steps"),
                                 preference=float(c.get("preference", 0.5)),
                                 pref_sensitivity=float(c.get("pref_sensitivity", 0.0)),
                                 theta=float(c.get("theta", 0.0)),
                                 responsiveness=Responsiveness(float(r.get("early_mult", 1.0)),
                                                               float(r.get("late_mult", 1.0)),
                                                               float(r.get("breakpoint", 0.5)))))
    close = obj.get("betting_close", "last")
    bc = BettingClose.kth(int(close["kth"])) if isinstance(close, dict) else BettingClose(close)
    cfg = RaceConfig(track_length=float(obj.get("track_length", 2000.0)), competitors=tuple(parsed),
                     dt=float(obj.get("dt", 1.0)), conditions=float(obj.get("conditions", 0.5)),
                     betting_close=bc, tick_limit=int(obj.get("tick_limit", 1_000_000)))
    cfg.validate()
    return cfg


def load_experiment(path) -> tuple[dict, RaceConfig, int]:
    doc = json.loads(Path(path).read_text())
    return doc, parse_race(doc.get("race", {})), int(doc.get("seed", 0))


def write_trajectory_csv(path, traj: Trajectory) -> None:
    if traj.ticks is None:
        raise ValueError("trajectory was recorded without per-tick snapshots")
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["tick", "competitor_id", "position"])
        for tick, row in enumerate(traj.ticks):
            for cid, pos in zip(traj.competitor_ids, row):
                w.writerow([tick, cid, repr(pos)])


def write_finish_csv(path, traj: Trajectory) -> None:
    ranks = {cid: rank for rank, cid in enumerate(traj.finish_order, start=1)}
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["competitor_id", "finish_tick", "finish_rank"])
        for cid, tick in zip(traj.competitor_ids, traj.finish_ticks):
            w.writerow([cid, tick, ranks[cid]])


def write_race_runs_csv(path, results: list[RaceResult]) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["run", "winner", "winner_ticks", "n_ticks", "finish_order"])
        for r in results:
            w.writerow([r.run_index, r.winner, r.winner_ticks, r.n_ticks, "-".join(r.finish_order)])


def write_pmf_csv(path, pmf: OutcomePMF) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["outcome", "count", "frequency"])
        for key in sorted(pmf.counts):
            w.writerow([key, pmf.counts[key], repr(pmf.counts[key] / pmf.n_samples)])


def read_pmf_csv(path) -> OutcomePMF:
    counts: dict[str, int] = {}
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header is None or header[:2] != ["outcome", "count"]:
            raise ValueError(f"{path}: not a PMF table (header {header!r})")
        for row in reader:
            if row:
                counts[row[0]] = int(row[1])
    if not counts:
        raise ValueError(f"{path}: PMF table has no rows")
    return OutcomePMF("order" if any("-" in k for k in counts) else "winner", sum(counts.values()), counts)


def write_bench_csv(path, points: list[BenchPoint]) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["n_competitors", "mean_s", "sd_s", "cv", "reps"])
        for p in points:
            w.writerow([p.n_competitors, repr(p.mean_s), repr(p.sd_s), repr(p.cv), p.reps])
