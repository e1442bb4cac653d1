"""Loaders for the committed golden vectors (tests/golden/, made by make_golden.py from the reference)."""

from __future__ import annotations

import functools
import gzip
import json
import os

from paper_2108_02419_b200.race import (
    Competitor,
    LogNormalSteps,
    RaceConfig,
    RaceState,
    Responsiveness,
    UniformSteps,
)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def config_from_dict(d: dict) -> RaceConfig:
    comps = []
    for c in d["competitors"]:
        if c["family"] == "uniform":
            steps = UniformSteps(c["lo"], c["hi"])
        else:
            steps = LogNormalSteps(c["mu"], c["sigma"], c["scale"])
        comps.append(Competitor(c["id"], steps, preference=c["preference"], pref_sensitivity=c["pref_sensitivity"],
                                theta=c["theta"], responsiveness=Responsiveness(c["early_mult"], c["late_mult"],
                                                                                 c["breakpoint"])))
    return RaceConfig(track_length=d["track_length"], competitors=tuple(comps), dt=d.get("dt", 1.0),
                      conditions=d["conditions"], tick_limit=d["tick_limit"])


def state_from_dict(d: dict) -> RaceState:
    return RaceState(d["tick"], list(d["positions"]), list(d["prev_steps"]), list(d["finish_ticks"]),
                     d.get("blocked_steps", 0))


@functools.lru_cache(None)
def rng_vectors() -> dict:
    with open(os.path.join(GOLDEN, "rng.json")) as fh:
        return json.load(fh)


@functools.lru_cache(None)
def race_corpus() -> list:
    with gzip.open(os.path.join(GOLDEN, "races.json.gz"), "rt") as fh:
        return json.load(fh)["corpus"]


@functools.lru_cache(None)
def c2() -> dict:
    with open(os.path.join(GOLDEN, "c2.json")) as fh:
        return json.load(fh)


@functools.lru_cache(None)
def acceptance() -> dict:
    """tests/golden/acceptance.json.gz (make_acceptance_golden.py): reference criteria 7 and 8."""
    with gzip.open(os.path.join(GOLDEN, "acceptance.json.gz"), "rt") as fh:
        return json.load(fh)


def plain_race(spec: dict) -> RaceConfig:
    """The reference tests' make_race (tests/conftest.py:6-8): n identical U(lo, hi) runners c1..cn."""
    return RaceConfig(track_length=spec["length"],
                      competitors=tuple(Competitor(f"c{i + 1}", UniformSteps(spec["lo"], spec["hi"]))
                                        for i in range(spec["n"])))
