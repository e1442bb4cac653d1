"""The C-ABI from plain C (examples/c_abi_demo.c, no Python in the loop): compiled with gcc against
include/bbe_sim.h and the in-tree library, run, and its MT-mode probabilities checked against the
oracle for the same derive_seed(11, "run", i) seeds."""

import os
import subprocess

import numpy as np

import pytest

import oracle
from paper_2108_02419_b200.race import Competitor, RaceConfig, RaceState, UniformSteps

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_drives_the_library(tmp_path):
    exe = str(tmp_path / "c_abi_demo")
    lib_dir = os.path.join(ROOT, "paper_2108_02419_b200", "_lib")
    subprocess.run(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", lib_dir, "-lbbe_sim",
                    f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.splitlines()
    rows = {line.split()[0]: [float(x) for x in line.split("probs")[1].split()] for line in out}
    assert set(rows) == {"native", "native64", "mt", "multi64", "rp_mt"}
    n, d = 10, 20000
    comps = tuple(Competitor(f"c{c}", UniformSteps(10.0 + c % 3, 20.0 + c % 4), theta=8.0 if c % 2 else 0.0)
                  for c in range(n))
    cfg = RaceConfig(2000.0, comps)
    st = RaceState(65, [900.0 + 12.5 * c for c in range(n)], [15.0] * n, [None] * n)
    ref = oracle.batch(cfg, d, state=st, master=11, threads=8)
    assert rows["mt"] == [(int(w) + 1) / (d + n) for w in ref["wins"]]
    assert abs(sum(rows["native"]) - 1.0) < 1e-9
    # NATIVE64 (seed 7): the oracle's restatement of the same Philox stream, and bbe_simulate_multi
    # gives the single-call tallies
    ref64 = oracle.batch_px(cfg, d, 7, state=st, threads=8)
    assert rows["native64"] == [(int(w) + 1) / (d + n) for w in ref64["wins"]]
    assert rows["multi64"] == rows["native64"]
    # bbe_rp_predict with random.Random(5) as the bettor: the reference's rp_predict over its seeds
    import random

    bettor = random.Random(5)
    seeds = [bettor.getrandbits(64) for _ in range(d)]
    ref = oracle.batch(cfg, d, state=st, seeds=np.array(seeds, np.uint64), threads=8)
    assert rows["rp_mt"] == [(int(w) + 1) / (d + n) for w in ref["wins"]]
    pos = int([line for line in out if line.startswith("rp_mt")][0].split()[2])
    assert pos == bettor.getstate()[1][624]
