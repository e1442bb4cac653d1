"""CPU-side checks of the boundary: the C-ABI library loads, exports every symbol the header declares,
its host-only functions agree with the reference, and the product path refuses to run without a GPU
(no CPU fallback)."""

import os
import random
import re

import numpy as np
import pytest

from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.agents import dry_run_seeds
from paper_2108_02419_b200.race import Competitor, RaceConfig, RaceConfigError, UniformSteps
from golden_io import rng_vectors

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "bbe_sim.h")).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|float|void|const char\*)\s+(bbe_\w+)\(", src, re.M)))


def test_library_exports_every_header_symbol():
    L = sim.lib()
    declared = header_symbols()
    assert declared and set(declared) == set(sim.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.bbe_version() == sim.ABI_VERSION == 5


def test_tally_layout():
    L = sim.lib()
    for n in (1, 2, 5, 6, 7, 10, 20, 40, 128):
        nperm = 1
        for i in range(2, n + 1):
            nperm *= i
        nperm = nperm if n <= 6 else 0
        assert L.bbe_tally_len(n) == n + n * n + nperm + 6
        assert L.bbe_tally_offset(n, 0) == 0
        assert L.bbe_tally_offset(n, 1) == n
        assert L.bbe_tally_offset(n, 3) == n + n * n + nperm
    assert L.bbe_tally_len(0) == -1 and L.bbe_tally_len(129) == -1


def test_derive_seeds_matches_reference():
    L = sim.lib()
    for d in rng_vectors()["derive_seed_run"]:
        out = np.zeros(1, np.uint64)
        assert L.bbe_derive_seeds(int(d["master"]), d["i"], 1, out.ctypes.data_as(sim._P(sim.ctypes.c_uint64))) == 0
        assert int(out[0]) == int(d["seed"])


@pytest.mark.parametrize("d,pre", [(1, 0), (257, 0), (312, 3), (5000, 1)])
def test_dry_run_seeds_match_sequential_getrandbits(d, pre):
    """bbe_mt_getrandbits64 advances a CPython Random exactly like d x getrandbits(64) (agents.py:164)."""
    a, b = random.Random(11), random.Random(11)
    for _ in range(pre):
        a.random(), b.random()
    seeds = dry_run_seeds(a, d)
    assert [int(s) for s in seeds] == [b.getrandbits(64) for _ in range(d)]
    assert a.random() == b.random() and a.randrange(7) == b.randrange(7)  # same position afterwards
    c = random.Random(11)
    assert dry_run_seeds(c, d, want=False) is None and c.getstate() != random.Random(11).getstate()
    e, f = random.Random(5), random.Random(5)
    assert int(dry_run_seeds(e, d, first_only=True)[0]) == f.getrandbits(64)
    for _ in range(d - 1):
        f.getrandbits(64)
    assert e.getstate() == f.getstate()


def test_inplace_mt_layout_verified():
    from paper_2108_02419_b200 import agents

    assert agents._inplace_ok()  # CPython 3.12: RandomObject {PyObject_HEAD; int index; uint32_t state[624]}


def test_non_random_generators_fall_back_to_getrandbits():
    class Sys(random.Random):  # a subclass is not advanced in place
        pass

    a, b = Sys(3), random.Random(3)
    assert [int(s) for s in dry_run_seeds(a, 9)] == [b.getrandbits(64) for _ in range(9)]


def test_libm_exp_table_located_and_verified():
    """MT mode's lognormal steps need the host libm's exp bit for bit (Lib/random.py lognormvariate)."""
    assert sim.lib().bbe_mt_exp_exact() == 1


def test_validation_mirrors_reference_errors():
    bad = [
        RaceConfig(0.0, (Competitor("a", UniformSteps(1, 2)),)),
        RaceConfig(10.0, ()),
        RaceConfig(10.0, (Competitor("a", UniformSteps(1, 2)), Competitor("a", UniformSteps(1, 2)))),
        RaceConfig(10.0, (Competitor("a", UniformSteps(3, 2)),)),
        RaceConfig(10.0, (Competitor("a", UniformSteps(1, 2), theta=-1.0),)),
        RaceConfig(10.0, (Competitor("a", UniformSteps(1, 2)),), tick_limit=0),
    ]
    for cfg in bad:
        with pytest.raises(RaceConfigError):
            sim.pack_config(cfg)


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    cfg = RaceConfig(100.0, (Competitor("a", UniformSteps(1, 2)), Competitor("b", UniformSteps(1, 2))))
    with pytest.raises(sim.BackendUnavailable):
        sim.simulate_batch(None, cfg, 10, 1)


def test_batched_stream_advance_matches_sequential_getrandbits():
    """bbe_mt_advance64_many (a tick's bettors in one call, threads over generators) leaves every
    generator exactly where d sequential getrandbits(64) calls leave it and returns the values."""
    import random

    from paper_2108_02419_b200.agents import dry_run_seeds_many

    ds = [0, 1, 7, 311, 1000, 20000] * 6
    out_lens = [d if i % 3 else min(d, 1) for i, d in enumerate(ds)]
    a = [random.Random(1000 + i) for i in range(len(ds))]
    b = [random.Random(1000 + i) for i in range(len(ds))]
    outs = dry_run_seeds_many(a, ds, out_lens)
    for r, d, k, o in zip(b, ds, out_lens, outs):
        vals = [r.getrandbits(64) for _ in range(d)]
        if k:
            assert [int(x) for x in o] == vals[:k]
        else:
            assert o is None
    assert all(x.getstate() == y.getstate() for x, y in zip(a, b))


def test_generator_writes_hold_the_gil():
    """bbe_mt_advance64 writes a random.Random in place; bound through ctypes.PyDLL it holds the GIL,
    so a second thread using the same generator never sees (or makes) a half-written state.  Every
    operation consumes whole MT words, so whatever the interleaving the final state is the start
    advanced by the total number of words drawn."""
    import threading

    rng = random.Random(2021)
    calls_a, calls_b = 300, 20000
    d = 3000

    def a():
        for _ in range(calls_a):
            dry_run_seeds(rng, d, want=False)

    def b():
        for _ in range(calls_b):
            rng.random()

    ta, tb = threading.Thread(target=a), threading.Thread(target=b)
    ta.start(), tb.start()
    ta.join(), tb.join()
    ref = random.Random(2021)
    for _ in range(calls_a * d * 2 + calls_b * 2):
        ref.getrandbits(32)
    assert rng.getstate() == ref.getstate()


def test_duplicate_generators_advance_in_list_order():
    """bbe_mt_advance64_many with one generator listed several times: advanced once per listing, in
    order, by a single thread (no two threads write the same state)."""
    from paper_2108_02419_b200.agents import dry_run_seeds_many

    g1, g2 = random.Random(5), random.Random(6)
    rngs = [g1, g2, g1, g1, g2] * 8
    ds = [70000, 3, 70000, 5, 70000] * 8
    outs = dry_run_seeds_many(rngs, ds, [2] * len(rngs))
    r1, r2 = random.Random(5), random.Random(6)
    for r, d, o in zip(rngs, ds, outs):
        ref = r1 if r is g1 else r2
        vals = [ref.getrandbits(64) for _ in range(d)]
        assert [int(x) for x in o] == vals[:2]
    assert g1.getstate() == r1.getstate() and g2.getstate() == r2.getstate()
