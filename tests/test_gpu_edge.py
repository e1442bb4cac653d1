"""Edge cases the reference handles (degenerate fields, finished states, divergence,
maximum sizes), through every mode of the kernel."""

import numpy as np
import pytest

import oracle
from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.race import (
    Competitor,
    LogNormalSteps,
    RaceConfig,
    RaceConfigError,
    RaceState,
    Responsiveness,
    UniformSteps,
)

pytestmark = pytest.mark.gpu


def _field(n, theta=0.0, L=80.0):
    return RaceConfig(L, tuple(Competitor(f"c{i}", UniformSteps(2.0 + i % 3, 6.0 + i % 4), theta=theta * (i % 2))
                               for i in range(n)))


@pytest.mark.parametrize("mode", ["native", "mt"])
def test_zero_sims_and_single_competitor(mode):
    cfg = _field(1)
    r = sim.simulate_batch(None, cfg, 0, 1, mode=mode, seed_master=1)
    assert r.wins.tolist() == [0] and r.competitor_steps == 0
    r = sim.simulate_batch(None, cfg, 1000, 1, mode=mode, seed_master=1, records=True)
    assert r.wins.tolist() == [1000] and (r.order == 0).all()
    if mode == "mt":
        o = oracle.run_race(cfg, oracle.derive_seed_run(1, 7))
        assert r.final_positions[7].tolist() == o.final_positions.tolist()


@pytest.mark.parametrize("mode", ["native", "mt", "inject"])
def test_state_already_finished(mode):
    cfg = _field(3)
    st = RaceState(12, [90.0, 85.0, 81.0], [5.0, 5.0, 5.0], [11, 12, 12])
    kw = {}
    if mode == "inject":
        kw = dict(draws=np.zeros(0), draw_offsets=np.zeros(4, np.int64))
    if mode == "mt":
        kw = dict(seeds=np.arange(3, dtype=np.uint64))
    r = sim.simulate_batch(st, cfg, 3, 5, mode=mode, records=True, **kw)
    # finish tick first, then larger overshoot (L - pos smaller): c0 (11), then c1 (85 > 81), then c2
    assert (r.order == [0, 1, 2]).all() and r.competitor_steps == 0
    assert (r.finish_ticks == [11, 12, 12]).all()


@pytest.mark.parametrize("mode", ["native", "mt"])
def test_divergence_everywhere(mode):
    cfg = RaceConfig(100.0, (Competitor("a", UniformSteps(1.0, 1.0)), Competitor("b", UniformSteps(1.0, 1.0))),
                     tick_limit=10)
    with pytest.raises(sim.SimDivergedError) as e:
        sim.simulate_batch(None, cfg, 500, 1, mode=mode, seed_master=1, sim_offset=40)
    assert e.value.sim_index == 40
    st = RaceState(50, [10.0, 20.0], [1.0, 1.0], [None, None])
    with pytest.raises(sim.SimDivergedError):
        sim.simulate_batch(st, cfg, 5, 1, mode=mode, seeds=np.arange(5, dtype=np.uint64) if mode == "mt" else None)
    # a limit that is exactly enough: 2 ticks from 98 with unit steps
    ok = RaceConfig(100.0, cfg.competitors, tick_limit=2)
    st2 = RaceState(50, [98.0, 98.5], [1.0, 1.0], [None, None])
    r = sim.simulate_batch(st2, ok, 4, 1, mode=mode, seeds=np.arange(4, dtype=np.uint64) if mode == "mt" else None,
                           records=True)
    assert (r.finish_ticks == [52, 52]).all() and (r.order == [1, 0]).all()


def test_negative_positions_are_shifted_not_misordered():
    """Native mode keys positions by their float bits after an offset; a state with negative
    positions must behave like the same state shifted (statistically) and order exactly."""
    fixed = lambda v: UniformSteps(v, v)  # noqa: E731
    cfg = RaceConfig(10.0, (Competitor("a", fixed(4.0), theta=3.0), Competitor("b", fixed(3.0))))
    st = RaceState(0, [-5.0, -3.0], [2.0, 2.0], [None, None])
    r = sim.simulate_batch(st, cfg, 16, 1, records=True)
    o = oracle.simulate_from(st, cfg, 1)  # degenerate draws: the same race for any seed
    assert (r.order == o.order.tolist()).all() and (r.finish_ticks == o.finish_ticks.tolist()).all()
    assert (r.final_positions == o.final_positions.tolist()).all() and (r.blocked == o.blocked).all()


@pytest.mark.parametrize("n", [31, 32, 33, 64, 97, 128])
def test_large_fields_native_layouts(n):
    cfg = _field(n, theta=1.5, L=60.0)
    r = sim.simulate_batch(None, cfg, 20_000, 9, records=True)
    assert int(r.wins.sum()) == 20_000 and (np.sort(r.order, axis=1) == np.arange(n)).all()
    ref = oracle.batch(cfg, 4000, master=9, threads=8)
    # mean race length in competitor-timesteps agrees with the reference's within 1 %
    assert abs(r.competitor_steps / 20_000 - ref["ct"] / 4000) / (ref["ct"] / 4000) < 0.01


def _mixed_field(n, L=60.0):
    """Uniform and lognormal competitors with alternating theta: blocked steps and rejections in
    every slot of a multi-slot lane layout."""
    comps = []
    for i in range(n):
        steps = LogNormalSteps(0.4 + 0.01 * (i % 7), 0.35, 2.0) if i % 3 == 0 else UniformSteps(2.0 + i % 3, 5.0 + i % 4)
        comps.append(Competitor(f"c{i}", steps, theta=1.2 * (i % 2)))
    return RaceConfig(L, tuple(comps))


@pytest.mark.parametrize("n", [33, 40, 64, 65, 97, 128])
def test_mt_multi_slot_fields_bit_exact(n):
    """n > 32 puts K = ceil(n/32) competitors in every lane; the speculative MT rounds then span
    the slots in index order (slot-major) -- positions, ticks and orders must stay bit-exact."""
    cfg = _mixed_field(n)
    seeds = oracle.rp_seeds(11, 300)
    r = sim.simulate_batch(None, cfg, 300, mode="mt", seeds=seeds, records=True)
    assert int(r.wins.sum()) == 300
    for i in (0, 1, 2, 150, 299):
        o = oracle.run_race(cfg, int(seeds[i]))
        assert r.final_positions[i].tolist() == o.final_positions.tolist()
        assert r.finish_ticks[i].tolist() == o.finish_ticks.tolist()
        assert r.order[i].tolist() == o.order.tolist()
        assert int(r.blocked[i]) == o.blocked
    # a continuation state (simulate_from) with finished and racing competitors
    st = RaceState(6, [3.0 + 0.5 * (i % 11) for i in range(n)], [2.5] * n,
                   [5 if i == 4 else None for i in range(n)])
    st.positions[4] = 61.0
    r = sim.simulate_batch(st, cfg, 100, mode="mt", seeds=seeds[:100], records=True)
    for i in (0, 57, 99):
        o = oracle.simulate_from(st, cfg, int(seeds[i]))
        assert r.final_positions[i].tolist() == o.final_positions.tolist()
        assert r.order[i].tolist() == o.order.tolist()


def test_lognormal_zero_sigma_and_responsiveness_edges():
    comps = (Competitor("a", LogNormalSteps(1.0, 0.0, 2.0)),
             Competitor("b", UniformSteps(5.0, 6.0), responsiveness=Responsiveness(0.5, 2.0, 0.0)),
             Competitor("c", UniformSteps(5.0, 6.0), responsiveness=Responsiveness(2.0, 0.5, 1.0)))
    cfg = RaceConfig(50.0, comps)
    seeds = oracle.rp_seeds(3, 500)
    r = sim.simulate_batch(None, cfg, 500, mode="mt", seeds=seeds, records=True)
    for i in (0, 1, 499):
        o = oracle.run_race(cfg, int(seeds[i]))
        assert r.final_positions[i].tolist() == o.final_positions.tolist()


@pytest.mark.parametrize("n", [3, 12, 31, 40, 100])
def test_native_front_runner_ties_are_exact(n):
    """Degenerate U(v, v) steps on a half-integer grid make every FP32 operation exact, so native
    mode must reproduce the reference race bit for bit -- including rivals on identical positions,
    where the front runner is the lowest index (race.py:244-264), within a slot and across slots."""
    rng = np.random.default_rng(n)
    comps = tuple(Competitor(f"c{i}", UniformSteps(v, v), theta=float(th))
                  for i, (v, th) in enumerate(zip(rng.integers(1, 9, n) * 0.5, rng.choice([0.0, 1.0, 2.5], n))))
    cfg = RaceConfig(60.0, comps)
    pos = rng.integers(0, 12, n) * 0.5  # many shared positions
    prev = rng.integers(1, 9, n) * 0.5
    st = RaceState(3, pos.tolist(), prev.tolist(), [None] * n)
    r = sim.simulate_batch(st, cfg, 8, 1, records=True)
    o = oracle.simulate_from(st, cfg, 1)
    assert o.blocked > 0
    for i in range(8):
        assert r.final_positions[i].tolist() == o.final_positions.tolist()
        assert r.finish_ticks[i].tolist() == o.finish_ticks.tolist()
        assert r.order[i].tolist() == o.order.tolist()
        assert int(r.blocked[i]) == o.blocked
    # from the start line (run_race: priming draws, everyone level at 0.0)
    r = sim.simulate_batch(None, cfg, 4, 1, records=True)
    o = oracle.run_race(cfg, 1)
    for i in range(4):
        assert r.final_positions[i].tolist() == o.final_positions.tolist()
        assert r.order[i].tolist() == o.order.tolist()
        assert int(r.blocked[i]) == o.blocked


@pytest.mark.parametrize("mode", ["native", "mt", "inject"])
def test_multi_part_split_is_invisible(mode):
    """bbe_simulate_multi: any number of parts (mapped round-robin onto the visible GPUs) gives the
    single-launch tallies and per-sim outputs bit for bit; errors keep the smallest failing index."""
    cfg = _mixed_field(7)
    n_sims = 1001
    kw = {}
    if mode == "mt":
        kw = dict(seeds=oracle.rp_seeds(5, n_sims))
    if mode == "inject":
        seeds = oracle.rp_seeds(6, n_sims)
        recs = [oracle.run_race(cfg, int(s), record=True) for s in seeds]
        offs = np.zeros(n_sims + 1, np.int64)
        offs[1:] = np.cumsum([r.draws_used for r in recs])
        kw = dict(draws=np.concatenate([r.draws[: r.draws_used] for r in recs]), draw_offsets=offs)
    one = sim.simulate_batch(None, cfg, n_sims, 3, mode=mode, records=True, perms=False, **kw)
    for parts in (1, 3, 8):
        r = sim.simulate_batch(None, cfg, n_sims, 3, mode=mode, records=True, parts=parts, **kw)
        assert (r.wins == one.wins).all() and (r.ranks == one.ranks).all()
        assert r.competitor_steps == one.competitor_steps and r.blocked_steps == one.blocked_steps
        assert (r.order == one.order).all() and (r.finish_ticks == one.finish_ticks).all()
        assert (r.final_positions == one.final_positions).all() and (r.blocked == one.blocked).all()
    # divergence in a later part is reported with its global index
    slow = RaceConfig(100.0, (Competitor("a", UniformSteps(1.0, 1.0)), Competitor("b", UniformSteps(1.0, 1.0))),
                      tick_limit=10)
    with pytest.raises(sim.SimDivergedError) as e:
        sim.simulate_batch(None, slow, 300, 1, mode="native", sim_offset=40, parts=4)
    assert e.value.sim_index == 40


@pytest.mark.parametrize("mode", ["native", "native64", "mt"])
def test_multi_tally_only_device_path(mode):
    """bbe_simulate_multi without per-sim outputs: every part adds into one device tally per GPU and
    the devices are combined by one grouped NCCL all-reduce (one GPU here: the device accumulation,
    no collective) -- tallies equal one launch's bit for bit, with perms, for any number of parts;
    MT derives run seeds on the device (seed_master) like run_batch."""
    cfg = _mixed_field(5)
    n_sims = 20_011
    kw = dict(seed_master=4321) if mode == "mt" else {}
    one = sim.simulate_batch(None, cfg, n_sims, 3, mode=mode, perms=True, **kw)
    for parts in (1, 2, 7):
        r = sim.simulate_batch(None, cfg, n_sims, 3, mode=mode, perms=True, parts=parts, **kw)
        assert (r.wins == one.wins).all() and (r.ranks == one.ranks).all() and (r.perms == one.perms).all()
        assert r.competitor_steps == one.competitor_steps and r.blocked_steps == one.blocked_steps
        assert r.kernel_ms > 0


@pytest.mark.parametrize("mode", ["native", "mt"])
def test_group_wins_equal_per_group_winner_counts(mode):
    """req.group_size: per-group winner counts from the kernel equal the host split of the per-sim
    winners (ragged last group, MT seeding chunks, multi-part shards on group edges)."""
    cfg = _mixed_field(6)
    n_sims, g = 140_000, 1000  # > one MT seeding chunk (131072)
    kw = dict(seeds=oracle.rp_seeds(9, n_sims)) if mode == "mt" else {}
    ref = sim.simulate_batch(None, cfg, n_sims, 5, mode=mode, winners=True, ranks=False, **kw)
    want = np.bincount((np.arange(n_sims) // g) * 6 + ref.winner, minlength=((n_sims + g - 1) // g) * 6)
    r = sim.simulate_batch(None, cfg, n_sims, 5, mode=mode, ranks=False, group_size=g, **kw)
    assert r.group_wins.reshape(-1).tolist() == want.tolist()
    r = sim.simulate_batch(None, cfg, 2500, 5, mode=mode, ranks=False, group_size=300, parts=3,
                           **({"seeds": kw["seeds"][:2500]} if kw else {}))
    w = sim.simulate_batch(None, cfg, 2500, 5, mode=mode, winners=True, ranks=False,
                           **({"seeds": kw["seeds"][:2500]} if kw else {})).winner
    assert r.group_wins.reshape(-1).tolist() == np.bincount((np.arange(2500) // 300) * 6 + w, minlength=9 * 6).tolist()


def test_concurrent_host_threads_and_overlapping_calls():
    """Calls from several host threads (and several begin/end calls in flight from one thread) each
    lease their own context: results equal the sequential ones."""
    import threading

    cfg = _mixed_field(8)
    want = {seed: sim.simulate_batch(None, cfg, 20_000, seed, ranks=True).ranks.copy() for seed in range(8)}
    got = {}

    def work(seed):
        got[seed] = sim.simulate_batch(None, cfg, 20_000, seed, ranks=True).ranks

    threads = [threading.Thread(target=work, args=(seed,)) for seed in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert all((got[s] == want[s]).all() for s in range(8))
    pend = [sim.simulate_batch_begin(None, cfg, 20_000, seed, ranks=True) for seed in range(3)]
    for seed, p in reversed(list(enumerate(pend))):
        assert (p.end().ranks == want[seed]).all()


def test_mt_multi_slot_divergence_finished_and_trajectories():
    """K > 1 in the exact kernel: tick-limit divergence, pre-finished competitors and recorded
    trajectories all follow the reference (oracle) for a 40-runner field."""
    cfg = _mixed_field(40)
    # trajectories (run_race(record=True)) from the start line
    seeds = oracle.rp_seeds(21, 3)
    r = sim.simulate_batch(None, cfg, 3, mode="mt", seeds=seeds, records=True, trajectory_ticks=400)
    for i, s in enumerate(seeds):
        o = oracle.run_race(cfg, int(s))
        assert r.final_positions[i].tolist() == o.final_positions.tolist()
        for k in (1, 5, int(o.n_ticks_run) // 2):
            _, pos, prev, _, _ = oracle.advance_from_start(cfg, int(s), k)
            assert r.traj_positions[i, k].tolist() == pos.tolist()
            assert r.traj_prev_steps[i, k].tolist() == prev.tolist()
    # a state where some runners already finished, continued in MT mode
    n = 40
    st = RaceState(9, [62.0 if i % 7 == 0 else 2.0 + 0.5 * (i % 13) for i in range(n)], [3.0] * n,
                   [8 if i % 7 == 0 else None for i in range(n)])
    r = sim.simulate_batch(st, cfg, 4, mode="mt", seeds=np.tile(seeds[:2], 2), records=True)
    for i in range(4):
        o = oracle.simulate_from(st, cfg, int(seeds[i % 2]))
        assert r.order[i].tolist() == o.order.tolist() and r.finish_ticks[i].tolist() == o.finish_ticks.tolist()
    # divergence: the first sim that runs out of ticks is reported by global index
    tight = RaceConfig(cfg.track_length, cfg.competitors, tick_limit=5)
    with pytest.raises(sim.SimDivergedError) as e:
        sim.simulate_batch(None, tight, 6, mode="mt", seeds=oracle.rp_seeds(3, 6), sim_offset=100)
    assert e.value.sim_index == 100


@pytest.mark.parametrize("mode", ["native", "mt"])
def test_continuation_is_pure_and_deterministic(mode):
    """tests/test_race.py:232-235, 285-300: simulate_from never mutates its input state, the same
    seed gives the same result, a different seed a different one."""
    cfg = _mixed_field(10)
    st = RaceState(7, [3.0 + i for i in range(10)], [2.0] * 10, [None] * 10)
    snapshot = (st.tick, list(st.positions), list(st.prev_steps), list(st.finish_ticks))
    kw = lambda s: dict(seeds=oracle.rp_seeds(s, 2000)) if mode == "mt" else {}  # noqa: E731
    a = sim.simulate_batch(st, cfg, 2000, 5, mode=mode, records=True, **kw(5))
    b = sim.simulate_batch(st, cfg, 2000, 5, mode=mode, records=True, **kw(5))
    c = sim.simulate_batch(st, cfg, 2000, 6, mode=mode, records=True, **kw(6))
    assert (st.tick, st.positions, st.prev_steps, st.finish_ticks) == snapshot
    assert (a.order == b.order).all() and (a.final_positions == b.final_positions).all()
    assert not (a.order == c.order).all()
    assert sim.simulate_from(st, cfg, 123, mode=mode) == sim.simulate_from(st, cfg, 123, mode=mode)


@pytest.mark.parametrize("mode", ["native", "mt"])
def test_extreme_step_laws_terminate_or_diverge_cleanly(mode):
    """Heavy-tailed lognormal steps (sigma 4: steps from ~1e-5 to ~1e5), tiny steps that need
    nextafter, and a huge track: every sim finishes or is reported diverged -- no hang, no garbage."""
    heavy = RaceConfig(500.0, (Competitor("h", LogNormalSteps(0.0, 4.0, 1.0), theta=2.0),
                               Competitor("u", UniformSteps(5.0, 15.0), theta=1.0),
                               Competitor("g", LogNormalSteps(2.0, 0.1, 1.0))))
    def kw(key, n):
        return dict(seeds=oracle.rp_seeds(key, n)) if mode == "mt" else {}

    r = sim.simulate_batch(None, heavy, 5000, 3, mode=mode, records=True, **kw(3, 5000))
    assert int(r.wins.sum()) == 5000 and (np.sort(r.order, axis=1) == np.arange(3)).all()
    assert np.isfinite(r.final_positions).all() or mode == "native"
    tiny = RaceConfig(1.0, (Competitor("t", LogNormalSteps(-80.0, 0.0, 1.0)),), tick_limit=50)
    with pytest.raises(sim.SimDivergedError):
        sim.simulate_batch(None, tiny, 10, 1, mode=mode, **kw(4, 10))
    far = RaceConfig(1e6, (Competitor("a", UniformSteps(4e4, 6e4)), Competitor("b", UniformSteps(4.5e4, 5.5e4), theta=5e3)))
    r = sim.simulate_batch(None, far, 2000, 9, mode=mode, ranks=True, **kw(9, 2000))
    assert int(r.wins.sum()) == 2000


@pytest.mark.parametrize("mode", ["mt", "native"])
def test_rp_predict_c_entry_errors(mode):
    """bbe_rp_predict: a dry run past tick_limit raises with the first failing dry-run index (both MT
    halves included) and leaves the bettor's stream where the reference leaves it -- advanced by
    first_diverged + 1 draws, as rp_predict raises inside that dry run (agents.py:164); bad arguments
    are rejected."""
    import ctypes
    import random

    from paper_2108_02419_b200.agents import rp_predict

    cfg = RaceConfig(100.0, (Competitor("a", UniformSteps(1.0, 1.0)), Competitor("b", UniformSteps(1.0, 1.0))),
                     tick_limit=10)
    st = RaceState(50, [10.0, 20.0], [1.0, 1.0], [None, None])
    d = 40_000
    rng, twin = random.Random(3), random.Random(3)
    with pytest.raises(sim.SimDivergedError) as e:
        rp_predict(st, cfg, d, rng, mode=mode)
    assert e.value.sim_index == 0
    for _ in range(e.value.sim_index + 1):
        twin.getrandbits(64)
    assert rng.getstate() == twin.getstate()
    pk = sim.pack_config(cfg)
    stc, keep = sim.pack_state(st, pk.n)
    mt = np.zeros(624, np.uint32)
    pos = np.array([625], np.int32)  # outside 0..624
    wins = np.zeros(2, np.uint64)
    rc = sim.lib().bbe_rp_predict(ctypes.byref(pk.race), pk.comps, ctypes.byref(stc), 10, sim.MODES[mode],
                                  mt.ctypes.data, pos.ctypes.data, wins.ctypes.data, None)
    assert rc == 1
    pos[0] = 0
    rc = sim.lib().bbe_rp_predict(ctypes.byref(pk.race), pk.comps, ctypes.byref(stc), 10, sim.MODES["inject"],
                                  mt.ctypes.data, pos.ctypes.data, wins.ctypes.data, None)
    assert rc == 1
