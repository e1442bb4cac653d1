"""MT mode: the kernel regenerates each simulation's CPython MT19937 stream from its seed
(seeding.py:62-64) and consumes it exactly as race.py does, so outputs equal the reference's for the
same seeds -- no recorded draws needed.

Uniform step laws are bit-exact by construction (MT19937, random(), uniform() are exact integer/IEEE
operations).  Lognormal steps also run the reference's Kinderman-Monahan loop; the final exp() is
CUDA's double exp, which can differ from glibc's in the last bit for rare arguments -- those tests
assert exact outcomes and report any last-bit position differences.
"""

import numpy as np
import pytest

import oracle
from golden_io import c2, config_from_dict, race_corpus, state_from_dict
from paper_2108_02419_b200 import sim
from paper_2108_02419_b200.agents import rp_predict

pytestmark = pytest.mark.gpu


def _has_lognormal(cfg):
    return any(not hasattr(c.steps, "lo") for c in cfg.competitors)


def test_golden_corpus_from_seeds():
    exact_pos = total = pos_ulp_mismatch = 0
    for case in race_corpus():
        cfg = config_from_dict(case["config"])
        for path in ("run_race", "simulate_from"):
            exp = case[path]
            st = None if path == "run_race" else state_from_dict(exp["state"])
            if exp["error"] is not None:
                with pytest.raises(sim.SimDivergedError):
                    sim.simulate_batch(st, cfg, 1, mode="mt", seeds=np.array([exp["seed"]], np.uint64))
                continue
            r = sim.simulate_batch(st, cfg, 1, mode="mt", seeds=np.array([exp["seed"]], np.uint64), records=True)
            total += 1
            assert r.order[0].tolist() == exp["order"], case["name"]
            assert r.finish_ticks[0].tolist() == exp["finish_ticks"], case["name"]
            assert int(r.blocked[0]) == exp["blocked"], case["name"]
            same = r.final_positions[0].tolist() == exp["final_positions"]
            if not _has_lognormal(cfg) or sim.lib().bbe_mt_exp_exact():
                assert same, case["name"]
            exact_pos += same
            pos_ulp_mismatch += not same
    print(f"MT golden: {total} races, exact positions {exact_pos}, last-bit position differences {pos_ulp_mismatch}")
    assert pos_ulp_mismatch == 0 or not sim.lib().bbe_mt_exp_exact()


def test_rp_predict_mt_equals_reference():
    import random

    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    agent = random.Random(g["agent_seed"])
    probs = rp_predict(st, cfg, g["d"], agent, mode="mt")
    assert probs == tuple(g["probs"])
    assert agent.random() == g["agent_next_random"]  # the bettor's stream advanced exactly as the reference's


def test_rp_predict_mt_split_launches_equal_oracle():
    """d >= 2 * _MT_SPLIT_MIN runs as two overlapped launches: the probabilities are still the
    reference algorithm's over the bettor's d getrandbits(64) seeds, and the stream advances by d."""
    import random

    from paper_2108_02419_b200 import agents

    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    d = 2 * agents._MT_SPLIT_MIN + 7
    agent, twin = random.Random(5), random.Random(5)
    probs = rp_predict(st, cfg, d, agent, mode="mt")
    seeds = np.array([twin.getrandbits(64) for _ in range(d)], np.uint64)
    ob = oracle.batch(cfg, d, state=st, seeds=seeds, threads=8)
    n = cfg.n_competitors
    assert probs == tuple((int(w) + 1) / (d + n) for w in ob["wins"])
    assert agent.random() == twin.random()


@pytest.mark.parametrize("n_sims", [1, 97, 20_000])
def test_c2_batch_matches_oracle(n_sims):
    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    seeds = oracle.rp_seeds(99, n_sims)
    r = sim.simulate_batch(st, cfg, n_sims, mode="mt", seeds=seeds, records=True)
    ob = oracle.batch(cfg, n_sims, state=st, seeds=seeds, winners=True, threads=8)
    assert r.winner.tolist() == ob["winners"].tolist()
    assert r.wins.tolist() == ob["wins"].tolist() and (r.ranks == ob["ranks"]).all()
    assert r.competitor_steps == ob["ct"] and r.blocked_steps == ob["blocked"]


def test_run_batch_seeds_derived_on_device():
    """seeds=None: sim i uses derive_seed(master, "run", sim_offset + i), as run_batch (batch.py:117-119)."""
    from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps

    cfg = RaceConfig(300.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0), theta=3.0 * (i % 2))
                                  for i in range(5)))
    r = sim.simulate_batch(None, cfg, 5000, mode="mt", seed_master=20260818, records=True, perms=True)
    ob = oracle.batch(cfg, 5000, master=20260818, winners=True, threads=8)
    assert r.winner.tolist() == ob["winners"].tolist()
    assert (r.ranks == ob["ranks"]).all()
    # a shard starting at sim 1200 reproduces the same per-sim results
    part = sim.simulate_batch(None, cfg, 800, mode="mt", seed_master=20260818, sim_offset=1200, records=True)
    assert part.winner.tolist() == r.winner[1200:2000].tolist()
    for i in (0, 1, 4999):
        o = oracle.run_race(cfg, oracle.derive_seed_run(20260818, i))
        assert r.final_positions[i].tolist() == o.final_positions.tolist()
        assert r.order[i].tolist() == o.order.tolist()


def test_chunked_seeding_over_131072_sims():
    from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps

    cfg = RaceConfig(60.0, tuple(Competitor(f"c{i + 1}", UniformSteps(5.0, 9.0)) for i in range(3)))
    n = 140_000
    r = sim.simulate_batch(None, cfg, n, mode="mt", seed_master=3, records=True)
    for i in (0, 131071, 131072, 139999):
        o = oracle.run_race(cfg, oracle.derive_seed_run(3, i))
        assert r.order[i].tolist() == o.order.tolist() and r.final_positions[i].tolist() == o.final_positions.tolist()
    ob = oracle.batch(cfg, n, master=3, threads=8)
    assert r.wins.tolist() == ob["wins"].tolist()


def test_single_simulate_from_matches_reference_seed():
    from paper_2108_02419_b200.race import simulate_from

    case = next(c for c in race_corpus() if c["simulate_from"]["error"] is None
                and not _has_lognormal(config_from_dict(c["config"])))
    cfg = config_from_dict(case["config"])
    sf = case["simulate_from"]
    order = simulate_from(state_from_dict(sf["state"]), cfg, sf["seed"], mode="mt")
    assert order == tuple(cfg.competitor_ids[c] for c in sf["order"])


def test_device_resident_mt_with_device_seeds():
    """bbe_simulate_async in MT mode with the per-sim seeds already in device memory (the path a
    device-resident caller uses): the device tally equals the host call's for the same seeds."""
    import ctypes

    import torch

    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    seeds = oracle.rp_seeds(77, 3000)
    want = sim.simulate_batch(st, cfg, 3000, mode="mt", seeds=seeds)
    dl = sim.DeviceLauncher(st, cfg)
    d_seeds = torch.from_numpy(seeds.view(np.int64)).cuda()
    tally = torch.zeros(dl.tally_len, dtype=torch.int64, device="cuda")
    req = sim.BbeRequest(3000, 0, 0, sim.MODES["mt"], 0, None, None, d_seeds.data_ptr(), 0, 0)
    stream = torch.cuda.current_stream().cuda_stream
    rc = sim.lib().bbe_simulate_async(ctypes.byref(dl.pk.race), dl.pk.comps, ctypes.byref(dl.st), ctypes.byref(req),
                                      None, ctypes.c_void_p(tally.data_ptr()), ctypes.c_void_p(stream))
    assert rc == 0, sim.last_error()
    t = tally.cpu().numpy().view(np.uint64)
    n = cfg.n_competitors
    assert t[:n].tolist() == want.wins.tolist()
    assert t[n:n + n * n].reshape(n, n).tolist() == want.ranks.tolist()
    assert int(t[dl.off["ct"]]) == want.competitor_steps


@pytest.mark.parametrize("mode", ["mt", "native"])
@pytest.mark.parametrize("d", [1, 3000, 2 * 16384 + 3])
def test_rp_predict_c_entry_equals_python_path(mode, d):
    """rp_predict on a plain random.Random takes the one-call C entry (bbe_rp_predict); a subclass
    takes the Python path (dry_run_seeds + simulate_batch).  Same probabilities, same stream."""
    import random

    class Sub(random.Random):
        pass

    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    a, b = random.Random(77), Sub(77)
    assert rp_predict(st, cfg, d, a, mode=mode) == rp_predict(st, cfg, d, b, mode=mode)
    assert a.getstate() == b.getstate()
