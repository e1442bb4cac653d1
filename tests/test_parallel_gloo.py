"""Multi-rank sharding on CPU: world_size-2 gloo processes run the real sharding and tally-reduction
code of paper_2108_02419_b200.parallel, with each rank's shard tallied by the CPU oracle (the GPU
kernel is exercised by tests/test_gpu_native.py::test_sharding_and_lane_layout_invariance).  The
reduced tallies must equal the single-process tallies exactly -- the worker-count invariance the
reference guarantees for run_batch (tests/test_batch.py:38-42)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_02419_b200.parallel import (
    TallyLayout,
    decode_tally,
    encode_first,
    reduce_tally,
    settle_first_fields,
    shard_range,
)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_tally(cfg, state, lo, hi, master, layout):
    import oracle

    seeds = np.array([oracle.derive_seed_run(master, i) for i in range(lo, hi)], np.uint64)
    out = oracle.batch(cfg, hi - lo, state=state, seeds=seeds) if hi > lo else None
    t = np.zeros(layout.length, np.int64)
    if out is not None:
        n = layout.n
        t[:n] = out["wins"].astype(np.int64)
        t[n:n + n * n] = out["ranks"].reshape(-1).astype(np.int64)
        t[layout.ct] = out["ct"]
        t[layout.ct + 1] = out["blocked"]
    return t


def _worker(rank, world, port, n_sims, master, result_q, fail=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from golden_io import c2, config_from_dict, state_from_dict

    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    layout = TallyLayout.for_n(cfg.n_competitors)
    lo, hi = shard_range(n_sims, rank, world)
    t = torch.from_numpy(_oracle_tally(cfg, st, lo, hi, master, layout))
    # a synthetic failure on rank 1 at its second sim: the reduction must keep the smallest index
    if fail and rank == 1:
        t[layout.ct + 2] += 1
        t[layout.ct + 4] = encode_first(lo + 1)
    if fail and rank == 0 and world > 2:
        t[layout.ct + 2] += 1
        t[layout.ct + 4] = encode_first(hi + 5)
    # count the collectives: the success path must issue exactly one (the SUM)
    calls = []
    orig = dist.all_reduce
    dist.all_reduce = lambda *a, **k: (calls.append(k.get("op")), orig(*a, **k))[1]
    try:
        own = reduce_tally(t, layout)
        settle_first_fields(t, own, layout)
    finally:
        dist.all_reduce = orig
    result_q.put((rank, t.numpy().copy(), len(calls)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_tally_equals_single_process(world):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from golden_io import c2, config_from_dict, state_from_dict

    n_sims, master = 301, 77
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_sims, master, q)) for r in range(world)]
    for p in procs:
        p.start()
    got_q = [q.get(timeout=120) for _ in range(world)]
    results = {r: t for r, t, _ in got_q}
    assert all(c == 2 for _, _, c in got_q)  # a failure: SUM + the MAX of the first-failure fields
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    layout = TallyLayout.for_n(cfg.n_competitors)
    whole = _oracle_tally(cfg, st, 0, n_sims, master, layout)
    for r in range(world):
        got = decode_tally(results[r].view(np.uint64), layout)
        assert got.wins.tolist() == whole[:layout.n].tolist()
        assert (got.ranks.reshape(-1) == whole[layout.n:layout.n * (layout.n + 1)]).all()
        assert got.competitor_steps == whole[layout.ct] and got.blocked_steps == whole[layout.ct + 1]
        assert got.n_diverged == (1 if world == 2 else 2)
        assert got.first_diverged == shard_range(n_sims, 1, world)[0] + 1


def test_success_path_is_one_all_reduce():
    """No failure anywhere: one SUM all-reduce, and the first-failure fields read as 'none'."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from golden_io import c2, config_from_dict, state_from_dict

    world, n_sims, master = 2, 64, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_sims, master, q, False)) for r in range(world)]
    for p in procs:
        p.start()
    got_q = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    layout = TallyLayout.for_n(cfg.n_competitors)
    whole = _oracle_tally(cfg, st, 0, n_sims, master, layout)
    for _, t, calls in got_q:
        assert calls == 1
        got = decode_tally(t.view(np.uint64), layout)
        assert got.wins.tolist() == whole[:layout.n].tolist()
        assert got.n_diverged == 0 and got.first_diverged == -1 and got.first_bad_draws == -1


def test_shard_ranges_partition():
    for n in (0, 1, 7, 100_000, 10**9 + 7):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_first_index_encoding_orders_under_signed_max():
    vals = [encode_first(i) for i in (0, 5, 10**12)]
    assert max(vals) == encode_first(0) and encode_first(-1) == 0
    assert all(0 < v < 2**63 for v in vals)
