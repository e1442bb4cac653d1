"""bench.py's multi-rank harness on CPU: world-size-2 gloo processes run bench.run_strong_job -- the
same shard / launch / single-SUM-all-reduce / max-over-ranks code the GPU bench runs over NCCL --
with each rank's shard simulated by the C oracle's NATIVE64 stream (oracle.batch_px, bit-exact with
the kernel: tests/test_gpu_native64.py).  The reduced tally of every step must equal the oracle's
tally over the whole sim range, the value must be sims x steps / the max-over-ranks time, and the
reference arm must print the same ``config`` as ours."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _tally_from_oracle(out, layout):
    t = np.zeros(layout.length, np.int64)
    n = layout.n
    t[:n] = out["wins"].astype(np.int64)
    t[n:n + n * n] = out["ranks"].reshape(-1).astype(np.int64)
    t[layout.ct] = out["ct"]
    t[layout.ct + 1] = out["blocked"]
    return t


def _worker(rank, world, port, total, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2108_02419_b200.parallel import TallyLayout

    cfg = bench.uniform_field(6, 300.0)
    layout = TallyLayout.for_n(6)
    calls = []

    def launch(tally, n_sims, seed, sim_offset):
        calls.append((n_sims, seed, sim_offset))
        if n_sims:
            out = oracle.batch_px(cfg, n_sims, seed, sim_offset=sim_offset)
            assert out["rc"] == 0
            tally += torch.from_numpy(_tally_from_oracle(out, layout))

    collectives = []
    orig = dist.all_reduce
    dist.all_reduce = lambda *a, **k: (collectives.append(k.get("op")), orig(*a, **k))[1]
    try:
        total_ms, local, last, ct, blk = bench.run_strong_job(launch, layout, total, steps, 1, rank=rank, world=world,
                                                              device="cpu", timer=bench.WallTimer(), seed0=77)
    finally:
        dist.all_reduce = orig
    q.put((rank, total_ms, local, last, ct, calls, len(collectives)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_strong_job_two_ranks_equals_whole_range(world):
    import oracle
    from paper_2108_02419_b200.parallel import TallyLayout

    total, steps = 3001, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = bench.free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    layout = TallyLayout.for_n(6)
    cfg = bench.uniform_field(6, 300.0)
    whole = _tally_from_oracle(oracle.batch_px(cfg, total, 77 + 1 + steps - 1), layout)
    max_ms = max(sum(r[2]) for r in res)
    for rank, total_ms, local, last, ct, calls, n_coll in res:
        assert np.array_equal(last, whole), "reduced tally == the whole range's tally"
        assert total_ms == pytest.approx(max_ms)  # every rank reports the max over ranks
        # shards: contiguous, disjoint, covering [0, total)
        lo, hi = calls[0][2], calls[0][2] + calls[0][0]
        assert (lo, hi) == (total * rank // world, total * (rank + 1) // world)
        # warm-up + timed steps, each ONE SUM all-reduce; then the MAX of the step time
        assert n_coll == (1 + steps) + 1
    assert sum(r[4] for r in res) == 2 * res[0][4]  # ct: job totals, the same on every rank


def test_spawn_command_uses_torchrun_on_loopback():
    cmd = bench.spawn_command(4, ["--gpus", "4", "--steps", "2"], 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


def test_ops_per_ct():
    # SURVEY 8d values at f_free = 1 (FP32 state): n = 5 -> 51, 10 -> 71, 20 -> 111
    assert [bench.ops_per_ct(n, 1.0, native64=False) for n in (5, 10, 20)] == [51, 71, 111]
    # FP64 state: two Philox words per 53-bit draw; the scan-free C5 field
    assert bench.ops_per_ct(20, 1.0, scan=False, native64=True) == 57


def test_reference_arm_prints_our_config():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--ref-sample", "16"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"] == bench.job_config(bench.C5_SIMS, 1)
    assert line["e2e"]["value"] == line["value"] and line["cpu_baseline"]["cores"] >= 1
    assert line["dtype"] == "f64" and line["scaling"] == "strong"
