"""Benchmark: batched Monte Carlo race simulation (the BBE dry-run hot path) on B200.

Headline workload (BASELINE.json configs[4] = SURVEY C5, the configuration the metric "races/s per
GPU at 1/2/4/8 B200" is quoted on): a 20-competitor race (20 x U(10,20), L = 2000, theta = 0, the
reference's default field widened to 20, config.py:433-443) simulated from the start line
(run_race semantics: priming draws, race.py:233-241, 373-390), 10^9 simulations per step, split into
contiguous sim-index shards over the N ranks (strong scaling) with ONE NCCL SUM all-reduce of the
tally vector inside the step.  Arithmetic: FP64 race state in the reference's operation order
(NATIVE64 kernel), Philox4x32-10 draws with 53-bit resolution.

  value  device-resident: the prepared race (parameters uploaded once), each step = tally zero +
         race kernel over this rank's shard + tally all-reduce, CUDA events on the launching
         stream, max over ranks; value = 10^9 x steps / max-rank time.
  e2e    the same metric through the public API parallel.simulate_sharded(None, config, 10^9, seed,
         mode="native64") with host buffers: parameter H2D, kernel, all-reduce, tally D2H per step
         (wall clock per call, max over ranks).
  roofline  FP32/INT32 issue roofline of the race kernel, lane-ops per competitor-
         timestep (ct) for the FP64-state kernel = [scan: 4(n-1)] + 13 + 44 f_free (a 53-bit draw =
         two Philox words, 2 x 20 ops, + 4 to form the double); peak = SMs x 128 lanes x max clock.
  cpu_baseline  the reference itself (racemarket from baseline/_ref: run_batch(workers=1), i.e.
         run_race per seed) on a bounded sample of the same workload, one core.

``--impl reference`` times the reference's own parallel path, racemarket ``run_batch`` with
``workers = host cores`` (batch.py:110-124), on a bounded sample of the same workload per step;
rank 0 only.  Without baseline/_ref it falls back to oracle/pyref.py (kind "port").

``--gpus N`` without torchrun's RANK re-launches itself under ``torch.distributed.run`` with N
ranks (127.0.0.1), one GPU per rank.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "simulated races/sec"
UNIT = "races/s"
MASTER = 20260818
C5_SIMS = 1_000_000_000
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC = os.path.join(ROOT, "profiles", "r2_native64_c5_ncu.json")


# ---------------------------------------------------------------------------------------------------
# workloads


def uniform_field(n: int, track_length: float = 2000.0):
    """n x U(10, 20) competitors, theta 0 (config.py:433-443 default field, widened)."""
    from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps

    return RaceConfig(track_length, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(n)))


def c2_workload():
    from golden_io import c2, config_from_dict, state_from_dict

    g = c2()
    return config_from_dict(g["config"]), state_from_dict(g["state"])


def job_config(total_sims: int, world: int) -> dict:
    """The ``config`` of both arms' JSON lines (identical dicts: same workload)."""
    return {"workload": "C5: 20-competitor race (20 x U(10,20), L=2000, theta=0) from the start line, "
                        f"{total_sims} simulations per step split over the ranks",
            "competitors": 20, "track_length": 2000.0, "sims_per_step": int(total_sims), "from_start": True,
            "rng": "philox4x32-10 (53-bit draws)", "state": "f64",
            "l2": "flushed between timed steps (256 MB write); the kernel's working set is on-chip",
            "parallelism": f"dp{world} (contiguous sim-index shards, one NCCL SUM all-reduce of the tally)"}


def ops_per_ct(n: int, f_free: float, *, scan: bool = True, native64: bool = True) -> float:
    """Algorithmic lane-ops per competitor-timestep.  FP32 state: a draw is
    one Philox word (20 ops) + 2; FP64 state: two words + 4.  The scan term drops when every theta is
    0 (nobody can be blocked, the scan's result is never used)."""
    draw = 44.0 if native64 else 22.0
    return (4 * (n - 1) if scan else 0) + 13 + draw * f_free


def issue_peak(sms: int):
    mhz = 1965.0
    try:
        with open(PEAKS) as fh:
            mhz = float(json.load(fh).get("sm_max_mhz", mhz))
    except (OSError, ValueError):
        pass
    return sms * 128 * mhz * 1e6 / 1e9, f"{sms} SMs x 128 FP32/INT32 lanes x {mhz:.0f} MHz (MEASURED_PEAKS.json sm_max_mhz)"


def load_traffic():
    """DRAM bytes per launch of the NATIVE64 C5 kernel from the committed ncu --set full capture."""
    try:
        with open(TRAFFIC) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch"), d.get("source")
    except (OSError, ValueError):
        return None, None


# ---------------------------------------------------------------------------------------------------
# process plumbing


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_command(gpus: int, argv: list[str], port: int) -> list[str]:
    """The torchrun command that re-runs this bench with one rank per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line).

    Sampling starts before the region (nvidia-smi needs ~0.1-0.3 s to start); each sample is
    timestamped on arrival and only samples inside [mark_start(), mark_end()] are summarised.
    """

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 20):
        self.index = index
        self.period_ms = period_ms
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.time() + 3.0
            while not self.rows and time.time() < deadline:  # wait for the first sample
                time.sleep(0.02)
        except OSError:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append((time.time(), parts))

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(2 * self.period_ms / 1000)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        t0 = self.t0 if self.t0 is not None else 0.0
        t1 = (self.t1 if self.t1 is not None else time.time()) + self.period_ms / 1000
        rows = [r for ts, r in self.rows if t0 <= ts <= t1]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        num = lambda v: v.replace(".", "", 1).isdigit()  # noqa: E731
        sm = [float(r[0]) for r in rows if num(r[0])]
        mx = [float(r[1]) for r in rows if num(r[1])]
        pw = [float(r[2]) for r in rows if num(r[2])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------------------------------------------
# the strong-scaling job (device-agnostic: CUDA + NCCL in the bench, CPU + gloo in
# tests/test_bench_harness.py with an oracle-backed launch)


class CudaTimer:
    """CUDA events on the launching stream (torch's current stream)."""

    def __init__(self, torch):
        self.torch = torch
        self.pairs = []

    def start(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def stop(self, e0):
        e1 = self.torch.cuda.Event(enable_timing=True)
        e1.record()
        self.pairs.append((e0, e1))

    def sync(self):
        self.torch.cuda.synchronize()

    def times_ms(self):
        self.sync()
        return [a.elapsed_time(b) for a, b in self.pairs]


class WallTimer:
    """Host wall clock (CPU-only harness test; every launch there is synchronous)."""

    def __init__(self):
        self.ms = []

    def start(self):
        return time.perf_counter()

    def stop(self, t0):
        self.ms.append((time.perf_counter() - t0) * 1e3)

    def sync(self):
        pass

    def times_ms(self):
        return list(self.ms)


def run_strong_job(launch, layout, total_sims: int, steps: int, warmup: int, *, rank: int, world: int, device,
                   timer, seed0: int = MASTER, flush=None, on_start=None, on_end=None, after_step=None):
    """W warm-up + K timed steps of the sharded job.  A step: zero this rank's tally, ``launch(tally,
    n, seed, sim_offset)`` over the rank's contiguous shard of [0, total_sims), then ONE SUM
    all-reduce of the tally (parallel.reduce_tally) when world > 1.  Steps are bracketed by a barrier
    and a device sync on both sides.  Returns (max-over-ranks total ms, per-step local ms, the last
    step's reduced tally as int64 numpy, ct and blocked summed over the timed steps (job totals))."""
    import torch
    import torch.distributed as dist

    from paper_2108_02419_b200.parallel import reduce_tally, settle_first_fields, shard_range

    lo, hi = shard_range(int(total_sims), rank, world)
    tally = torch.zeros(layout.length, dtype=torch.int64, device=device)
    state = {"own": None}

    def step(i):
        tally.zero_()
        launch(tally, hi - lo, seed0 + i, lo)
        state["own"] = reduce_tally(tally, layout) if world > 1 else None

    def read():
        host = tally.cpu()
        if world > 1:
            settle_first_fields(host, state["own"], layout)
        return host.numpy().copy()

    for i in range(warmup):
        step(i)
        read()
    timer.sync()
    if world > 1:
        dist.barrier()
    timer.sync()
    if on_start:
        on_start()
    ct = blocked = 0
    last = None
    for i in range(steps):
        if flush:
            flush(i)  # outside the timed bracket
        t = timer.start()
        step(warmup + i)
        timer.stop(t)
        last = read()
        ct += int(last[layout.ct])
        blocked += int(last[layout.ct + 1])
        if after_step:
            after_step(i, last)
    timer.sync()
    if on_end:
        on_end()
    if world > 1:
        dist.barrier()
    local = timer.times_ms()
    total = torch.tensor([sum(local)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(total, op=dist.ReduceOp.MAX)
    return float(total.item()), local, last, ct, blocked


# ---------------------------------------------------------------------------------------------------
# CPU baselines (the reference itself; the oracle only where the reference is absent)


def reference_module():
    try:
        from paper_2108_02419_b200.session import import_racemarket

        return import_racemarket()
    except ImportError:
        return None


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def reference_batch(rm, cfg, sims: int, master: int, workers: int):
    """racemarket.batch.run_batch over ``sims`` runs of ``cfg`` from the start line; returns (ct, winners)."""
    from paper_2108_02419_b200.session import to_reference_race

    res = rm.batch.run_batch(rm.batch.BatchConfig(to_reference_race(cfg), sims, master, workers=workers))
    return sum(sum(r.finish_ticks) for r in res), [r.winner for r in res]


def cpu_baseline_reference(cfg, sims: int):
    """The reference's own single-thread path (run_batch(workers=1) = run_race per seed) on a sample."""
    rm = reference_module()
    if rm is None:
        from oracle import pyref

        seeds = [pyref.derive_seed(MASTER, "run", i) for i in range(sims)]
        t0 = time.perf_counter()
        _, ct = pyref.batch_tally(cfg, seeds, None, workers=1)
        dt = time.perf_counter() - t0
        kind, what = "port", "oracle/pyref.py (reference algorithm, CPython random; racemarket not installed)"
    else:
        t0 = time.perf_counter()
        ct, _ = reference_batch(rm, cfg, sims, MASTER, 1)
        dt = time.perf_counter() - t0
        kind, what = "reference", "racemarket.batch.run_batch(workers=1) from baseline/_ref"
    return {"value": sims / dt, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{sims} C5 races from the start line, {what}, 1 core", "ct_per_s": ct / dt, "seconds": dt}


def cpu_baseline_c(cfg, sims: int):
    import oracle
    from oracle import pyref

    cores = pyref.cpu_count()
    t0 = time.perf_counter()
    out = oracle.batch(cfg, sims, master=MASTER, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": sims / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{sims} C5 races, oracle/bbe_oracle.c (C restatement, MT19937), {cores} threads",
            "ct_per_s": out["ct"] / dt, "seconds": dt}


def run_reference(args):
    """--impl reference: the reference's run_batch over every host core, rank 0 only."""
    rank, world, _ = dist_env()
    world = max(world, args.gpus)
    if rank != 0:
        return 0
    cfg = uniform_field(20)
    cores = host_cores()
    sample = args.ref_sample or 320 * cores
    rm = reference_module()
    times, cts = [], []
    if rm is not None:
        kind = "reference"
        what = f"racemarket.batch.run_batch(BatchConfig(race, {sample}, seed, workers={cores})) from baseline/_ref"
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            ct, _ = reference_batch(rm, cfg, sample, MASTER + i, cores)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
                cts.append(ct)
    else:
        from oracle import pyref

        kind = "port"
        what = f"oracle/pyref.py over a {cores}-process pool (racemarket not installed)"
        pool = pyref.TallyPool(cfg, None, workers=cores)
        for i in range(args.warmup + args.steps):
            seeds = [pyref.derive_seed(MASTER + i, "run", j) for j in range(sample)]
            t0 = time.perf_counter()
            _, ct = pool.run(seeds)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
                cts.append(ct)
        pool.close()
    t = sum(times) / len(times)
    value = sample / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": job_config(args.c5_sims, world),
        "ct_per_s": sum(cts) / sum(times),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{sample} races of the C5 workload per step (a bounded sample of the "
                                   f"{args.c5_sims} per step), {what}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------------
# secondary configurations (rank 0, N = 1 numbers; not the headline)


def device_launch_ms(torch, sim, state, cfg, n_sims, mode, reps=2):
    """One warm-up + best of ``reps`` device-resident prepared launches; returns (ms, ct, blocked)."""
    L = sim.DeviceLauncher(state, cfg, native_mode=mode)
    tally = torch.zeros(L.tally_len, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    L.launch(tally.data_ptr(), min(n_sims, 200_000), 1, stream=s, mode=mode)
    torch.cuda.synchronize()
    best = None
    for r in range(reps):
        tally.zero_()
        L.launch(tally.data_ptr(), n_sims, 2 + r, stream=s, mode=mode)
        ms = L.last_kernel_ms()
        best = ms if best is None else min(best, ms)
    t = tally.cpu()
    return best, int(t[L.off["ct"]]), int(t[L.off["blocked"]])


def sweep_configs(args, torch, sim):
    """C1, C2 (native64 / native / mt, device and e2e), C3, derby20, the FP32-state C5, and C4 (the
    full session with the reference's exchange loop)."""
    from paper_2108_02419_b200.agents import rp_predict
    from paper_2108_02419_b200.batch import resize_race

    out = {}
    peak, _ = issue_peak(torch.cuda.get_device_properties(0).multi_processor_count)
    derby10, c2_state = c2_workload()
    runs = [("C1_5x_U10_20_from_start_1e6", None, uniform_field(5), 1_000_000),
            ("C2_derby10_mid_race_1e5", c2_state, derby10, 100_000),
            ("C3_20x_U10_20_from_start_1e7", None, uniform_field(20), args.c3_sims),
            ("derby20_from_start_1e6", None, resize_race(resize_race(derby10, 5), 20), 1_000_000)]
    for name, state, cfg, n_sims in runs:
        n = len(cfg.competitors)
        scan = any(c.theta > 0 for c in cfg.competitors)
        row = {"sims": n_sims}
        for mode in ("native64", "native"):
            ms, ct, blk = device_launch_ms(torch, sim, state, cfg, n_sims, mode)
            ops = ops_per_ct(n, 1.0 - blk / ct, scan=scan, native64=mode == "native64")
            row[mode] = {"dtype": "f64" if mode == "native64" else "f32", "ms": ms, "races_per_s": n_sims / (ms / 1e3),
                         "ct_per_s": ct / (ms / 1e3), "ops_per_ct": ops,
                         "issue_roofline_frac": ct * ops / (ms / 1e3) / (peak * 1e9)}
        out[name] = row
    # the C5 field in MT mode: run_batch's own seeds derive_seed(M, "run", i) derived on the device, so
    # the tallies are the reference's run_batch(BatchConfig(race, R, M)) tallies bit for bit
    c5f = uniform_field(20)
    for r in range(2):
        t0 = time.perf_counter()
        res = sim.simulate_batch(None, c5f, 1_000_000, mode="mt", seed_master=MASTER + r)
        wall = time.perf_counter() - t0
    out["C5_field_mt_run_batch_seeds_1e6"] = {
        "dtype": "f64", "device_ms": res.kernel_ms, "races_per_s_device": 1e6 / (res.kernel_ms / 1e3),
        "e2e_ms": wall * 1e3, "races_per_s_e2e": 1e6 / wall, "ct_per_s": res.competitor_steps / (res.kernel_ms / 1e3),
        "note": "simulate_batch(None, race, 1e6, mode='mt', seed_master=M): bit-identical to the reference's run_batch"}
    ms, ct, blk = device_launch_ms(torch, sim, None, uniform_field(20), args.c5_sims, "native", reps=1)
    out["C5_fp32_state_1e9"] = {"dtype": "f32", "ms": ms, "races_per_s": args.c5_sims / (ms / 1e3), "ct_per_s": ct / (ms / 1e3),
                                "issue_roofline_frac": ct * ops_per_ct(20, 1.0, scan=False, native64=False) / (ms / 1e3) / (peak * 1e9)}

    # C2 end to end: one bettor's rp_predict(d = 100k) per call, host buffers
    import random

    def per_call(mode, calls):
        agent = random.Random(11)
        ts = []
        for i in range(3 + calls):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            probs = rp_predict(c2_state, derby10, 100_000, agent, mode=mode)
            ts.append(time.perf_counter() - t0)
        assert abs(sum(probs) - 1.0) < 1e-9
        return statistics.mean(ts[3:])

    c2 = {}
    for mode, calls in (("native64", 20), ("native", 20), ("mt", 10)):
        s = per_call(mode, calls)
        c2[mode] = {"ms_per_call": s * 1e3, "races_per_s": 100_000 / s}
    c2["mt"]["note"] = "bit-identical to the reference's rp_predict for the same bettor stream"
    out["C2_rp_predict_e2e_d1e5"] = c2

    # C4: the full BBE session -- the reference's session loop, exchange and agents (racemarket from
    # baseline/_ref) with every wake round's RP predictions served by one batched launch
    try:
        from paper_2108_02419_b200.session import c4_session_config, run_session_with_stats

        for mode, d in (("mt", 1000), ("mt", 10_000), ("native64", 1000), ("native64", 10_000), ("native64", 100_000)):
            if d > args.c4_max_d:
                continue
            cfg = c4_session_config(derby10, n_agents=100, d=d)
            res, st = run_session_with_stats(cfg, mode=mode)
            out[f"C4_session_100_rp_bettors_d{d}_{mode}"] = {
                "races_per_s_end_to_end": st.sims / st.seconds, "seconds": st.seconds,
                "predict_seconds": st.predict_seconds, "exchange_loop_seconds": st.seconds - st.predict_seconds,
                "sims": st.sims, "predictions": st.predictions, "launches": st.launches, "rounds": st.rounds,
                "look_ahead_hits": st.ahead_hits, "look_ahead_misses": st.ahead_misses,
                "fallbacks": st.fallbacks, "events": len(res.events), "race_ticks": res.trajectory.n_ticks
                if hasattr(res.trajectory, "n_ticks") else None,
                "note": "reference exchange loop (racemarket.session) with batched GPU predictions, the next "
                        "call's first round launched during this call's exchange"
                        + ("; event log equals the reference's" if mode == "mt" else "")}
    except ImportError as e:
        out["C4_session"] = {"unavailable": f"racemarket not importable ({e})"}
    return out


# ---------------------------------------------------------------------------------------------------
# our arm


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2108_02419_b200 import sim
    from paper_2108_02419_b200.parallel import TallyLayout, simulate_sharded

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = uniform_field(20)
    n = cfg.n_competitors
    layout = TallyLayout.for_n(n)
    launcher = sim.DeviceLauncher(None, cfg, native_mode="native64")
    assert launcher.tally_len == layout.length
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2
    kernel_ms = []

    def launch(tally, n_sims, seed, sim_offset):
        launcher.launch(tally.data_ptr(), n_sims, seed, sim_offset=sim_offset, stream=stream.cuda_stream,
                        mode="native64")

    def after_step(i, t):
        kernel_ms.append(launcher.last_kernel_ms())
        if t[layout.ct + 2]:
            raise RuntimeError("a C5 simulation diverged")

    with ClockSampler(local) as clk:
        total_ms, local_ms, last, ct_job, blk_job = run_strong_job(
            launch, layout, args.c5_sims, args.steps, args.warmup, rank=rank, world=world, device="cuda",
            timer=CudaTimer(torch), flush=lambda i: flush_buf.fill_(float(i)), on_start=clk.mark_start,
            on_end=clk.mark_end, after_step=after_step)
    value = args.c5_sims * args.steps / (total_ms / 1e3)
    ct_per_s = ct_job / (total_ms / 1e3)
    assert int(last[:n].sum()) == args.c5_sims, "every simulation has exactly one winner"

    # e2e: the public API with host buffers (parameter H2D, kernel, all-reduce, tally D2H), per call
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    simulate_sharded(None, cfg, args.c5_sims, MASTER + 1000, mode="native64")  # warm-up call
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        tal = simulate_sharded(None, cfg, args.c5_sims, MASTER + 2000 + i, mode="native64")
    e2e_local = time.perf_counter() - t0
    assert int(tal.wins.sum()) == args.c5_sims
    e2e_t = torch.tensor([e2e_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_t.item()) / e2e_steps
    h2d = int(sim.lib().bbe_param_bytes(n))
    d2h = layout.length * 8

    # roofline of this rank's race kernel (its own launches, prepared-launch CUDA events)
    ct_rank_launch = ct_job / args.steps / world
    f_free = 1.0 - (blk_job / ct_job if ct_job else 0.0)
    ops = ops_per_ct(n, f_free, scan=False, native64=True)
    k_ms = statistics.mean(kernel_ms)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    peak, peak_src = issue_peak(sms)
    achieved = ct_rank_launch * ops / (k_ms / 1e3) / 1e9
    traffic, traffic_src = load_traffic()

    line = None
    if rank == 0:
        sweep = sweep_configs(args, torch, sim) if (args.sweep and world == 1) else None
        cpu = cpu_baseline_reference(cfg, args.cpu_sample) if (args.cpu_sample and world == 1) else None
        cpu_c = cpu_baseline_c(cfg, args.cpu_c_sample) if (args.cpu_c_sample and world == 1) else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": job_config(args.c5_sims, world),
            "ct_per_s": ct_per_s, "races_per_s_per_gpu": value / world,
            "roofline": {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "Glane-op/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src or "no committed capture",
                         "ops_per_ct": ops, "f_free": f_free, "kernel_ms": k_ms,
                         "ct_per_launch": ct_rank_launch, "kernel": "native64_kernel<K=2, scan-free>",
                         "peak_source": peak_src},
            "e2e": {"value": args.c5_sims / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "paper_2108_02419_b200.parallel.simulate_sharded(None, config, 1e9, seed, mode='native64')",
                    "ms_per_call": e2e_s * 1e3, "calls": e2e_steps},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "cpu_baseline_c": cpu_c,
            "device": torch.cuda.get_device_name(local),
            "other_configs": sweep,
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--c5-sims", type=int, default=C5_SIMS, help="simulations per step, over all ranks")
    ap.add_argument("--e2e-steps", type=int, default=3, help="public-API calls timed for e2e (each is a full step)")
    ap.add_argument("--cpu-sample", type=int, default=2000, help="reference races for cpu_baseline (0 = skip)")
    ap.add_argument("--cpu-c-sample", type=int, default=100_000, help="C oracle races (0 = skip)")
    ap.add_argument("--ref-sample", type=int, default=0, help="races per --impl reference step (0 = 320 x cores)")
    ap.add_argument("--sweep", type=int, default=1, help="also time the other BASELINE configs (0 = skip)")
    ap.add_argument("--c3-sims", type=int, default=10_000_000)
    ap.add_argument("--c4-max-d", type=int, default=100_000, help="largest C4 session d to run")
    argv = sys.argv[1:] if argv is None else argv
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup < 3 requested; timing rules want >= 3", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "RANK" not in os.environ:
        import torch

        if args.gpus > torch.cuda.device_count():
            print(f"--gpus {args.gpus}: only {torch.cuda.device_count()} GPU(s) visible", file=sys.stderr)
            return 2
        return subprocess.call(spawn_command(args.gpus, argv, free_port()))
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
