"""Benchmark: batched Monte Carlo race continuation (the BBE dry-run hot path) on B200.

Workload (BASELINE.json configs[1]): derby.json resized to 10 runners
(uniform / preference-sensitive / lognormal / theta=8 blocking / closer), mid-race state
make_rng(3) + initial_state + 65 ticks (tests/golden/c2.json, generated from the reference), and
100,000 continuations per call -- one rp_predict call of one bettor.  A step = one such call.

  value  device-resident: bbe_simulate_async into a device tally on torch's stream, CUDA events,
         max over ranks; N>1 = weak scaling (each rank its own 100k-sim shard, disjoint sim indices)
         plus the NCCL all-reduce of the tally vector inside the step.
  e2e    through the public API agents.rp_predict(state, config, d, rng) with host buffers: agent
         stream advance, parameter H2D, kernel, tally D2H, Laplace probabilities.
  roofline  FP32/INT32 issue roofline of the race kernel: lane-ops per competitor-
         timestep (ct) = 4(n-1) + 13 + 22*f_free; achieved = ct/s * ops/ct; peak = 148 SMs x 128
         lanes x max SM clock.
  cpu_baseline  oracle/pyref.py (the reference's algorithm in the reference's language and RNG),
         single thread, bounded sample.

``--impl reference`` times that same pure-Python restatement with every host core (process pool,
the reference's run_batch fan-out style) on the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

SIMS_PER_CALL = 100_000
METRIC = "simulated races/sec"
UNIT = "races/s"


def load_workload():
    from golden_io import c2, config_from_dict, state_from_dict

    g = c2()
    return config_from_dict(g["config"]), state_from_dict(g["state"])


def ops_per_ct(n: int, f_free: float) -> float:
    return 4 * (n - 1) + 13 + 22 * f_free


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


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


def cpu_baseline_pyref(cfg, state, n_sims: int):
    from oracle import pyref

    seeds = [pyref.derive_seed(20260818, "bench", i) for i in range(n_sims)]
    t0 = time.perf_counter()
    wins, ct = pyref.batch_tally(cfg, seeds, state, workers=1)
    dt = time.perf_counter() - t0
    return {"value": n_sims / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{n_sims} C2 continuations, oracle/pyref.py (reference algorithm, CPython random), 1 thread",
            "ct_per_s": ct / dt, "seconds": dt}


def cpu_baseline_c(cfg, state, n_sims: int):
    import oracle
    from oracle import pyref

    cores = pyref.cpu_count()
    t0 = time.perf_counter()
    out = oracle.batch(cfg, n_sims, state=state, master=20260818, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": n_sims / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{n_sims} C2 continuations, oracle/bbe_oracle.c (C restatement, MT19937), {cores} threads",
            "ct_per_s": out["ct"] / dt, "seconds": dt}


def run_reference(args):
    """--impl reference: the reference algorithm on all host cores (rank 0 only)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import pyref

    cfg, state = load_workload()
    cores = pyref.cpu_count()
    sample = args.ref_sample
    times, cts = [], []
    pool = pyref.TallyPool(cfg, state, workers=cores)
    for i in range(args.warmup + args.steps):
        seeds = [pyref.derive_seed(20260818, "ref", i, j) for j in range(sample)]
        t0 = time.perf_counter()
        wins, ct = pool.run(seeds)
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
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2: derby10 mid-race (tick 65) continuation, rp_predict dry runs",
                   "sims_per_step": sample, "competitors": 10},
        "ct_per_s": sum(cts) / sum(times),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{sample} C2 continuations per step, oracle/pyref.py over a {cores}-process pool"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def sweep_configs(args, torch, sim):
    """The other BASELINE.json configs, device-resident NATIVE launches (one warm-up + one timed each):
    C1 = 5 x U(10,20), L=2000 from the start line (1,000 sims, the reference's CPU case, and 10^6);
    C3 = 20 x U(10,20), L=2000, 10^7 sims; derby20 = derby.json resized to 20, 10^6 sims; C5 = the C3
    field at 10^9 sims in one launch (the per-GPU shard of the scaling config)."""
    from golden_io import c2, config_from_dict
    from paper_2108_02419_b200.batch import resize_race
    from paper_2108_02419_b200.race import Competitor, RaceConfig, UniformSteps

    def uniform_field(n):
        return RaceConfig(2000.0, tuple(Competitor(f"c{i + 1}", UniformSteps(10.0, 20.0)) for i in range(n)))

    derby10 = config_from_dict(c2()["config"])
    derby5 = resize_race(derby10, 5)
    runs = [("C1_5x_U10_20_from_start_1e3", uniform_field(5), 1_000),
            ("C1_5x_U10_20_from_start_1e6", uniform_field(5), 1_000_000),
            ("C3_20x_U10_20_from_start_1e7", uniform_field(20), args.c3_sims),
            ("derby20_from_start_1e6", resize_race(derby5, 20), 1_000_000),
            ("C5_20x_U10_20_from_start_1e9", uniform_field(20), args.c5_sims)]
    out = {}
    stream = torch.cuda.current_stream()
    for name, cfg, n_sims in runs:
        L = sim.DeviceLauncher(None, cfg)
        tally = torch.zeros(L.tally_len, dtype=torch.int64, device="cuda")
        L.launch(tally.data_ptr(), min(n_sims, 100_000), 1, stream=stream.cuda_stream)
        torch.cuda.synchronize()
        tally.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        L.launch(tally.data_ptr(), n_sims, 2, stream=stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        t = tally.cpu()
        ct = int(t[L.off["ct"]])
        blocked = int(t[L.off["blocked"]])
        n = len(cfg.competitors)
        scan = any(c.theta > 0 for c in cfg.competitors)
        # with every theta = 0 no competitor can be blocked (gap > 0 = theta), so the front-runner
        # scan's result is never used: the algorithmic ops drop the 4(n-1) scan term
        ops = ops_per_ct(n, 1.0 - blocked / ct) - (0 if scan else 4 * (n - 1))
        out[name] = {"sims": n_sims, "ms": ms, "races_per_s": n_sims / (ms / 1e3), "ct_per_s": ct / (ms / 1e3),
                     "ct_per_race": ct / n_sims, "ops_per_ct": ops,
                     "issue_roofline_frac": ct * ops / (ms / 1e3) / 37.22e12, "scan_needed": scan}
    # C4: 100 RP bettors, every wake (1 s period, 1 s jitter) predicting with d dry runs on the live
    # race; all wakes that share a race state run as one launch (session dispatch batching).  The
    # host exchange loop (order book, matching) is not part of this path and is not run.
    from paper_2108_02419_b200.session import run_dry_run_session

    for mode, d in (("mt", 1000), ("native", 1000), ("native", 10000)):
        run_dry_run_session(derby5, n_agents=100, d=d, master_seed=20260818, opening_period=5.0, mode=mode)
        r = run_dry_run_session(derby5, n_agents=100, d=d, master_seed=20260818, opening_period=5.0, mode=mode)
        out[f"C4_session_100_rp_bettors_d{d}_{mode}"] = {
            "predictions": len(r.predictions), "launches": r.launches, "sims": r.sims, "seconds": r.seconds,
            "races_per_s_end_to_end": r.sims_per_second, "race_ticks": r.ticks,
            "note": "live race + wake schedule + batched predictions; exchange loop not run"}
    return out


def load_traffic():
    p = os.path.join(ROOT, "profiles", "race_kernel_ncu.json")
    if os.path.exists(p):
        try:
            with open(p) as fh:
                return json.load(fh).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            return None
    return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2108_02419_b200 import sim
    from paper_2108_02419_b200.agents import rp_predict

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, state = load_workload()
    n = cfg.n_competitors
    from paper_2108_02419_b200.parallel import TallyLayout, reduce_tally

    launcher = sim.DeviceLauncher(state, cfg)
    layout = TallyLayout.for_n(n)
    tally = torch.zeros(launcher.tally_len, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2
    stream = torch.cuda.current_stream()
    sims = args.sims
    seed = 20260818

    def step(i):
        tally.zero_()
        launcher.launch(tally.data_ptr(), sims, seed + i, sim_offset=rank * sims, stream=stream.cuda_stream)
        if world > 1:
            reduce_tally(tally, layout)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kernel_ms = []
    ct_total = blocked_total = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        clk.mark_start()
        for i in range(args.steps):
            flush.fill_(float(i))  # L2 flush between timed iterations (outside the event bracket)
            ev[i][0].record(stream)
            step(args.warmup + i)
            ev[i][1].record(stream)
            kernel_ms.append(launcher.last_kernel_ms())
            t = tally.cpu()
            ct_total += int(t[launcher.off["ct"]])
            blocked_total += int(t[launcher.off["blocked"]])
        torch.cuda.synchronize()
        clk.mark_end()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_local = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms = float(t_local.item())
    ms_per_step = total_ms / args.steps
    sims_all = sims * world * args.steps
    value = sims_all / (total_ms / 1e3)
    # ct over all ranks: after the all-reduce the tally holds the job total for that step
    ct_all = ct_total if world > 1 else ct_total
    ct_per_s = ct_all / (total_ms / 1e3)

    # roofline of the race kernel (this rank), from its own CUDA-event kernel durations
    f_free = 1.0 - (blocked_total / ct_total if ct_total else 0.0)
    ops = ops_per_ct(n, f_free)
    k_ms = statistics.mean(kernel_ms)
    ct_launch = ct_total / args.steps / (world if world > 1 else 1)
    achieved = ct_launch * ops / (k_ms / 1e3) / 1e9  # Glane-op/s
    name = torch.cuda.get_device_name(local)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    max_mhz = 1965.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            max_mhz = float(json.load(fh).get("sm_max_mhz", max_mhz))
    except (OSError, ValueError):
        pass
    peak = sms * 128 * max_mhz * 1e6 / 1e9  # Glane-op/s

    line = None
    if rank == 0:
        # e2e through the public API (host buffers; agent stream advance + H2D params + D2H tally)
        import random

        def time_calls(mode, steps):
            agent = random.Random(11)
            ts = []
            for i in range(args.warmup + steps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                probs = rp_predict(state, cfg, sims, agent, mode=mode)
                ts.append(time.perf_counter() - t0)
            assert abs(sum(probs) - 1.0) < 1e-9
            return statistics.mean(ts[args.warmup:])

        e2e_s = time_calls("native", args.steps)
        # one H2D per call: the race-parameter block (64-byte aligned) followed by the zeroed tally
        h2d = ((int(sim.lib().bbe_param_bytes(n)) + 63) // 64) * 64 + launcher.tally_len * 8
        d2h = launcher.tally_len * 8
        # MT mode: the reference's own MT19937 streams, bit-identical results (seeds are H2D inputs)
        mt_steps = max(3, min(args.steps, 20))
        e2e_mt_s = time_calls("mt", mt_steps)
        # device time of one MT batch of the same size (seeding + race kernels, one stream, CUDA events)
        mt_seeds = np.arange(1, sims + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
        mt_kernel_ms = min(sim.simulate_batch(state, cfg, sims, mode="mt", seeds=mt_seeds, ranks=False).kernel_ms
                           for _ in range(3))

        sweep = sweep_configs(args, torch, sim) if args.sweep else None
        cpu = cpu_baseline_pyref(cfg, state, args.cpu_sample) if args.cpu_sample else None
        cpu_c = cpu_baseline_c(cfg, state, args.cpu_c_sample) if args.cpu_c_sample else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C2: derby10 mid-race (tick 65) continuation, one rp_predict call = "
                                   f"{sims} dry runs per GPU", "competitors": n, "sims_per_gpu_per_step": sims,
                       "rng": "philox4x32-10", "l2": "flushed between timed steps (256 MB write)",
                       "parallelism": f"dp{world} (disjoint sim index shards + NCCL tally all-reduce)"},
            "ct_per_s": ct_per_s,
            "roofline": {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "Glane-op/s",
                         "frac": achieved / peak, "traffic": load_traffic(),
                         "ops_per_ct": ops, "f_free": f_free, "kernel_ms": k_ms,
                         "peak_source": f"{sms} SMs x 128 FP32/INT32 lanes x {max_mhz:.0f} MHz (MEASURED_PEAKS.json sm_max_mhz)"},
            "e2e": {"value": sims / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "paper_2108_02419_b200.agents.rp_predict(mode='native')", "ms_per_call": e2e_s * 1e3},
            "mt_exact": {"e2e_value": sims / e2e_mt_s, "unit": UNIT, "ms_per_call": e2e_mt_s * 1e3,
                         "device_ms": mt_kernel_ms, "h2d_bytes_per_step": h2d + 8 * sims, "d2h_bytes_per_step": d2h,
                         "api": "rp_predict(mode='mt'): bit-identical to the reference for the same seeds"},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "cpu_baseline_c": cpu_c,
            "device": name,
            "other_configs": sweep,
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--sims", type=int, default=SIMS_PER_CALL)
    ap.add_argument("--cpu-sample", type=int, default=10000, help="pyref sims for cpu_baseline (0 = skip)")
    ap.add_argument("--cpu-c-sample", type=int, default=200_000, help="C oracle sims (0 = skip)")
    ap.add_argument("--ref-sample", type=int, default=2000, help="sims per --impl reference step")
    ap.add_argument("--sweep", type=int, default=1, help="also time the other BASELINE configs (0 = skip)")
    ap.add_argument("--c3-sims", type=int, default=10_000_000)
    ap.add_argument("--c5-sims", type=int, default=1_000_000_000, help="C5 on this GPU (the per-GPU shard)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup < 3 requested; timing rules want >= 3", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
