"""GPU command line for the simulation products (mirrors `racemarket race|batch|bench|compare`,
cli.py:33-52, for race configs):

    python -m paper_2108_02419_b200 race    --config derby.json --out out/ [--seed S]
    python -m paper_2108_02419_b200 batch   --config derby.json --out out/ [--replications R] [--mode mt|native]
    python -m paper_2108_02419_b200 bench   --config derby.json --out out/
    python -m paper_2108_02419_b200 compare pmf_a.csv pmf_b.csv

Exit codes follow the reference: 0 ok, 1 simulation failure, 2 usage/config error.  One JSON line
per command on stdout.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

from . import batch as B
from . import products as P
from .race import RaceConfigError, RaceDivergedError
from .seeding import derive_seed
from .sim import run_race, simulate_batch


def _emit(obj) -> None:
    print(json.dumps(obj, separators=(",", ":")), flush=True)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2108_02419_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("race", "batch", "bench"):
        p = sub.add_parser(name)
        p.add_argument("--config", required=True)
        p.add_argument("--out", required=True)
        p.add_argument("--seed", type=int)
        p.add_argument("--mode", choices=["mt", "native"], default="mt")
        if name == "batch":
            p.add_argument("--replications", type=int)
    c = sub.add_parser("compare")
    c.add_argument("pmf_a")
    c.add_argument("pmf_b")
    args = ap.parse_args(argv)
    try:
        if args.cmd == "compare":
            r = B.compare_pmf(P.read_pmf_csv(args.pmf_a), P.read_pmf_csv(args.pmf_b))
            _emit({"command": "compare", "method": r.method, "statistic": r.statistic, "p_value": r.p_value,
                   "dof": r.dof})
            return 0
        doc, cfg, seed = P.load_experiment(args.config)
        if args.seed is not None:
            seed = args.seed
        out = Path(args.out)
        out.mkdir(parents=True, exist_ok=True)
        if args.cmd == "race":
            traj = run_race(cfg, derive_seed(seed, "race"), record=True, mode="mt")
            P.write_trajectory_csv(out / "trajectory.csv", traj)
            P.write_finish_csv(out / "finish.csv", traj)
            _emit({"command": "race", "winner": traj.winner, "n_ticks": traj.n_ticks, "out": str(out)})
        elif args.cmd == "batch":
            reps = args.replications or int(doc.get("batch", {}).get("replications", 1000))
            if args.mode == "mt":
                results = B.run_batch(B.BatchConfig(cfg, reps, seed))
                pmf = B.pmf_from_results(results)
                P.write_race_runs_csv(out / "runs.csv", results)
            else:
                res = simulate_batch(None, cfg, reps, seed, mode="native", perms=True)
                pmf = B.pmf_from_tally(res)
            P.write_pmf_csv(out / "pmf.csv", pmf)
            _emit({"command": "batch", "replications": reps, "distinct_outcomes": len(pmf.counts), "out": str(out)})
        else:
            bc = doc.get("bench", {})
            points = B.bench(cfg, tuple(bc.get("n_competitors", (5, 10, 20, 40))), int(bc.get("replications", 100)),
                             int(bc.get("timing_reps", 5)), seed, mode="native")
            P.write_bench_csv(out / "bench.csv", points)
            _emit({"command": "bench", "points": [[p.n_competitors, p.mean_s, p.cv] for p in points], "out": str(out)})
        return 0
    except (RaceConfigError, ValueError, OSError) as exc:
        _emit({"error": str(exc)})
        return 2
    except (RaceDivergedError, B.BatchRunError, RuntimeError) as exc:
        _emit({"error": str(exc)})
        return 1


if __name__ == "__main__":
    sys.exit(main())
