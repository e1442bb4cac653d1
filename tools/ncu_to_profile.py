"""Turn an ncu --set full report of the race kernel into the committed profile summary.

Usage: python tools/ncu_to_profile.py gpurun_out/prof.ncu-rep profiles/<name> [ct_per_launch]

Writes <name>.json (machine-readable: duration, DRAM bytes per launch, IPC, pipe utilisation, stall
breakdown, warp instructions per competitor-timestep) and <name>.md (the same, readable).
bench.py reads profiles/race_kernel_ncu.json for roofline.traffic.
"""

import csv
import io
import json
import subprocess
import sys


def page(rep, p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    ct = int(sys.argv[3]) if len(sys.argv) > 3 else None
    det = page(rep, "details")
    h = det[0]
    m = {}
    kernel = None
    for r in det[1:]:
        d = dict(zip(h, r))
        kernel = d.get("Kernel Name", kernel)
        m[d["Metric Name"]] = (d["Metric Value"], d.get("Metric Unit", ""))
    raw = page(rep, "raw")
    rd = dict(zip(raw[0], raw[2] if len(raw) > 2 else raw[1]))

    def f(k):
        try:
            return float(str(rd.get(k, "nan")).replace(",", ""))
        except ValueError:
            return None

    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(k) for k in rd
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(v for v in stalls.values() if v) or 1.0
    stalls = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda x: -(x[1] or 0)) if v}
    dram = (f("dram__bytes_read.sum") or 0) + (f("dram__bytes_write.sum") or 0)
    inst = float(m["Executed Instructions"][0].replace(",", ""))
    out = {
        "kernel": kernel,
        "duration_us": float(m["Duration"][0].replace(",", "")) * (1e-3 if m["Duration"][1] == "ns" else 1.0)
        if m["Duration"][1] in ("ns", "us") else float(m["Duration"][0]) * 1e3,
        "dram_bytes_per_launch": dram,
        "executed_warp_instructions": inst,
        "warp_instructions_per_ct": inst / ct if ct else None,
        "ipc_active": float(m["Executed Ipc Active"][0]),
        "issue_slots_busy_pct": float(m["Issue Slots Busy"][0]),
        "achieved_occupancy_pct": float(m["Achieved Occupancy"][0]),
        "theoretical_occupancy_pct": float(m["Theoretical Occupancy"][0]),
        "registers_per_thread": float(m["Registers Per Thread"][0]),
        "avg_active_threads_per_warp": float(m["Avg. Active Threads Per Warp"][0]),
        "grid": m["Grid Size"][0],
        "pipe_pct_of_peak_active": {p: f(f"sm__inst_executed_pipe_{p}.avg.pct_of_peak_sustained_active")
                                    for p in ("alu", "fma", "lsu", "xu", "uniform", "fp64", "cbu", "adu")},
        "stall_fraction": stalls,
        "competitor_timesteps_per_launch": ct,
    }
    with open(dst + ".json", "w") as fh:
        json.dump(out, fh, indent=1)
    lines = [f"# ncu --set full summary: `{kernel}`", "",
             f"- duration: {out['duration_us']:.1f} us; DRAM read+write per launch: {dram:.0f} B",
             f"- executed warp instructions: {inst:.0f}" + (f" ({inst / ct:.2f} per competitor-timestep)" if ct else ""),
             f"- IPC (active): {out['ipc_active']}; issue slots busy: {out['issue_slots_busy_pct']}%",
             f"- occupancy achieved/theoretical: {out['achieved_occupancy_pct']}% / {out['theoretical_occupancy_pct']}%;"
             f" registers/thread: {out['registers_per_thread']:.0f}; active threads/warp: "
             f"{out['avg_active_threads_per_warp']}",
             "- pipe utilisation (% of peak, active cycles): " + ", ".join(
                 f"{k} {v:.1f}" for k, v in out["pipe_pct_of_peak_active"].items() if v),
             "- stall breakdown (share of sampled warp-cycles): " + ", ".join(
                 f"{k} {v * 100:.1f}%" for k, v in list(stalls.items())[:8]), ""]
    with open(dst + ".md", "w") as fh:
        fh.write("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
