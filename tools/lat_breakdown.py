"""Per-call overhead breakdown: simulate_batch vs the raw C call vs the kernel (64 sims, C2)."""
import os, sys, time, ctypes, random
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from golden_io import c2, config_from_dict, state_from_dict
from paper_2108_02419_b200 import sim
g = c2(); cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
for mode in ("native", "mt"):
    seeds = np.arange(1, 65, dtype=np.uint64)
    kw = dict(seeds=seeds) if mode == "mt" else {}
    for _ in range(5): sim.simulate_batch(st, cfg, 64, 7, mode=mode, ranks=False, **kw)
    t0 = time.perf_counter(); R = 200
    ks = []
    for _ in range(R):
        r = sim.simulate_batch(st, cfg, 64, 7, mode=mode, ranks=False, **kw); ks.append(r.kernel_ms)
    t = (time.perf_counter() - t0) / R
    # raw C call with prepared structs
    pk = sim.pack_config(cfg); stc, keep = sim.pack_state(st, pk.n)
    req = sim.BbeRequest(64, 0, 7, sim.MODES[mode], 0, None, None, None, 0)
    if mode == "mt": req.seeds = seeds.ctypes.data
    wins = np.zeros(pk.n, np.uint64)
    res = sim.BbeResult(wins.ctypes.data)
    L = sim.lib()
    t0 = time.perf_counter()
    for _ in range(R):
        L.bbe_simulate(ctypes.byref(pk.race), pk.comps, ctypes.byref(stc), ctypes.byref(req), ctypes.byref(res))
    tc = (time.perf_counter() - t0) / R
    print(f"{mode}: simulate_batch {t*1e6:.1f} us, raw C {tc*1e6:.1f} us, kernel(events) {np.median(ks)*1e3:.1f} us")
