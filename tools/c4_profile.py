"""cProfile of one C4 dry-run session (100 RP bettors, d = 1000, native): where the host time goes."""
import cProfile, pstats, sys, os
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from golden_io import c2, config_from_dict
from paper_2108_02419_b200.batch import resize_race
from paper_2108_02419_b200.session import run_dry_run_session
derby5 = resize_race(config_from_dict(c2()["config"]), 5)
run_dry_run_session(derby5, n_agents=100, d=1000, master_seed=20260818, opening_period=5.0, mode="native")
pr = cProfile.Profile(); pr.enable()
r = run_dry_run_session(derby5, n_agents=100, d=1000, master_seed=20260818, opening_period=5.0, mode="native")
pr.disable()
print(r.seconds, r.launches)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
