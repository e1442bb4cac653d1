"""The oracle's Philox4x32-10 and NATIVE64 draw source (CPU; the checker of tests/test_gpu_native64.py).

Pinned to an independent implementation: ATen's philox_engine, through the known-answer vectors of
tests/golden/philox.json (tests/golden/make_philox_golden.py), which include the Random123 KAT
(key 0, counter 0 -> 6627e8d5 e169c58d bc57ac4c 9b00dbd8).
"""

import json
import os

import numpy as np

import oracle
from golden_io import GOLDEN, c2, config_from_dict, plain_race, state_from_dict


def test_philox_matches_aten_vectors():
    with open(os.path.join(GOLDEN, "philox.json")) as fh:
        g = json.load(fh)
    assert len(g["vectors"]) >= 64
    for v in g["vectors"]:
        assert oracle.philox4x32_10(v["counter"], v["key"]) == v["out"], v
    assert g["vectors"][0]["out"] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


def test_px_batch_is_deterministic_and_shard_invariant():
    cfg = plain_race({"n": 5, "lo": 10.0, "hi": 20.0, "length": 400.0})
    a = oracle.batch_px(cfg, 300, 77, records=True)
    b = oracle.batch_px(cfg, 300, 77, threads=3, records=True)
    assert (a["order"] == b["order"]).all() and (a["final_positions"] == b["final_positions"]).all()
    lo = oracle.batch_px(cfg, 120, 77, records=True)
    hi = oracle.batch_px(cfg, 180, 77, sim_offset=120, records=True)
    assert (np.concatenate([lo["order"], hi["order"]]) == a["order"]).all()
    assert int(a["wins"].sum()) == 300 and a["ct"] > 0


def test_px_draws_are_the_reference_transforms():
    # a uniform U(v, v) field is RNG-independent: the Philox stream must give the MT race exactly
    cfg = plain_race({"n": 4, "lo": 3.0, "hi": 3.0, "length": 40.0})
    px = oracle.batch_px(cfg, 1, 5, records=True)
    mt = oracle.run_race(cfg, 1)
    assert px["order"][0].tolist() == mt.order.tolist()
    assert px["final_positions"][0].tolist() == mt.final_positions.tolist()
    # derby (lognormal + blocking) from the C2 state: a proper probability vector, ct like the MT oracle's
    g = c2()
    cfg, st = config_from_dict(g["config"]), state_from_dict(g["state"])
    r = oracle.batch_px(cfg, 2000, 11, state=st, threads=4)
    m = oracle.batch(cfg, 2000, state=st, master=11, threads=4)
    assert r["rc"] == 0 and int(r["wins"].sum()) == 2000
    assert abs(r["ct"] / m["ct"] - 1.0) < 0.02
