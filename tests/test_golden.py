"""Golden fixtures produced by the unmodified reference (tests/golden/make_golden.py):
the CPU restatement must reproduce them (CPU test), and so must the CUDA
engine (GPU tests)."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from helpers import same_float, sim_config

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def check_row(row, g):
    assert same_float(float(row["goodput"]), g["goodput"])
    assert same_float(float(row["ratio_mean"]), g["ratio_mean"])
    assert same_float(float(row["ratio_std"]), g["ratio_std"])
    assert same_float(float(row["cv"]), g["cv"])
    assert int(row["completed"]) == g["completed"] and int(row["met"]) == g["met"]
    assert int(row["decisions"]) == g["decisions"]
    assert [int(x) for x in row["n_kind"]] == g["n_kind"]
    assert str(int(row["decision_hash"])) == g["decision_hash"]


def orc_row(o):
    return {"goodput": o.goodput, "ratio_mean": o.ratio_mean, "ratio_std": o.ratio_std, "cv": o.cv,
            "completed": o.completed, "met": o.met, "decisions": o.decisions, "n_kind": list(o.n_kind),
            "decision_hash": o.decision_hash}


def test_restatement_reproduces_config1(orc):
    g = GOLDEN["config1"]
    r = orc.run(O.make_config(), records=True, decisions=True)
    check_row(orc_row(r.out), g["row"])
    csv = O.decisions_to_csv(r.decisions)
    assert hashlib.sha256(csv.encode()).hexdigest() == g["decisions_csv_sha256"]
    assert csv.splitlines()[:6] == g["decisions_csv_head"]
    for rec, c in zip(r.records, g["completion_times"]):
        assert same_float(rec.completion_time, c)


def test_restatement_reproduces_sweep(orc):
    g = GOLDEN["sweep"]
    base = O.make_config(mix="w3", n=g["n"], seed=g["seed"])
    s = orc.sweep(base, g["mixes"], g["rps"], g["caps"], True, g["repeats"])
    assert list(s["goodput"]) == g["goodput"]
    assert [list(x) for x in s["summary"]] == g["summary"] or all(
        same_float(a, b) for x, y in zip(s["summary"], g["summary"]) for a, b in zip(x, y))
    assert [list(map(int, x)) for x in s["best_cap"]] == g["best_cap"]


def test_restatement_reproduces_calibration(orc):
    g = GOLDEN["calibration"]
    loads, speeds = orc.profile(seed=g["profile_seed"])
    assert hashlib.sha256(loads.tobytes()).hexdigest() == g["loads_sha256"]
    assert hashlib.sha256(speeds.tobytes()).hexdigest() == g["speeds_sha256"]
    cal = orc.calibrate(loads, speeds)
    assert cal["best_family"] == g["best_family"] and cal["best_params"] == g["best_params"]


@pytest.mark.gpu
def test_engine_reproduces_config1(engine):
    g = GOLDEN["config1"]
    res = engine.run_batch([sim_config("w1", 4.0, 100, 42)], records=True, decisions=True,
                           decision_cap=1 << 15)
    check_row(res.rows[0], g["row"])
    decs = [type("D", (), {k: d[k] for k in d.dtype.names}) for d in res.decisions[0]]
    csv = O.decisions_to_csv(decs)
    assert hashlib.sha256(csv.encode()).hexdigest() == g["decisions_csv_sha256"]
    for i, c in enumerate(g["completion_times"]):
        assert same_float(res.completion_times[0, i], c)
        assert same_float(res.admit_times[0, i], g["admit_times"][i])
        assert bool(res.demoted[0, i]) == bool(g["demoted"][i])


@pytest.mark.gpu
def test_engine_reproduces_sweep(engine):
    import paper_2506_19677_b200 as S
    g = GOLDEN["sweep"]
    base = sim_config("w3", 1.0, g["n"], g["seed"])
    base.repeats = g["repeats"]
    res = engine.sweep(S.SweepGrid(g["mixes"], g["rps"], g["caps"], True), base)
    assert [r.goodput for r in res.rows] == g["goodput"]
    assert [str(int(h)) for h in res.traj_rows["decision_hash"]] == g["decision_hash"]
    for k, m in enumerate(g["mixes"]):
        s = res.summary[m]
        vals = [s.saber_mean_goodput, s.best_static_mean_goodput, s.delta, s.saber_pooled_cv,
                s.best_static_pooled_cv, s.saber_rps_mean_cv, s.best_static_rps_mean_cv]
        assert all(same_float(a, b) for a, b in zip(vals, g["summary"][k]))


@pytest.mark.gpu
def test_engine_reproduces_gate_soundness_counts(engine):
    g = GOLDEN["gate_soundness"]
    models = [(0, (100.0, 0.05, 0.001)), (1, (90.0, 0.06, 35.0))]
    cfgs, runs = [], 0
    for mix in ("w1", "w2", "w3"):
        for rps in (2.0, 6.0, 20.0):
            for seed in range(1, 7):
                cfgs.append(sim_config(mix, rps, 400, seed * 977 + 13, workload_seed=seed * 7919 + runs,
                                       model=models[(runs + seed) % 2]))
                runs += 1
    res = engine.run_batch(cfgs)
    assert int(res.rows["n_kind"][:, 0].sum()) == g["admissions"]
    assert int(res.rows["n_kind"][:, 2].sum() + res.rows["n_kind"][:, 3].sum()) == g["rejections"]
