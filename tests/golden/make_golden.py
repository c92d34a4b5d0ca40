#!/usr/bin/env python3
"""Regenerates tests/golden/golden.json from the UNMODIFIED reference
(oracle/_ref/libsaber_ref.so, built by `make -C oracle` from
/root/reference/proj/core/src).  Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin the restatement oracle and the CUDA engine to the reference's
own outputs on BASELINE config 1, a small config-2 style sweep, the acceptance
gate-soundness grid, and the calibration pipeline.
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402


def row(o):
    return {"goodput": o.goodput, "ratio_mean": o.ratio_mean, "ratio_std": o.ratio_std, "cv": o.cv,
            "completed": o.completed, "met": o.met, "decisions": o.decisions,
            "n_kind": list(o.n_kind), "decision_hash": str(o.decision_hash)}


def main():
    ref = O.Oracle("reference")
    g = {"source": "oracle/_ref/libsaber_ref.so (reference compiled from /root/reference/proj/core/src)"}

    # BASELINE config 1
    cfg = O.make_config(mix="w1", rps=4.0, n=100, seed=42)
    r = ref.run(cfg, records=True, decisions=True)
    csv = O.decisions_to_csv(r.decisions)
    g["config1"] = {
        "row": row(r.out),
        "decisions_csv_sha256": hashlib.sha256(csv.encode()).hexdigest(),
        "decisions_csv_head": csv.splitlines()[:6],
        "completion_times": [x.completion_time for x in r.records],
        "admit_times": [x.admit_time for x in r.records],
        "demoted": [x.demoted for x in r.records],
        "last_arrival": r.out.last_arrival,
    }

    # small sweep (config-2 shape)
    base = O.make_config(mix="w3", n=50, seed=42)
    mixes, rps, caps, reps = ["w1", "w2", "w3"], [2.0, 10.0, 20.0], [10, 50], 2
    s = ref.sweep(base, mixes, rps, caps, True, reps, jobs=0)
    g["sweep"] = {"mixes": mixes, "rps": rps, "caps": caps, "repeats": reps, "n": 50, "seed": 42,
                  "goodput": list(s["goodput"]), "ratio_mean": [None if x != x else x for x in s["ratio_mean"]],
                  "summary": [list(x) for x in s["summary"]], "best_cap": [list(map(int, x)) for x in s["best_cap"]]}

    # per-row decision hashes of the same grid through run()
    hashes = []
    for m in mixes:
        for rr in rps:
            for c in caps + [0]:
                for i in range(reps):
                    c2 = O.make_config(mix=m, rps=rr, n=50, seed=42 + i, mode=O.STATIC if c else O.SABER, cap=c)
                    hashes.append(str(ref.run(c2).out.decision_hash))
    g["sweep"]["decision_hash"] = hashes

    # acceptance gate-soundness grid (acceptance_main.cpp:84-194)
    models = [(O.USL, (100.0, 0.05, 0.001)), (O.LOGISTIC, (90.0, 0.06, 35.0))]
    adm = rej = 0
    runs = 0
    for mix in ("w1", "w2", "w3"):
        for rr in (2.0, 6.0, 20.0):
            for seed in range(1, 7):
                c = O.make_config(mix=mix, rps=rr, n=400, seed=seed * 977 + 13,
                                  workload_seed=seed * 7919 + runs, model=models[(runs + seed) % 2])
                o = ref.run(c).out
                adm += o.n_kind[0]
                rej += o.n_kind[2] + o.n_kind[3]
                runs += 1
    g["gate_soundness"] = {"runs": runs, "admissions": adm, "rejections": rej}

    # calibration pipeline (SURVEY §8(d) models)
    loads, speeds = ref.profile(seed=42)
    cal = ref.calibrate(loads, speeds)
    g["calibration"] = {"profile_seed": 42, "samples": int(len(loads)),
                        "loads_sha256": hashlib.sha256(loads.tobytes()).hexdigest(),
                        "speeds_sha256": hashlib.sha256(speeds.tobytes()).hexdigest(),
                        "best_family": cal["best_family"], "best_params": cal["best_params"],
                        "params": cal["params"], "r2": cal["r2"], "ok": cal["ok"]}

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
