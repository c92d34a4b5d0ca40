#!/usr/bin/env python3
"""BASELINE config 4: batched USL/linear/logistic fitting + calibrate selection
over synthetic profiled latency curves (SURVEY §8(d) recipe: truth usl
v1~U[50,150], sigma~U[0,0.2], kappa~U[0,0.005], loads 1..50, 1% noise).

    python benchmarks/fit_bench.py [--curves 1000000] [--cpu-sample 2000]

Prints one JSON line: GPU fits/s (all three families + selection, inputs from
host buffers through saber_cuda_fit_batch), the per-launch device time, and
the reference (oracle/_ref: saber::calibrate per curve) on a bounded sample
with all host threads.
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def curves(n, seed=2026, m=50):
    rng = np.random.default_rng(seed)
    truth = np.stack([rng.uniform(50, 150, n), rng.uniform(0, 0.2, n), rng.uniform(0, 0.005, n)], 1)
    L = np.arange(1, m + 1, dtype=np.float64)
    denom = 1.0 + truth[:, 1:2] * (L - 1.0) + truth[:, 2:3] * L * (L - 1.0)
    speeds = truth[:, 0:1] / denom * (1.0 + 0.01 * (rng.random((n, m)) - 0.5))
    loads = np.tile(np.arange(1, m + 1, dtype=np.int32), n)
    return loads, speeds.reshape(-1), np.arange(0, n * m + 1, m, dtype=np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--curves", type=int, default=1_000_000)
    ap.add_argument("--cpu-sample", type=int, default=2000)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import paper_2506_19677_b200 as S
    loads, speeds, offsets = curves(args.curves)
    S.fit_batch(loads[:50 * 1000], speeds[:50 * 1000], offsets[:1001], calibrate=True)  # warm-up
    walls, devs = [], []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        res = S.fit_batch(loads, speeds, offsets, calibrate=True)
        walls.append(time.perf_counter() - t0)
        devs.append(res.device_ms)
    per_family = {}
    for fam, name in enumerate(["usl", "logistic", "linear"]):
        r = S.fit_batch(loads, speeds, offsets, family_mask=1 << fam)
        per_family[name] = {"fits_per_s_device": args.curves / (r.device_ms / 1e3),
                            "ok": int((r.status[fam] == 0).sum()),
                            "mean_lm_iterations": float(r.iterations[fam].mean())}
    out = {"config": "config4: fit usl+logistic+linear + calibrate over synthetic curves (m=50)",
           "curves": args.curves, "gpu_calibrations_per_s_e2e": args.curves / min(walls),
           "gpu_calibrations_per_s_device": args.curves / (min(devs) / 1e3),
           "device_ms": min(devs), "per_family": per_family,
           "best_family_counts": np.bincount(res.best_family + 2, minlength=5).tolist()}
    import oracle as O
    if O.reference_available() and args.cpu_sample > 0:
        ref = O.Oracle("reference")
        k = args.cpu_sample
        cores = os.cpu_count() or 1

        def one(c):
            lo, hi = offsets[c], offsets[c + 1]
            return ref.calibrate(loads[lo:hi], speeds[lo:hi])["best_family"]

        t0 = time.perf_counter()
        with ThreadPoolExecutor(cores) as ex:
            cpu_best = list(ex.map(one, range(k)))
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": k / dt, "unit": "calibrations/s", "cores": cores,
                               "kind": "reference",
                               "sample": f"saber::calibrate on the first {k} curves, {cores} threads"}
        out["same_best_family_on_sample"] = bool(np.array_equal(np.array(cpu_best), res.best_family[:k]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
