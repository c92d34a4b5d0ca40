"""LM fast-path soak: the fit kernel's fast passes (family-specialised,
window-checked unchecked division, clamp-free exponent when provably bounded;
csrc/fit_kernel.cu) against the same kernel with SABER_LM_IEEE=1 (IEEE division
and clamped exponent in every pass), bit for bit: parameters, r^2, status,
selected family, iteration and trial counts.  Prints one JSON line.

    python tools/fit_soak.py [--config4 1000000] [--steep 200000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "benchmarks"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2506_19677_b200 as S  # noqa: E402
import recipes  # noqa: E402
from test_gpu_fit import _steep_logistic_curves  # noqa: E402


def compare(loads, speeds, offsets):
    os.environ.pop("SABER_LM_IEEE", None)
    fast = S.fit_batch(loads, speeds, offsets, calibrate=True)
    os.environ["SABER_LM_IEEE"] = "1"
    slow = S.fit_batch(loads, speeds, offsets, calibrate=True)
    os.environ.pop("SABER_LM_IEEE", None)
    bad = {
        "params": int((fast.params.view(np.uint64) != slow.params.view(np.uint64)).sum()),
        "r2": int((fast.r2.view(np.uint64) != slow.r2.view(np.uint64)).sum()),
        "status": int((fast.status != slow.status).sum()),
        "best_family": int((fast.best_family != slow.best_family).sum()),
        "iterations": int((fast.iterations != slow.iterations).sum()),
        "trials": int((fast.trials != slow.trials).sum()),
    }
    return bad, int(fast.iterations.sum()), fast.device_ms, slow.device_ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config4", type=int, default=1_000_000)
    ap.add_argument("--steep", type=int, default=200_000)
    a = ap.parse_args()
    t0 = time.time()
    out = {"what": "LM fast passes vs SABER_LM_IEEE=1 (IEEE division, clamped exponent), bit for bit",
           "sets": {}}
    for name, data in (("config4", recipes.config4_curves(a.config4)[:3]),
                       ("steep_logistic", _steep_logistic_curves(a.steep))):
        bad, iters, fms, sms = compare(*data)
        out["sets"][name] = {"curves": len(data[2]) - 1, "lm_iterations": iters, "mismatches": bad,
                             "device_ms_fast": fms, "device_ms_ieee": sms}
    out["mismatches_total"] = sum(sum(v["mismatches"].values()) for v in out["sets"].values())
    out["wall_s"] = time.time() - t0
    print(json.dumps(out))
    return 1 if out["mismatches_total"] else 0


if __name__ == "__main__":
    sys.exit(main())
