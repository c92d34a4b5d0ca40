"""Parity soak: many random trajectory configurations (the generator of the
GPU parity tests, tests/helpers.py random_configs) through the engine's C ABI,
every row and every completion time compared bit for bit with the C
restatement (and a sample with the compiled reference).  Prints one JSON line.

    python tools/parity_soak.py [--configs 4000] [--ref-sample 400] [--seed 1]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)

import oracle as O  # noqa: E402  (checker)
import paper_2506_19677_b200 as S  # noqa: E402
from helpers import compare_row, orc_config, random_configs, same_float  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, default=4000)
    ap.add_argument("--ref-sample", type=int, default=400)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--batch", type=int, default=500)
    ap.add_argument("--n-choices", default="1,7,50,100,130")
    ap.add_argument("--windows", default="1,2,3,8,8,16")
    a = ap.parse_args()
    orc = O.Oracle("restatement")
    ref = O.Oracle("reference") if O.reference_available() else None
    nch = tuple(int(x) for x in a.n_choices.split(","))
    wins = tuple(int(x) for x in a.windows.split(","))
    cfgs = random_configs(a.configs, seed=a.seed, n_choices=nch, windows=wins)
    bad, decisions, checked_ref, t0 = [], 0, 0, time.time()
    for b0 in range(0, len(cfgs), a.batch):
        chunk = cfgs[b0:b0 + a.batch]
        res = S.run_batch(chunk)
        for k, cfg in enumerate(chunk):
            o = orc.run(orc_config(cfg), records=True)
            errs = compare_row(res.rows[k], o.out)
            for i, rec in enumerate(o.records):
                if not same_float(res.completion_times[k, i], rec.completion_time):
                    errs.append(f"completion[{i}]")
                    break
            decisions += int(res.rows[k]["decisions"])
            if ref is not None and (b0 + k) < a.ref_sample:
                r = ref.run(orc_config(cfg))
                errs += ["ref:" + e for e in compare_row(res.rows[k], r.out, counters=False)]
                checked_ref += 1
            if errs:
                bad.append((b0 + k, errs[:4]))
    print(json.dumps({"trajectories": len(cfgs), "mismatches": len(bad), "first_mismatches": bad[:10],
                      "decisions_compared": decisions, "vs_compiled_reference": checked_ref,
                      "generator": f"tests/helpers.py random_configs(seed={a.seed}): mixes w1-w3, rps 0.5-35, "
                                   f"n in {{{a.n_choices}}}, saber/static, caps 1-100, windows {{{a.windows}}}, "
                                   "ticks 0.003-0.05, prefill 0/500/2000, jitter 0-0.5, usl/linear/logistic models",
                      "seconds": round(time.time() - t0, 1)}))


if __name__ == "__main__":
    main()
