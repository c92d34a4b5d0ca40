"""Why streaks end (instrumented engine, see tools/streak_stats.py for the
build): per trajectory, streaks bound by the engine (Kb: next prefill end /
completion), the next arrival, a demotion scan or the draw stream, the
horizon/other; the same for failed attempts (K < 2); and ticks whose streak
condition is false (sblock / idle engine / gate admitted / other)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2506_19677_b200 as S  # noqa: E402


def unpack(v):
    v = v.astype(np.int64)
    return np.stack([(v >> (16 * q)) & 0xFFFF for q in range(4)], 1)


def report(name, rows, mask):
    r = rows[mask]
    k2 = unpack(r["refresh_entries"]).sum(0) / mask.sum()
    k1 = unpack(r["ledger_scanned"]).sum(0) / mask.sum()
    nc = unpack(r["prefill_updates"]).sum(0) / mask.sum()
    print(f"{name}: ticks/traj {r['ticks'].mean():.0f}")
    print("   streaks (K>=2) ended by  Kb %.1f  arrival %.1f  demote/draws %.1f  other %.1f" % tuple(k2))
    print("   attempts K<2 bound by    Kb %.1f  arrival %.1f  demote/draws %.1f  other %.1f" % tuple(k1))
    print("   no attempt: sblock %.1f  A==0 %.1f  gate admitted %.1f  other %.1f" % tuple(nc))


def main():
    grid = S.SweepGrid(bench.MIXES, bench.RPS, bench.CAPS, True)
    base = S.SimConfig()
    base.workload.num_requests = bench.N_REQ
    base.model = S.SpeedModel(S.ModelFamily.Usl, bench.CAL_USL)
    base.repeats = 16
    base.seed = bench.BASE_SEED
    p = S.SweepPlan(grid, base)
    p.run()
    rows, _, _, _ = p.fetch(summary=False)
    keys = S.sweep_row_keys(grid, base)
    saber = np.array([k[2] == S.SchedulerMode.Saber for k in keys])
    report("config2 static", rows, ~saber)
    report("config2 saber", rows, saber)
    rps = np.array([k[1] for k in keys])
    for rv in (2.0, 10.0, 20.0):
        report(f"   saber rps {rv}", rows, saber & (rps == rv))


if __name__ == "__main__":
    main()
