"""Cycle split of SABER trajectories on a config-3 style grid (SABER only,
W1-W3 x the 12 ablation rates, one model family), with the instrumented engine
(make BUILD=build_stats LIB=libsaber_b200_stats.so EXTRA_NVFLAGS=-DSABER_STREAK_STATS;
run with SABER_LIB=paper_2506_19677_b200/libsaber_b200_stats.so).

    python tools/saber_sections.py [--seeds 64] [--family usl]

n_kind[0] gate-streak decisions, [1] streak slot sweeps, [2] scheduler step of
normal ticks, [3] normal engine passes, [4] whole trajectory (cycles);
rng_draws = refresh-scan cycles, gate_candidates = refresh scans,
last_arrival = ticks inside streaks, horizon = streaks,
decision_hash = quiet passes << 32 | exact passes."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "benchmarks"))
import ablation_bench as AB  # noqa: E402
import paper_2506_19677_b200 as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=64)
    ap.add_argument("--family", default="usl")
    args = ap.parse_args()
    fam, p = AB.MODELS[args.family]
    grid = S.SweepGrid(AB.MIXES, AB.RPS, [], True)
    base = S.SimConfig(model=S.SpeedModel(fam, p), repeats=args.seeds, seed=42)
    plan = S.SweepPlan(grid, base)
    plan.run()
    plan.run()
    rows, _, _, _ = plan.fetch(summary=False)
    keys = S.sweep_row_keys(grid, base)
    rps = np.array([k[1] for k in keys])
    mix = np.array([k[0] for k in keys])
    nk = rows["n_kind"].astype(np.float64)
    tot = nk[:, 4].sum()
    parts = [nk[:, q].sum() / tot for q in range(4)]
    h = rows["decision_hash"].astype(np.uint64)
    quiet = (h >> np.uint64(32)).astype(np.int64)
    exact = (h & np.uint64(0xFFFFFFFF)).astype(np.int64)
    print(f"saber/{args.family}: {len(rows)} traj, kcyc/traj {tot / len(rows) / 1e3:.0f} "
          f"(max {nk[:, 4].max() / 1e3:.0f})  gate-streak {parts[0]:.3f}  slot-streak {parts[1]:.3f}  "
          f"sched-step {parts[2]:.3f} (refresh scans {rows['rng_draws'].sum() / tot:.3f}, "
          f"{rows['gate_candidates'].mean():.0f}/traj)  engine {parts[3]:.3f}  rest {1 - sum(parts):.3f}")
    T = rows["ticks"].sum()
    print(f"  ticks/traj {T / len(rows):.0f}  streak ticks {rows['last_arrival'].sum() / T:.3f}  "
          f"streaks/traj {rows['horizon'].mean():.0f}  quiet/traj {quiet.mean():.0f}  "
          f"exact/traj {exact.mean():.0f}  decisions/traj {rows['decisions'].mean():.0f}")
    for m in AB.MIXES:
        line = []
        for r in AB.RPS:
            sel = (mix == m) & (rps == r)
            line.append(f"{nk[sel, 4].mean() / 1e3:5.0f}")
        print(f"  {m} kcyc/traj by rps {AB.RPS}: {' '.join(line)}")
    for m in AB.MIXES:
        line = []
        for r in AB.RPS:
            sel = (mix == m) & (rps == r)
            line.append(f"{rows['ticks'][sel].mean():5.0f}/{rows['last_arrival'][sel].sum() / rows['ticks'][sel].sum():.2f}")
        print(f"  {m} ticks/streak-frac by rps: {' '.join(line)}")


if __name__ == "__main__":
    main()
