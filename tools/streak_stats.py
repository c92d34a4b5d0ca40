"""Streak coverage on config 2 with the instrumented engine
(make BUILD=build_stats LIB=libsaber_b200_stats.so EXTRA_NVFLAGS=-DSABER_STREAK_STATS;
run with SABER_LIB=paper_2506_19677_b200/libsaber_b200_stats.so).  Rows carry
last_arrival = ticks inside streaks, horizon = streaks, decision_hash =
quiet passes << 32 | exact passes (outside streaks)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2506_19677_b200 as S  # noqa: E402


def main():
    grid = S.SweepGrid(bench.MIXES, bench.RPS, bench.CAPS, True)
    base = S.SimConfig()
    base.workload.num_requests = bench.N_REQ
    base.model = S.SpeedModel(S.ModelFamily.Usl, bench.CAL_USL)
    base.repeats = bench.SEEDS_PER_GPU
    base.seed = bench.BASE_SEED
    p = S.SweepPlan(grid, base)
    p.run()
    rows, _, _, _ = p.fetch(summary=False)
    keys = S.sweep_row_keys(grid, base)
    saber = np.array([k[2] == S.SchedulerMode.Saber for k in keys])
    rps = np.array([k[1] for k in keys])
    h = rows["decision_hash"].astype(np.uint64)
    quiet = (h >> np.uint64(32)).astype(np.int64)
    exact = (h & np.uint64(0xFFFFFFFF)).astype(np.int64)
    for name, m in [("static", ~saber), ("saber", saber)]:
        r = rows[m]
        T = r["ticks"].sum()
        st = r["last_arrival"].sum()
        ns = r["horizon"].sum()
        print(f"{name}: ticks/traj {T / m.sum():.0f}  streak ticks {st / T:.3f}  streaks/traj "
              f"{ns / m.sum():.0f}  mean K {st / max(ns, 1):.1f}  quiet passes/traj "
              f"{quiet[m].sum() / m.sum():.0f}  exact passes/traj {exact[m].sum() / m.sum():.0f}  "
              f"decisions/traj {r['decisions'].sum() / m.sum():.0f}")
        for rv in (1.0, 5.0, 10.0, 20.0):
            mm = m & (rps == rv)
            rr = rows[mm]
            print(f"   rps {rv:4.0f}: ticks {rr['ticks'].mean():7.0f} streak {rr['last_arrival'].sum() / rr['ticks'].sum():.3f}"
                  f" streaks {rr['horizon'].mean():6.0f} quiet {quiet[mm].mean():6.0f} exact {exact[mm].mean():6.0f}")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def durations():
    """Per-trajectory cycles (stats build stores them in n_kind[4])."""
    grid = S.SweepGrid(bench.MIXES, bench.RPS, bench.CAPS, True)
    base = S.SimConfig()
    base.workload.num_requests = bench.N_REQ
    base.model = S.SpeedModel(S.ModelFamily.Usl, bench.CAL_USL)
    base.repeats = bench.SEEDS_PER_GPU
    base.seed = bench.BASE_SEED
    p = S.SweepPlan(grid, base)
    p.run()
    p.run()
    rows, _, _, _ = p.fetch(summary=False)
    keys = S.sweep_row_keys(grid, base)
    cyc = rows["n_kind"][:, 4].astype(np.float64)
    import collections
    agg = collections.defaultdict(list)
    for k, c in zip(keys, cyc):
        agg[(k[0], k[1], "saber" if k[2] == S.SchedulerMode.Saber else "static")].append(c)
    print("total cycles (sum over trajectories) %.3e, max %.3e" % (cyc.sum(), cyc.max()))
    for mode in ("static", "saber"):
        for m in bench.MIXES:
            line = " ".join("%5.0f" % (np.mean(agg[(m, r, mode)]) / 1e3) for r in bench.RPS)
            print(f"{mode:6s} {m} kcyc/traj by rps 1..20: {line}")
    for mode in ("static", "saber"):
        for m in bench.MIXES:
            line = " ".join("%5.0f" % (np.max(agg[(m, r, mode)]) / 1e3) for r in bench.RPS)
            print(f"{mode:6s} {m} max kcyc by rps 1..20: {line}")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "dur":
    durations()


def sections():
    """Cycle split (stats build): n_kind[0] gate-streak decisions, [1] streak
    slot sweeps, [2] scheduler step of normal ticks, [3] normal engine passes,
    [4] whole trajectory."""
    grid = S.SweepGrid(bench.MIXES, bench.RPS, bench.CAPS, True)
    base = S.SimConfig()
    base.workload.num_requests = bench.N_REQ
    base.model = S.SpeedModel(S.ModelFamily.Usl, bench.CAL_USL)
    base.repeats = bench.SEEDS_PER_GPU
    base.seed = bench.BASE_SEED
    p = S.SweepPlan(grid, base)
    p.run()
    p.run()
    rows, _, _, _ = p.fetch(summary=False)
    keys = S.sweep_row_keys(grid, base)
    saber = np.array([k[2] == S.SchedulerMode.Saber for k in keys])
    nk = rows["n_kind"].astype(np.float64)
    for name, m in [("static", ~saber), ("saber", saber)]:
        tot = nk[m, 4].sum()
        parts = [nk[m, q].sum() / tot for q in range(4)]
        print(f"{name}: kcyc/traj {tot / m.sum() / 1e3:.0f}  gate-streak {parts[0]:.3f}  slot-streak {parts[1]:.3f}"
              f"  sched-step {parts[2]:.3f} (refresh scans {rows['rng_draws'][m].sum() / tot:.3f},"
              f" {rows['gate_candidates'][m].mean():.0f}/traj)  engine {parts[3]:.3f}  rest {1 - sum(parts):.3f}")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "sec":
    sections()
