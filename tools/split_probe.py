"""Times the config-2 sweep split into its static and SABER halves."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_19677_b200 as S
RPS = [float(r) for r in range(1, 21)]
base = S.SimConfig(model=S.SpeedModel(0, (99.999999999997357, 0.049999999999992085, 0.0010000000000001078)),
                   repeats=64, seed=42)
for name, grid in [("static", S.SweepGrid(["w1", "w2", "w3"], RPS, list(range(10, 101, 10)), False)),
                   ("saber", S.SweepGrid(["w1", "w2", "w3"], RPS, [], True)),
                   ("both", S.SweepGrid(["w1", "w2", "w3"], RPS, list(range(10, 101, 10)), True))]:
    plan = S.SweepPlan(grid, base)
    best = 1e9
    for _ in range(4):
        plan.run(); plan.summarize()
        best = min(best, plan.stats()[1])
    rows, _, _, _ = plan.fetch(summary=False)
    print(f"{name:7s} rows {plan.n_rows:6d} sim_kernel {best:7.2f} ms  ticks {rows['ticks'].sum():.3e} "
          f"decisions {rows['decisions'].sum():.3e}")
    plan.close()
