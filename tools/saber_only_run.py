"""Runs only the SABER half of config 2 (3,840 trajectories) once — for ncu."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2506_19677_b200 as S  # noqa: E402

base = S.SimConfig()
base.workload.num_requests = bench.N_REQ
base.model = S.SpeedModel(S.ModelFamily.Usl, bench.CAL_USL)
base.repeats = bench.SEEDS_PER_GPU
base.seed = bench.BASE_SEED
plan = S.SweepPlan(S.SweepGrid(bench.MIXES, bench.RPS, [], True), base)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    plan.run()
print("sim ms", plan.stats()[1])
