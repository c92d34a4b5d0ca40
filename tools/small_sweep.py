"""A small config-2 style sweep (for compute-sanitizer / debugging)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2506_19677_b200 as S  # noqa: E402

base = S.SimConfig()
base.workload.num_requests = bench.N_REQ
base.model = S.SpeedModel(S.ModelFamily.Usl, bench.CAL_USL)
base.repeats = int(sys.argv[1]) if len(sys.argv) > 1 else 2
base.seed = bench.BASE_SEED
plan = S.SweepPlan(S.SweepGrid(bench.MIXES, bench.RPS, bench.CAPS, True), base)
plan.run()
plan.summarize()
rows, _, summ, _ = plan.fetch()
print("ok", plan.n_rows, float(rows["goodput"].sum()))
