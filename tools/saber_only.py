import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_19677_b200 as S
RPS = [float(r) for r in range(1, 21)]
base = S.SimConfig(model=S.SpeedModel(0, (99.999999999997357, 0.049999999999992085, 0.0010000000000001078)),
                   repeats=64, seed=42)
plan = S.SweepPlan(S.SweepGrid(["w1", "w2", "w3"], RPS, [], True), base)
for _ in range(2):
    plan.run()
rows, _, _, _ = plan.fetch(summary=False)
import numpy as np
t = rows["ticks"]; order = np.argsort(-t)[:10]
keys = S.sweep_row_keys(S.SweepGrid(["w1", "w2", "w3"], RPS, [], True), base)
for i in order: print(keys[i], int(t[i]), int(rows["decisions"][i]), int(rows["passes"][i]), int(rows["decode_updates"][i]))
