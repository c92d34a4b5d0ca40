"""Wall-clock breakdown of the one-shot config-2 sweep (plan create / run /
summarize / fetch / destroy) — explains bench.py's e2e number."""
import os
import sys
import time

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
    for it in range(6):
        t = [time.perf_counter()]
        p = S.SweepPlan(grid, base)
        t.append(time.perf_counter())
        p.run()
        t.append(time.perf_counter())
        p.summarize()
        t.append(time.perf_counter())
        p.fetch(completion=False, summary=True)
        t.append(time.perf_counter())
        dev, sim, _ = p.stats()
        p.close()
        t.append(time.perf_counter())
        d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
        print(f"iter {it}: create {d[0]:.1f} run {d[1]:.1f} summ {d[2]:.1f} fetch {d[3]:.1f} "
              f"destroy {d[4]:.1f} ms | device {dev:.1f} sim {sim:.1f} ms", flush=True)
    for it in range(3):
        t0 = time.perf_counter()
        bench._one_shot(S, grid, base, 0)
        print(f"one_shot {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
