"""Timeline of bench.py's pipelined sweeps (CUDA events per stage)."""
import os
import sys

import torch

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
    plans = [S.SweepPlan(grid, base) for _ in range(2)]
    main_s = torch.cuda.current_stream()
    side = torch.cuda.Stream(priority=-1)  # high priority: its blocks go first
    done = [None, None]
    for pl in plans:
        pl.run(main_s.cuda_stream)
        pl.summarize(main_s.cuda_stream)
    torch.cuda.synchronize()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t0 = ev()
    t0.record(main_s)
    marks = []
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    nsteps = int(os.environ.get("PROBE_STEPS", "8"))
    for k in range(nsteps):
        if os.environ.get("PROBE_FLUSH"):
            flush.fill_(k)
        i = k % 2
        if done[i] is not None:
            main_s.wait_event(done[i])
        a = ev(); a.record(main_s)
        plans[i].launch(main_s.cuda_stream)
        b = ev(); b.record(main_s)
        side.wait_event(b)
        c = ev(); c.record(side)
        plans[i].summarize_launch(side.cuda_stream)
        d = ev(); d.record(side)
        done[i] = d
        marks.append((a, b, c, d))
    torch.cuda.synchronize()
    for k, (a, b, c, d) in enumerate(marks):
        print(f"step {k}: run {t0.elapsed_time(a):7.2f} -> {t0.elapsed_time(b):7.2f} ms   "
              f"summary {t0.elapsed_time(c):7.2f} -> {t0.elapsed_time(d):7.2f} ms")
    for pl in plans:
        pl.wait()
        print("sim ms", pl.stats()[1])


if __name__ == "__main__":
    main()
