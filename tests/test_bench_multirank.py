"""bench.py's N > 1 path (sharded sweep, all-reduce gather on the side
stream, pipelined summaries, max-over-ranks timing) run as two ranks on one
GPU with gloo (SABER_BENCH_DEVICE / SABER_BENCH_BACKEND test hooks): its
summary must equal a single-process sweep over the same 128 seeds."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_two_rank_bench_equals_one_sweep(engine):
    env = dict(os.environ, SABER_BENCH_DEVICE="0", SABER_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["trajectories_per_step"] == 2 * 42240
    sys.path.insert(0, ROOT)
    import bench
    S = engine
    grid = S.SweepGrid(bench.MIXES, bench.RPS, bench.CAPS, True)
    base = S.SimConfig()
    base.workload.num_requests = bench.N_REQ
    base.model = S.SpeedModel(S.ModelFamily.Usl, bench.CAL_USL)
    base.repeats = 2 * bench.SEEDS_PER_GPU
    base.seed = bench.BASE_SEED
    res = S.sweep(grid, base)
    for m in bench.MIXES:
        s = res.summary[m]
        got = line["summary"][m]
        assert got["delta"] == s.delta
        assert got["saber_mean_goodput"] == s.saber_mean_goodput
        assert got["best_static_mean_goodput"] == s.best_static_mean_goodput
