"""The engine's multi-GPU path (csrc/multi_gpu.cpp) on the one
GPU a test box has: the NCCL code runs with a one-rank communicator.

  * saber_cuda_sweep_multi (one process, a host thread per device,
    ncclCommInitAll) equals the single-device sweep bit for bit;
  * the one-process-per-GPU API (unique id -> saber_cuda_nccl_init ->
    saber_cuda_sweep_plan_gather -> root summary) equals it too;
  * bench.py's N > 1 code (engine NCCL gather, root-only summary, gloo
    plumbing) run under torchrun with SABER_BENCH_NCCL=1.
The sharding itself (disjoint strided shards reduce to the full sweep) is
covered on CPU by tests/test_sharding.py (world size 2, gloo)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _grid(S):
    grid = S.SweepGrid(["w1", "w3"], [2.0, 9.0, 17.0], [10, 40], True)
    base = S.SimConfig()
    base.workload.num_requests = 80
    base.model = S.SpeedModel(0, (99.999999999997357, 0.049999999999992085, 0.0010000000000001078))
    base.repeats = 6
    base.seed = 11
    return grid, base


def _same_result(a, b):
    assert [r.goodput for r in a.rows] == [r.goodput for r in b.rows]
    assert np.array_equal(a.traj_rows["decision_hash"], b.traj_rows["decision_hash"])
    for m in a.summary:
        x, y = a.summary[m], b.summary[m]
        assert np.array_equal(np.array([x.saber_pooled_cv, x.best_static_pooled_cv, x.delta,
                                        x.saber_rps_mean_cv, x.best_static_rps_mean_cv]).view(np.uint64),
                              np.array([y.saber_pooled_cv, y.best_static_pooled_cv, y.delta,
                                        y.saber_rps_mean_cv, y.best_static_rps_mean_cv]).view(np.uint64))
        assert x.best_cap_by_rps == y.best_cap_by_rps


def test_sweep_multi_equals_sweep(engine):
    S = engine
    grid, base = _grid(S)
    _same_result(S.sweep_multi(grid, base, [0]), S.sweep(grid, base))


def test_sweep_multi_rejects_a_repeated_device(engine):
    S = engine
    grid, base = _grid(S)
    with pytest.raises(S.InvalidArgument, match="appears twice"):
        S.sweep_multi(grid, base, [0, 0])


def test_per_process_nccl_gather_equals_sweep(engine):
    S = engine
    grid, base = _grid(S)
    comm = S.NcclComm(S.NcclComm.unique_id(), 1, 0, 0)
    try:
        pl = S.SweepPlan(grid, base, device=0, shard_index=0, shard_count=1)
        pl.run()
        pl.gather(comm, 0)
        pl.summarize()
        rows, _, summ, best = pl.fetch(summary=True)
        got = S.api._sweep_result(grid, base, rows, summ, best, 0.0)
        pl.close()
    finally:
        comm.close()
    _same_result(got, S.sweep(grid, base))


def test_bench_engine_nccl_path():
    env = dict(os.environ, SABER_BENCH_NCCL="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "1",
                        "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["e2e"]["value"] > 0
