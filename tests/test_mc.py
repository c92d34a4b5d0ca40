"""Bursty Monte-Carlo sweep (BASELINE config 5).

CPU: the host twin (saber_cuda_mc_trace) is deterministic, strictly
increasing, bursty (rate between rps and burst_factor*rps, over-dispersed
counts), and its traces replay identically through the C restatement and the
compiled reference.  GPU: every device row equals the oracle's replay of the
host twin's trace; sharded runs add up to the unsharded cell statistics.
"""
import math

import numpy as np
import pytest

import oracle as O
import paper_2506_19677_b200 as S
from helpers import compare_row, orc_config, orc_requests

GRID = S.SweepGrid(["w1", "w2", "w3"], [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 15, 20],
                   list(range(10, 101, 10)), True)
CAL_USL = (0, (99.999999999997357, 0.049999999999992085, 0.0010000000000001078))


def base(n=100, seed=7):
    b = S.SimConfig(model=S.SpeedModel(*CAL_USL), seed=seed)
    b.workload.num_requests = n
    return b


def test_trace_is_deterministic_and_increasing():
    a, ca = S.mc_trace(123, 10_000, GRID, base())
    b, cb = S.mc_trace(123, 10_000, GRID, base())
    assert [r.arrival_time for r in a] == [r.arrival_time for r in b]
    assert ca == cb
    arr = [r.arrival_time for r in a]
    assert all(y > x for x, y in zip(arr, arr[1:]))
    c, _ = S.mc_trace(124, 10_000, GRID, base())
    assert [r.arrival_time for r in c] != arr


def test_trace_cell_and_scheduler_seed_assignment():
    cells = 3 * 12 * 11
    for k in (0, 1, 10, 11, 395, 396, 1000):
        _, cfg = S.mc_trace(k, 2000, GRID, base(seed=50), scheduler_seeds=64)
        cell = k % cells
        v, mr = cell % 11, cell // 11
        assert cfg.workload.rps == float(GRID.rps_list[mr % 12])
        assert cfg.seed == 50 + k % 64
        if v == 10:
            assert cfg.scheduler.mode == S.SchedulerMode.Saber and cfg.model is not None
        else:
            assert cfg.scheduler.mode == S.SchedulerMode.Static
            assert cfg.scheduler.static_batch_size == GRID.caps[v]


def test_arrivals_are_bursty():
    # rps = 4 cells (index 3 in the rps list): k with (k % 396) // 11 % 12 == 3
    ks = [k for k in range(4000) if (k % 396) // 11 % 12 == 3][:120]
    gaps, counts = [], []
    for k in ks:
        reqs, cfg = S.mc_trace(k, 4000, GRID, base(n=200))
        arr = np.array([r.arrival_time for r in reqs])
        gaps.extend(np.diff(arr))
        counts.extend(np.bincount(arr.astype(int))[:int(arr[-1])])
    mean_gap = float(np.mean(gaps))
    assert 1 / (5 * 4.0) < mean_gap < 1 / 4.0  # between the burst and calm rates
    counts = np.array(counts)
    assert counts.var() / counts.mean() > 1.3  # over-dispersed: not Poisson


def test_trace_replays_identically_through_both_oracles(orc, ref):
    for k in (0, 10, 21, 395, 777):
        reqs, cfg = S.mc_trace(k, 1000, GRID, base())
        a = orc.run_with_requests(orc_config(cfg), orc_requests(reqs))
        b = ref.run_with_requests(orc_config(cfg), orc_requests(reqs))
        assert a.out.decision_hash == b.out.decision_hash
        assert a.out.goodput == b.out.goodput


@pytest.mark.gpu
def test_mc_rows_match_oracle_replay(engine, orc):
    n_traj = 4000
    res = engine.mc_sweep(n_traj, GRID, base(), rows=True, scheduler_seeds=256)
    assert int(res.cell_stats[:, 0].sum()) == n_traj
    assert int(res.cell_stats[:, 1].sum()) == n_traj * 100
    assert int(res.cell_hist.sum()) == n_traj * 100
    assert int(res.cell_stats[:, 3].sum()) == int(res.cell_hist[:, :-1].sum())
    rng = np.random.default_rng(1)
    bad = []
    for k in sorted(set(rng.integers(0, n_traj, 150).tolist()) | set(range(0, 396, 11))):
        reqs, cfg = S.mc_trace(k, n_traj, GRID, base(), scheduler_seeds=256)
        o = orc.run_with_requests(orc_config(cfg), orc_requests(reqs))
        errs = compare_row(res.rows[k], o.out)
        if errs:
            bad.append((k, errs[:3]))
    assert bad == []


@pytest.mark.gpu
def test_mc_shards_sum_to_unsharded(engine):
    n_traj = 3000
    full = engine.mc_sweep(n_traj, GRID, base(), scheduler_seeds=128)
    parts = [engine.mc_sweep(n_traj, GRID, base(), scheduler_seeds=128, shard_index=i, shard_count=3,
                             chunk=700) for i in range(3)]
    assert np.array_equal(sum(p.cell_stats for p in parts), full.cell_stats)
    assert np.array_equal(sum(p.cell_hist for p in parts), full.cell_hist)
