"""GPU parity: the CUDA engine against the CPU checkers, through the C ABI.

Bar: bit-exact rows — identical decision sequences (hash, count,
per-kind counts), completed/met counts, goodput and latency-ratio statistics,
and identical reference-algorithm event counts — for every trajectory.
"""
import math

import numpy as np
import pytest

import oracle as O
from helpers import (CAL_USL, GT, compare_row, orc_config, orc_requests, quantiles_from_records,
                     random_configs, same_float, sim_config)

pytestmark = pytest.mark.gpu


def test_config1_decisions_csv_byte_identical(engine, ref):
    """BASELINE config 1: W1, 4 RPS, SABER-USL, seed 42 (SURVEY §3(B) golden)."""
    cfg = sim_config("w1", 4.0, 100, 42)
    res = engine.run_batch([cfg], records=True, decisions=True, decision_cap=1 << 16)
    r = ref.run(orc_config(cfg), records=True, decisions=True)
    assert compare_row(res.rows[0], r.out, counters=False) == []
    assert int(res.rows[0]["decisions"]) == 17508
    assert list(res.rows[0]["n_kind"]) == [46, 54, 11344, 6010, 54]
    assert float(res.rows[0]["goodput"]) == 0.36
    gpu_csv = O.decisions_to_csv(
        [type("D", (), {k: d[k] for k in d.dtype.names}) for d in res.decisions[0]])
    assert gpu_csv == O.decisions_to_csv(r.decisions)
    # per-request records
    for i, rec in enumerate(r.records):
        assert same_float(res.completion_times[0, i], rec.completion_time)
        assert same_float(res.admit_times[0, i], rec.admit_time)
        assert bool(res.demoted[0, i]) == bool(rec.demoted)
        assert res.arrival_times[0, i] == rec.arrival_time


def test_random_trajectories_match_restatement(engine, orc):
    cfgs = random_configs(300, seed=7)
    res = engine.run_batch(cfgs)
    bad = []
    for k, cfg in enumerate(cfgs):
        o = orc.run(orc_config(cfg), records=True)
        errs = compare_row(res.rows[k], o.out)
        for i, rec in enumerate(o.records):
            if not same_float(res.completion_times[k, i], rec.completion_time):
                errs.append(f"completion[{i}]")
                break
        if errs:
            bad.append((k, errs[:4]))
    assert bad == []


@pytest.mark.parametrize("group", [1, 2, 4, 8, 16, 32])
@pytest.mark.parametrize("streak", [True, False])
def test_every_group_size_and_streak_mode(engine, orc, monkeypatch, group, streak):
    """Every trajectory-kernel configuration (SABER_GROUP lanes per trajectory,
    quiet streaks on/off, DESIGN.md §3.1/§3.5) is bit-exact."""
    monkeypatch.setenv("SABER_GROUP", str(group))
    if streak:
        monkeypatch.delenv("SABER_NO_STREAK", raising=False)
    else:
        monkeypatch.setenv("SABER_NO_STREAK", "1")
    cfgs = random_configs(96, seed=1000 + group)
    res = engine.run_batch(cfgs)
    bad = []
    for k, cfg in enumerate(cfgs):
        o = orc.run(orc_config(cfg), records=True)
        errs = compare_row(res.rows[k], o.out)
        for i, rec in enumerate(o.records):
            if not same_float(res.completion_times[k, i], rec.completion_time):
                errs.append(f"completion[{i}]")
                break
        if errs:
            bad.append((k, errs[:4]))
    assert bad == []


def test_random_trajectories_match_reference(engine, ref):
    cfgs = random_configs(120, seed=99)
    res = engine.run_batch(cfgs)
    bad = []
    for k, cfg in enumerate(cfgs):
        o = ref.run(orc_config(cfg))
        errs = compare_row(res.rows[k], o.out, counters=False)
        if errs:
            bad.append((k, errs[:4]))
    assert bad == []


def test_gate_soundness_runs_match_reference(engine, ref):
    """The acceptance gate-soundness grid (acceptance_main.cpp:84-194):
    54 SABER runs x 400 requests; 12,462 gated admissions + 946,494 rejections."""
    models = [(0, (100.0, 0.05, 0.001)), (1, (90.0, 0.06, 35.0))]
    cfgs = []
    runs = 0
    for mix in ("w1", "w2", "w3"):
        for rps in (2.0, 6.0, 20.0):
            for seed in range(1, 7):
                cfg = sim_config(mix, rps, 400, seed * 977 + 13,
                                 workload_seed=seed * 7919 + runs,
                                 model=models[(runs + seed) % 2])
                cfgs.append(cfg)
                runs += 1
    res = engine.run_batch(cfgs)
    admissions = int(res.rows["n_kind"][:, 0].sum())
    rejections = int(res.rows["n_kind"][:, 2].sum() + res.rows["n_kind"][:, 3].sum())
    assert (admissions, rejections) == (12462, 946494)
    for k, cfg in enumerate(cfgs[:12]):
        o = ref.run(orc_config(cfg))
        assert compare_row(res.rows[k], o.out, counters=False) == []


def test_exact_model_replay_scenarios(engine, orc):
    """acceptance_main.cpp:211-296 scenario class, replayed through
    run_with_requests (custom task names, per-request deadlines)."""
    import random
    import paper_2506_19677_b200 as S
    rng = random.Random(20260816)
    cfgs, reqs = [], []
    for _ in range(60):
        n = 71 + rng.randrange(41)
        rps = rng.uniform(3.0, 3.8)
        rs = []
        out = 200 + rng.randrange(101)
        sla = rng.uniform(1.35, 1.6) * out / 100.0
        rs.append(S.Request(0, "anchor", 0.0, 1 + rng.randrange(256), out, sla, sla))
        t = 0.05
        for i in range(1, n):
            t += -math.log1p(-rng.random()) / rps
            out = 150 + rng.randrange(151)
            sla = rng.uniform(8.0, 12.0) * out / 100.0
            rs.append(S.Request(i, "background", t, 1 + rng.randrange(256), out, sla, t + sla))
        cfg = sim_config("w3", rps, n, rng.randrange(1 << 63), window=1 + rng.randrange(8),
                         model=GT, gt=GT, prefill_rate=0.0, jitter=0.0)
        cfgs.append(cfg)
        reqs.append(rs)
    res = engine.run_batch(cfgs, reqs)
    for k in range(len(cfgs)):
        o = orc.run_with_requests(orc_config(cfgs[k]), orc_requests(reqs[k]))
        assert compare_row(res.rows[k], o.out) == [], k


def test_sweep_rows_and_summary_match_reference(engine, ref):
    import paper_2506_19677_b200 as S
    grid = S.SweepGrid(["w1", "w2", "w3"], [2.0, 10.0, 20.0], [10, 50, 30], True)
    base = sim_config("w3", 1.0, 60, 42)
    base.repeats = 3
    res = engine.sweep(grid, base)
    oc = orc_config(base)
    oc.has_model = 1
    r = ref.sweep(oc, grid.mixes, grid.rps_list, grid.caps, True, base.repeats, jobs=0)
    got = np.array([row.goodput for row in res.rows])
    assert np.array_equal(got, r["goodput"])
    for f in ("ratio_mean", "ratio_std", "cv"):
        a = np.array([getattr(row, f) for row in res.rows])
        assert np.array_equal(a, r[f], equal_nan=True), f
    for k, m in enumerate(grid.mixes):
        s = res.summary[m]
        vals = [s.saber_mean_goodput, s.best_static_mean_goodput, s.delta, s.saber_pooled_cv,
                s.best_static_pooled_cv, s.saber_rps_mean_cv, s.best_static_rps_mean_cv]
        for a, b in zip(vals, r["summary"][k]):
            assert same_float(a, b), (m, vals, list(r["summary"][k]))
        assert [s.best_cap_by_rps[float(x)] for x in grid.rps_list] == list(r["best_cap"][k])


def test_pipelined_plans_match_synchronous(engine):
    """The asynchronous plan API (launch / summarize_launch / wait) on two
    plans and two streams, as bench.py pipelines sweeps, gives exactly the
    synchronous rows and summary; the narrow summary grids included."""
    import torch
    import paper_2506_19677_b200 as S
    grid = S.SweepGrid(["w1", "w3"], [1.0, 4.0, 15.0], [10, 40], True)
    base = sim_config("w1", 1.0, 100, 42)
    base.repeats = 8
    ref_plan = S.SweepPlan(grid, base)
    ref_plan.run()
    ref_plan.summarize()
    rows0, _, summ0, best0 = ref_plan.fetch(summary=True)
    ref_plan.close()

    plans = [S.SweepPlan(grid, base) for _ in range(2)]
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream(priority=-1)
    done = [None, None]
    for k in range(5):
        i = k % 2
        if done[i] is not None:
            main.wait_event(done[i])
        plans[i].launch_sim(main.cuda_stream)
        e = torch.cuda.Event()
        e.record(main)
        side.wait_event(e)
        plans[i].metrics_launch(side.cuda_stream)  # narrow row metrics, as bench.py
        plans[i].summarize_launch(side.cuda_stream)
        d = torch.cuda.Event()
        d.record(side)
        done[i] = d
    torch.cuda.synchronize()
    for pl in plans:
        pl.wait()
        rows, _, summ, best = pl.fetch(summary=True)
        assert rows.tobytes() == rows0.tobytes()
        assert np.array_equal(best, best0)
        for a, b in zip(summ, summ0):
            for f in ("saber_mean_goodput", "best_static_mean_goodput", "delta", "saber_pooled_cv",
                      "best_static_pooled_cv", "saber_rps_mean_cv", "best_static_rps_mean_cv"):
                assert same_float(getattr(a, f), getattr(b, f)), f
        pl.close()


def test_draw_streams_grow_on_exhaustion(engine, monkeypatch):
    """Scheduler draw streams start far below the provable bound and grow
    (rerunning the sweep) when a trajectory exhausts one: a tiny initial cap
    gives exactly the rows of the default one."""
    import paper_2506_19677_b200 as S
    grid = S.SweepGrid(["w1", "w2"], [2.0, 12.0], [20], True)
    base = sim_config("w1", 1.0, 80, 42)
    base.repeats = 4
    a = S.sweep(grid, base)
    monkeypatch.setenv("SABER_DRAW_CAP", "16")
    b = S.sweep(grid, base)
    assert a.traj_rows.tobytes() == b.traj_rows.tobytes()


def test_latency_percentiles_match_restatement(engine, orc):
    cfgs = random_configs(160, seed=4242)
    res = engine.run_batch(cfgs)
    bad = []
    for k, cfg in enumerate(cfgs):
        o = orc.run(orc_config(cfg), records=True)
        want = quantiles_from_records(o.records)
        got = list(res.rows[k]["latency_q"])
        if not all(same_float(a, b) for a, b in zip(got, want)):
            bad.append((k, got, want))
    assert bad == []


def test_latency_percentiles_match_reference_cdf(engine, ref):
    """p50/p90/p99 of every row against the compiled reference's own cdf
    (saber::cdf over all records of saber::run, oracle/ref_harness.cpp)."""
    cfgs = random_configs(120, seed=5151)
    res = engine.run_batch(cfgs)
    bad = []
    for k, cfg in enumerate(cfgs):
        want = ref.latency_quantiles(orc_config(cfg))
        got = list(res.rows[k]["latency_q"])
        if not all(same_float(a, b) for a, b in zip(got, want)):
            bad.append((k, got, want))
    assert bad == []


@pytest.mark.parametrize("n", [200, 512])
def test_large_trajectories_match_restatement(engine, orc, n):
    """n up to the engine's limit (512): 4/8-word tier masks, multi-chunk
    streak sweeps (more slots than 4 per lane), long demotion scans."""
    import random
    rng = random.Random(n)
    cfgs = []
    for i in range(24):
        cfgs.append(sim_config(mix=rng.choice(["w1", "w2", "w3"]), rps=rng.choice([2.0, 8.0, 20.0, 40.0]),
                               n=n, seed=rng.randrange(1 << 40), mode=rng.choice([0, 1]),
                               cap=rng.choice([50, 200, 512]), window=rng.choice([3, 8, 16])))
    res = engine.run_batch(cfgs)
    bad = []
    for k, cfg in enumerate(cfgs):
        o = orc.run(orc_config(cfg), records=True)
        errs = compare_row(res.rows[k], o.out)
        for i, rec in enumerate(o.records):
            if not same_float(res.completion_times[k, i], rec.completion_time):
                errs.append(f"completion[{i}]")
                break
        if errs:
            bad.append((k, errs[:4]))
    assert bad == []


def test_one_shot_sweep_plan_reuse_is_exact(engine):
    """saber_cuda_sweep reuses the previous call's plan for the same grid (new
    inputs staged every call): seeds A, B, A give A's results twice and B's
    equal to a freshly created plan's."""
    import bench
    import paper_2506_19677_b200 as S
    grid = S.SweepGrid(["w1", "w3"], [2.0, 12.0], [20, 60], True)
    base = sim_config("w2", 1.0, 80, 42)
    base.repeats = 4
    a1 = bench._one_shot(S, grid, base, 0, results=True)
    base.seed = 977
    b = bench._one_shot(S, grid, base, 0, results=True)
    base.seed = 42
    a2 = bench._one_shot(S, grid, base, 0, results=True)
    for x, y in zip(a1, a2):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    base.seed = 977
    plan = S.SweepPlan(grid, base)
    plan.run()
    plan.summarize()
    rows, _, summ, best = plan.fetch()
    plan.close()
    st = b[0].reshape(-1, 4)
    for k, f in enumerate(("goodput", "ratio_mean", "ratio_std", "cv")):
        assert np.array_equal(st[:, k], rows[f].astype(np.float64), equal_nan=True), f
    assert np.array_equal(b[2], np.asarray(best))
