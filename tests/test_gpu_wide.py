"""GPU parity of the wide trajectory kernel: trajectories
with more than 512 requests or an admission window wider than 16, which the
reference accepts (workload.cpp:41-48 and types.cpp:94-100 only require
n >= 1 and window >= 1).  Same bar as tests/test_gpu_parity.py: bit-exact rows,
completion times and decision logs against the compiled reference and the C
restatement."""
import random

import numpy as np
import pytest

import oracle as O
from helpers import compare_row, orc_config, same_float, sim_config

pytestmark = pytest.mark.gpu


def _check(engine, orc, ref, cfgs, n_ref=None):
    res = engine.run_batch(cfgs)
    bad = []
    for k, cfg in enumerate(cfgs):
        o = orc.run(orc_config(cfg), records=True)
        errs = compare_row(res.rows[k], o.out)
        for i, rec in enumerate(o.records):
            if not same_float(res.completion_times[k, i], rec.completion_time):
                errs.append(f"completion[{i}]")
                break
        if ref is not None and (n_ref is None or k < n_ref):
            errs += ["ref: " + e for e in compare_row(res.rows[k], ref.run(orc_config(cfg)).out,
                                                      counters=False)]
        if errs:
            bad.append((k, cfg.workload.num_requests, cfg.scheduler.window_size, errs[:4]))
    return bad


@pytest.mark.parametrize("n", [513, 1000, 2500])
def test_many_requests_match_reference(engine, orc, ref, n):
    """n beyond the register tier masks: SABER and static, every mix."""
    rng = random.Random(n)
    cfgs = [sim_config(mix=rng.choice(["w1", "w2", "w3"]), rps=rng.choice([2.0, 8.0, 20.0, 60.0]),
                       n=n, seed=rng.randrange(1 << 40), mode=rng.choice([0, 0, 1]),
                       cap=rng.choice([20, 100, 600]), window=rng.choice([3, 8, 16]))
            for _ in range(12)]
    assert _check(engine, orc, ref, cfgs, n_ref=6) == []


@pytest.mark.parametrize("window", [17, 32, 33, 64, 1000])
def test_wide_windows_match_reference(engine, orc, ref, window):
    """Windows beyond the nibble Fisher-Yates (64-bit draws, any width); the
    effective window is min(window, |high tier|), scheduler.cpp:61-62."""
    rng = random.Random(window)
    cfgs = [sim_config(mix=rng.choice(["w1", "w2", "w3"]), rps=rng.choice([4.0, 20.0, 40.0]),
                       n=rng.choice([100, 300]), seed=rng.randrange(1 << 40), mode=0,
                       window=window, model=rng.choice([(0, (100.0, 0.05, 0.001)),
                                                        (1, (90.0, 0.06, 35.0))]))
            for _ in range(10)]
    assert _check(engine, orc, ref, cfgs, n_ref=5) == []


def test_wide_decision_log_byte_identical(engine, ref):
    """Trace mode on the wide kernel: the full decisions.csv and the per-request
    admit / completion / demotion records equal the reference's."""
    for cfg in (sim_config("w1", 20.0, 700, 42, window=8), sim_config("w3", 30.0, 200, 7, window=24)):
        res = engine.run_batch([cfg], records=True, decisions=True, decision_cap=1 << 20)
        r = ref.run(orc_config(cfg), records=True, decisions=True)
        assert compare_row(res.rows[0], r.out, counters=False) == []
        gpu_csv = O.decisions_to_csv(
            [type("D", (), {k: d[k] for k in d.dtype.names}) for d in res.decisions[0]])
        assert gpu_csv == O.decisions_to_csv(r.decisions)
        for i, rec in enumerate(r.records):
            assert same_float(res.completion_times[0, i], rec.completion_time)
            assert same_float(res.admit_times[0, i], rec.admit_time)
            assert bool(res.demoted[0, i]) == bool(rec.demoted)


def test_wide_sweep_rows_and_summary_match_reference(engine, ref):
    """A sweep with n = 600 and window 20 runs on the wide kernel end to end
    (plan, streams of raw draws, row metrics with global latency scratch,
    summary) and equals saber::sweep."""
    import paper_2506_19677_b200 as S
    grid = S.SweepGrid(["w1", "w2"], [4.0, 20.0], [50, 300], True)
    base = sim_config("w3", 1.0, 600, 42, window=20)
    base.repeats = 2
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


def test_wide_latency_percentiles(engine, orc):
    """Exact p50/p90/p99 of rows longer than the shared-memory rank buffer."""
    cfgs = [sim_config("w2", 10.0, 900, 5, mode=1, cap=200), sim_config("w1", 3.0, 1200, 9)]
    res = engine.run_batch(cfgs)
    for k, cfg in enumerate(cfgs):
        o = orc.run(orc_config(cfg), records=True)
        lat = sorted((r.completion_time - r.arrival_time) if r.completion_time == r.completion_time
                     else float("inf") for r in o.records)
        n = len(lat)
        for t, p in enumerate((0.5, 0.9, 0.99)):
            j = next(i for i in range(n) if (i + 1) / n >= p)
            want = lat[j] if lat[j] != float("inf") else float("nan")
            assert same_float(float(res.rows[k]["latency_q"][t]), want)


def test_long_wide_trajectory_grows_its_draw_stream(engine, ref):
    """n = 2500 at 20 rps, 3 ms ticks, a 64-wide window: the provable draw bound is
    ~10^8 draws; run_batch starts each stream at 2^18 and grows it x8 when a
    trajectory exhausts it (the batch reruns), ending bit-exact."""
    cfg = sim_config("w2", 20.0, 2500, 11, window=64, tick=0.003)
    res = engine.run_batch([cfg])
    assert int(res.rows[0]["rng_draws"]) > 1 << 18
    assert compare_row(res.rows[0], ref.run(orc_config(cfg)).out, counters=False) == []

