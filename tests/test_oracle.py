"""CPU: pin the C restatement (oracle/liboracle.so) against the compiled
reference (oracle/_ref/libsaber_ref.so) and the reference's own known answers.
No GPU needed."""
import math

import numpy as np
import pytest

import oracle as O
from helpers import (CAL_USL, compare_row, orc_config, quantiles_from_records, random_configs,
                     sim_config)


def test_mt19937_64_known_answer(orc):
    lib = orc.lib
    lib.orc_mt19937_64_nth.restype = O.C.c_uint64
    lib.orc_mt19937_64_nth.argtypes = [O.C.c_uint64, O.C.c_int64]
    # C++ [rand.predef]: the 10000th invocation of a default-constructed
    # mt19937_64 (seed 5489) produces 9981545732273789042.
    assert lib.orc_mt19937_64_nth(5489, 10000) == 9981545732273789042


def test_config1_golden(orc, ref):
    """W1, 4 rps, calibrated USL, seed 42."""
    cfg = O.make_config()
    a = orc.run(cfg, records=True, decisions=True)
    b = ref.run(cfg, records=True, decisions=True)
    assert a.out.decisions == b.out.decisions == 17508
    assert list(a.out.n_kind) == list(b.out.n_kind) == [46, 54, 11344, 6010, 54]
    assert a.out.goodput == b.out.goodput == 0.36
    assert a.out.completed == 100
    assert a.out.decision_hash == b.out.decision_hash
    assert O.decisions_to_csv(a.decisions) == O.decisions_to_csv(b.decisions)
    assert abs(a.out.last_arrival - 26.617279) < 1e-6


@pytest.mark.parametrize("seed", [3, 11])
def test_random_trajectories(orc, ref, seed):
    for cfg in random_configs(40, seed=seed):
        oc = orc_config(cfg)
        a = orc.run(oc, records=True)
        b = ref.run(oc, records=True)
        assert a.out.decision_hash == b.out.decision_hash
        assert a.out.decisions == b.out.decisions
        for f in ("goodput", "ratio_mean", "ratio_std", "cv"):
            x, y = getattr(a.out, f), getattr(b.out, f)
            assert (math.isnan(x) and math.isnan(y)) or x == y
        for ra, rb in zip(a.records, b.records):
            assert (math.isnan(ra.completion_time) and math.isnan(rb.completion_time)) or \
                ra.completion_time == rb.completion_time
            assert ra.demoted == rb.demoted


def test_generate_matches(orc, ref):
    for mix in ("w1", "w2", "w3"):
        cfg = O.make_config(mix=mix, rps=7.5, n=200, seed=123456789)
        a = orc.generate(cfg)
        b = ref.generate(cfg)
        for x, y in zip(a, b):
            assert (x.arrival_time, x.deadline, x.input_tokens, x.max_output_tokens, x.task) == \
                (y.arrival_time, y.deadline, y.input_tokens, y.max_output_tokens, y.task)


def test_workload_properties(orc):
    """test_workload.cpp: dense ids / strict increase, jitter band, zero jitter,
    strict increase at rps=1e18."""
    reqs = orc.generate(O.make_config(mix="w3", rps=4.0, n=100, seed=7))
    arr = [r.arrival_time for r in reqs]
    assert all(b > a for a, b in zip(arr, arr[1:]))
    z = orc.generate(O.make_config(mix={O.SUMMARY: 1.0}, rps=4.0, n=50, seed=7, jitter=0.0))
    assert all(r.input_tokens == 31 and r.max_output_tokens == 30 for r in z)
    j = orc.generate(O.make_config(mix="w3", rps=4.0, n=500, seed=8, jitter=0.2))
    avg_out = [43, 387, 30, 617]
    assert all(0.8 * avg_out[r.task] - 0.5 <= r.max_output_tokens <= 1.2 * avg_out[r.task] + 0.5
               for r in j)
    f = orc.generate(O.make_config(mix="w3", rps=1e18, n=50, seed=9))
    arr = [r.arrival_time for r in f]
    assert all(b > a for a, b in zip(arr, arr[1:]))


def test_predict_known_answers(orc):
    """test_estimator.cpp:38-64."""
    assert orc.predict(O.USL, (100, 0, 0), 17) == 100
    assert orc.predict(O.USL, (100, 0.1, 0), 2) == 100 / 1.1
    assert orc.predict(O.USL, (100, 0.05, 0.001), 50) == 100 / 5.9
    assert orc.predict(O.LOGISTIC, (120, 0.1, 30), 30) == 60
    assert orc.predict(O.LINEAR, (-2, 10), 2) == 6
    assert orc.predict(O.LINEAR, (-2, 10), 100) == 1e-6
    assert abs(orc.predict(O.LOGISTIC, (120, 0.1, 30), 1) - 113.74157243058988) < 1e-12
    with pytest.raises(O.OracleError):
        orc.predict(O.USL, (100, 0, 0), 0)


def test_fit_known_answers(orc, ref):
    """test_estimator.cpp:66-118 restated: closed-form linear, constant data,
    noiseless recovery."""
    p, r2, err = orc.fit([1, 2], [10, 8], O.LINEAR)
    assert not err and abs(p[0] + 2) < 1e-12 and abs(p[1] - 12) < 1e-12 and r2 == 1.0
    p, r2, err = orc.fit([1, 2, 3], [42, 42, 42], O.LINEAR)
    assert not err and p[0] == 0 and p[1] == 42 and r2 == 1.0
    loads = np.arange(1, 51)
    for fam, truth, tol in [(O.USL, (100, 0.05, 0.001), 1e-4), (O.LOGISTIC, (120, 0.1, 30), 1e-4),
                            (O.LINEAR, (-0.8, 100.8), 1e-9)]:
        speeds = [orc.predict(fam, truth, int(L)) for L in loads]
        p, r2, err = orc.fit(loads, speeds, fam)
        q, r2b, errb = ref.fit(loads, speeds, fam)
        assert not err and p == q and r2 == r2b
        for k in range(len(truth)):
            assert abs(p[k] - truth[k]) <= tol * max(1, abs(truth[k]))


def test_profile_and_calibrate_match(orc, ref):
    la, sa = orc.profile(seed=42)
    lb, sb = ref.profile(seed=42)
    assert np.array_equal(la, lb) and np.array_equal(sa, sb)
    ca = orc.calibrate(la, sa)
    cb = ref.calibrate(lb, sb)
    assert ca["best_family"] == cb["best_family"] == O.USL
    assert ca["best_params"] == cb["best_params"]
    # the calibrated models used by every BASELINE config
    assert ca["best_params"] == list(CAL_USL[1])
    assert ca["params"][2][:2] == [-1.292318089365694, 72.295958816519274]


def test_sweep_matches_reference(orc, ref):
    base = O.make_config(mix="w3", n=40, seed=42)
    a = orc.sweep(base, ["w1", "w3"], [2.0, 15.0], [10, 30], True, 2)
    b = ref.sweep(base, ["w1", "w3"], [2.0, 15.0], [10, 30], True, 2, jobs=2)
    for k in ("goodput", "ratio_mean", "ratio_std", "cv", "summary"):
        assert np.array_equal(a[k], b[k], equal_nan=True), k
    assert np.array_equal(a["best_cap"], b["best_cap"])


def test_latency_quantiles_match_reference_cdf(orc, ref):
    """The quantile rule the GPU percentile tests apply to the restatement's
    records equals the reference's own cdf (saber::cdf over every record of
    saber::run, metrics.cpp:61-85)."""
    for cfg in random_configs(60, seed=777):
        oc = orc_config(cfg)
        want = ref.latency_quantiles(oc)
        got = quantiles_from_records(orc.run(oc, records=True).records)
        assert all((math.isnan(a) and math.isnan(b)) or a == b for a, b in zip(got, want)), (got, want)
