"""The reference's release gate (proj/tests/acceptance_main.cpp) reproduced on
the engine, pinned to the numbers the reference prints (proj/test_output.txt:
23-31) AND to the compiled reference run live (oracle/_ref):

  * exact-model guarantee (acceptance_main.cpp:195-296): 200 replayed
    scenarios from mt19937_64(20260816) -> 18,166 gated admissions, 0 misses,
    35,852 rejections, 0 demotions;
  * the shared grid pipeline (:494-533): profile(seed 20260816) -> calibrate
    -> sweep w1-w3 x default_rps_sweep x caps 10..100 + SABER, repeats 3 ->
    deltas w1 +7.36 / w2 -4.36 / w3 +4.19 pp (:535-550), pooled latency-ratio
    CV 1.068 vs 1.675 (:552-559), best caps w1 10..30, w2 10..40, w3 10..40
    (:561-578);
  * the USL-vs-linear ablation (:586-639): w2@20 rps linear 0.5133 vs usl
    0.4867.

Every engine value is compared bit for bit with the reference's."""
import math

import numpy as np
import pytest

import oracle as O
import paper_2506_19677_b200 as S

pytestmark = pytest.mark.gpu


class MT19937_64:
    """std::mt19937_64 (C++ [rand.eng.mers], default seeding) — the
    acceptance scenario generator's engine."""
    N, M = 312, 156
    MASK = (1 << 64) - 1

    def __init__(self, seed):
        self.mt = [0] * self.N
        self.mt[0] = seed & self.MASK
        for i in range(1, self.N):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & self.MASK
        self.i = self.N

    def _twist(self):
        mt, N, M = self.mt, self.N, self.M
        for k in range(N):
            y = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % N] & 0x7FFFFFFF)
            v = mt[(k + M) % N] ^ (y >> 1)
            if y & 1:
                v ^= 0xB5026F5AA96619E9
            mt[k] = v
        self.i = 0

    def __call__(self):
        if self.i >= self.N:
            self._twist()
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self.MASK


def test_mt19937_64_known_answer():
    """The C++ standard's check value: the 10000th output of a default-seeded
    (5489) mt19937_64 is 9981545732273789042."""
    g = MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


def _u01(rng):
    return float(rng() >> 11) * 2.0 ** -53


def _uniform(rng, lo, hi):
    return lo + (hi - lo) * _u01(rng)


USL_TRUTH = S.SpeedModel(S.ModelFamily.Usl, (100.0, 0.05, 0.001))


def exact_model_scenarios():
    """acceptance_main.cpp:211-258, draw for draw."""
    rng = MT19937_64(20260816)
    out = []
    for _ in range(200):
        n = 71 + rng() % 41
        rps = _uniform(rng, 3.0, 3.8)
        reqs = []
        a_in = 1 + rng() % 256
        a_out = 200 + rng() % 101
        a_sla = _uniform(rng, 1.35, 1.6) * a_out / 100.0
        reqs.append(S.Request(0, "anchor", 0.0, a_in, a_out, a_sla, a_sla))
        t = 0.05
        for i in range(1, n):
            t += -math.log1p(-_u01(rng)) / rps
            r_in = 1 + rng() % 256
            r_out = 150 + rng() % 151
            sla = _uniform(rng, 8.0, 12.0) * r_out / 100.0
            reqs.append(S.Request(i, "background", t, r_in, r_out, sla, t + sla))
        cfg = S.SimConfig()
        cfg.workload = S.WorkloadSpec(S.preset_mix("w3"), rps, n, 0, 0.0)
        cfg.scheduler = S.SchedulerConfig(S.SchedulerMode.Saber, 1 + rng() % 8, 0.01, 0)
        cfg.model = USL_TRUTH
        cfg.engine = S.EngineConfig(USL_TRUTH, 0.0)
        cfg.seed = rng()
        out.append((cfg, reqs))
    return out


def test_exact_model_guarantee_counts():
    """18,166 gated admissions, 0 misses, 35,852 rejections, 0 demotions
    (proj/test_output.txt:24) — one batched launch of 200 replays."""
    scen = exact_model_scenarios()
    res = S.run_batch([c for c, _ in scen], [r for _, r in scen], records=True)
    kinds = res.rows["n_kind"]
    rejections = int(kinds[:, 2].sum() + kinds[:, 3].sum())
    demotions, low_admits = int(kinds[:, 4].sum()), int(kinds[:, 1].sum())
    admitted = violations = 0
    for k, (_, reqs) in enumerate(scen):
        st = res.states[k, : len(reqs)]
        gated = ~np.isnan(st["admit_time"]) & (st["demoted"] == 0)
        admitted += int(gated.sum())
        violations += int((gated & (st["met_sla"] == 0)).sum())
    assert (admitted, violations, rejections, demotions, low_admits) == (18166, 0, 35852, 0, 0)


@pytest.fixture(scope="module")
def ref():
    if not O.reference_available():
        pytest.skip("oracle/_ref not built")
    return O.Oracle("reference")


@pytest.fixture(scope="module")
def grid():
    """The shared pipeline on the engine (acceptance_main.cpp:504-533)."""
    samples = S.profile(S.EngineConfig(), S.WorkloadSpec(S.preset_mix("w3"), 1.0, 1000, 20260816, 0.2),
                        50)
    report = S.calibrate(samples)
    base = S.SimConfig()
    base.workload = S.WorkloadSpec(S.preset_mix("w3"), 1.0, 100, 0, 0.2)
    base.model = report.best
    base.repeats = 3
    base.seed = 42
    g = S.SweepGrid(["w1", "w2", "w3"], S.default_rps_sweep(), list(range(10, 101, 10)), True)
    return samples, report, base, S.sweep(g, base)


def test_grid_pipeline_matches_reference_and_published_numbers(grid, ref):
    samples, report, base, res = grid
    assert report.best.family == S.ModelFamily.Usl
    # the reference's own pipeline, run live
    loads = np.array([s.load for s in samples], np.int32)
    speeds = np.array([s.speed for s in samples])
    rl, rs = ref.profile(seed=20260816)
    assert np.array_equal(rl, loads) and np.array_equal(rs, speeds)
    cal = ref.calibrate(rl, rs)
    assert cal["best_family"] == 0 and list(cal["best_params"]) == list(report.best.params)
    rb = O.make_config(mix="w3", rps=1.0, n=100, seed=42, model=(0, report.best.params))
    want = ref.sweep(rb, ["w1", "w2", "w3"], S.default_rps_sweep(), list(range(10, 101, 10)), True, 3)
    assert [r.goodput for r in res.rows] == [float(g) for g in want["goodput"]]
    for k, mix in enumerate(["w1", "w2", "w3"]):
        s = res.summary[mix]
        got = [s.saber_mean_goodput, s.best_static_mean_goodput, s.delta, s.saber_pooled_cv,
               s.best_static_pooled_cv, s.saber_rps_mean_cv, s.best_static_rps_mean_cv]
        assert got == list(want["summary"][k]), mix
    # the release-gate lines (proj/test_output.txt:28-30)
    deltas = {m: f"{res.summary[m].delta * 100.0:+.3g}" for m in ("w1", "w2", "w3")}
    assert deltas == {"w1": "+7.36", "w2": "-4.36", "w3": "+4.19"}
    w1 = res.summary["w1"]
    assert (f"{w1.saber_pooled_cv:.4g}", f"{w1.best_static_pooled_cv:.4g}") == ("1.068", "1.675")
    ranges = {m: (min(res.summary[m].best_cap_by_rps.values()), max(res.summary[m].best_cap_by_rps.values()))
              for m in ("w1", "w2", "w3")}
    assert ranges == {"w1": (10, 30), "w2": (10, 40), "w3": (10, 40)}


def test_estimator_ablation(grid, ref):
    """acceptance_main.cpp:586-639: usl vs linear fits of the same samples,
    adaptive cells only; cell means as the reference sums them."""
    samples, _, base, _ = grid
    usl = S.fit(samples, S.ModelFamily.Usl)
    lin = S.fit(samples, S.ModelFamily.Linear)
    loads = np.array([s.load for s in samples], np.int32)
    speeds = np.array([s.speed for s in samples])
    for f, m in ((O.USL, usl), (O.LINEAR, lin)):
        p, r2, err = ref.fit(loads, speeds, f)
        assert not err and p[: len(m.params)] == list(m.params)[: len(p)] and r2 == m.fit_r2
    g = S.SweepGrid(["w1", "w2", "w3"], S.default_rps_sweep(), [], True)

    def cell_means(model):
        cfg = S.SimConfig(base.workload, base.scheduler, model, base.engine, None, 3, 42)
        r = S.sweep(g, cfg)
        acc = {}
        for row in r.rows:
            s, c = acc.get((row.mix, row.rps), (0.0, 0))
            acc[(row.mix, row.rps)] = (s + row.goodput, c + 1)
        return {k: s / c for k, (s, c) in acc.items()}

    mu, ml = cell_means(usl), cell_means(lin)
    gap = max(abs(mu[k] - ml[k]) for k in mu)
    assert gap >= 0.02
    assert (f"{ml[('w2', 20.0)]:.4g}", f"{mu[('w2', 20.0)]:.4g}") == ("0.5133", "0.4867")
