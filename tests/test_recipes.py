"""The benchmark input recipes (benchmarks/recipes.py) follow SURVEY §8(d):
the vectorised mt19937_64 equals the C++ engine (its 10000th output from the
default seed is the standard's known answer, [rand.predef]) and config 4's
curves are the reference's predict() times the saber_bench.cpp noise model."""
import numpy as np

import recipes


def test_mt19937_64_known_answer():
    assert int(recipes.mt19937_64(5489, 10000)[-1]) == 9981545732273789042


def test_mt19937_64_matches_scalar_engine():
    from test_acceptance import MT19937_64
    m = MT19937_64(2026)
    want = [m() for _ in range(700)]
    assert [int(x) for x in recipes.mt19937_64(2026, 700)] == want


def test_config4_curves_follow_the_recipe(ref):
    loads, speeds, offsets, truth = recipes.config4_curves(8)
    m = 50
    u = recipes.uniform01(recipes.mt19937_64(2026, 8 * (3 + m))).reshape(8, 3 + m)
    assert np.array_equal(truth[:, 0], 50.0 + 100.0 * u[:, 0])
    for c in range(8):
        for L in (1, 2, 17, 50):
            want = ref.predict(0, list(truth[c]), L) * (1.0 + 0.01 * (u[c, 3 + L - 1] - 0.5))
            assert speeds[offsets[c] + L - 1] == want
    assert list(loads[:m]) == list(range(1, m + 1))
