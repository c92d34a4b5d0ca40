"""CPU: the arithmetic facts DESIGN.md §3 leans on, checked directly.

* x % d == x - umulhi(x, ceil(2^32/d)) * d for every x < 720720, d in 2..16
  (the kernel's Fisher-Yates modulo on draws stored mod lcm(1..16));
* (r % 720720) % d == r % d for d in 2..16 (lcm property);
* min_i fl(r_i / s) == fl(min_i r_i / s) and min_i fl(p_i - dt) == fl(min_i p_i - dt)
  (monotone correctly rounded division / subtraction);
* the demotion bound never exceeds the first tick at which the reference demotes.
"""
import math
import random

import numpy as np


def test_reciprocal_modulo_is_exact():
    x = np.arange(720720, dtype=np.uint64)
    for d in range(2, 17):
        inv = np.uint64((2 ** 32 + d - 1) // d)
        q = (x * inv) >> np.uint64(32)
        assert np.array_equal(x - q * np.uint64(d), x % np.uint64(d)), d


def test_lcm_modulus():
    assert math.lcm(*range(1, 17)) == 720720
    rng = np.random.default_rng(0)
    r = rng.integers(0, 2 ** 63, size=200000, dtype=np.uint64)
    for d in range(2, 17):
        assert np.array_equal((r % np.uint64(720720)) % np.uint64(d), r % np.uint64(d))


def test_monotone_rounding_rewrites():
    rng = random.Random(1)
    for _ in range(20000):
        s = rng.uniform(1e-3, 200.0)
        rs = [rng.uniform(0, 1000) * rng.choice([1, 1e-6, 1e-12]) for _ in range(rng.randint(1, 40))]
        assert min(r / s for r in rs) == min(rs) / s
        dt = rng.uniform(0, 0.02)
        ps = [dt + rng.uniform(0, 1) * rng.choice([1, 1e-9]) for _ in range(rng.randint(1, 10))]
        assert min(p - dt for p in ps) == min(ps) - dt


def demote_bound(m, dl, c):
    q = m / c
    return dl - q * (1.0 + 1e-9) - 1e-9 * (abs(dl) + 1.0)


def test_demotion_bound_is_conservative():
    """Walk the reference's accumulated tick clock; the first tick at which
    fl(m / fl(dl - t)) > c must never precede demote_after."""
    rng = random.Random(7)
    for _ in range(3000):
        c = rng.uniform(20.0, 150.0)
        m = float(rng.randint(1, 800))
        arrival = rng.uniform(0, 200.0)
        dl = arrival + rng.choice([1.0, 8.0, 12.0])
        tick = rng.choice([0.01, 0.003, 0.05])
        T = demote_bound(m, dl, c)
        t = 0.0
        # jump near the bound, then step like the reference (t = t + tick)
        k = max(0, int((T - 1.0) / tick))
        for _ in range(k):
            t = t + tick
        for _ in range(int(2.0 / tick) + 3):
            need = math.inf if t >= dl else m / (dl - t)
            if need > c:
                assert t >= T, (m, dl, c, t, T)
                break
            t = t + tick
