"""Synthetic inputs of the BASELINE configs, generated exactly as SURVEY §8(d)
specifies them (numpy, vectorised; no reference code).

* `mt19937_64(seed, count)`: the first `count` outputs of C++
  std::mt19937_64(seed) (default seeding, [rand.eng.mers]); the 312-word twist
  runs in its two data-parallel halves (words 0..155 read only old state,
  words 156..311 read the new words 0..155).
* `uniform01(x)`: the reference's `uniform01` (workload.cpp:17-19): the top 53
  bits times 2^-53.
* `config4_curves(n)`: config 4 — per curve, truth usl v1 = 50 + 100u,
  sigma = 0.2u, kappa = 0.005u, then for L = 1..m speed = predict(truth, L) *
  (1 + 0.01 (u - 0.5)) (the saber_bench.cpp:56-59 noise model), all u drawn in
  that order from one mt19937_64(2026) stream; predict is the reference's USL
  expression (estimator.cpp:19-21), evaluated left to right without FMA.
"""
import numpy as np

_N, _M = 312, 156
_UPPER = np.uint64(0xFFFFFFFF80000000)
_LOWER = np.uint64(0x7FFFFFFF)
_MATRIX = np.uint64(0xB5026F5AA96619E9)


def _seed_state(seed):
    mt = np.zeros(_N, dtype=np.uint64)
    x = seed & 0xFFFFFFFFFFFFFFFF
    mt[0] = x
    for i in range(1, _N):
        x = (6364136223846793005 * (x ^ (x >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        mt[i] = x
    return mt


def _twist(mt):
    one = np.uint64(1)
    new = np.empty_like(mt)
    y = (mt[:_M] & _UPPER) | (mt[1:_M + 1] & _LOWER)
    new[:_M] = mt[_M:] ^ (y >> one) ^ np.where(y & one, _MATRIX, np.uint64(0))
    nxt = np.concatenate([mt[_M + 1:], new[:1]])  # word k+1 (k = 311 wraps to the new word 0)
    y = (mt[_M:] & _UPPER) | (nxt & _LOWER)
    new[_M:] = new[:_M] ^ (y >> one) ^ np.where(y & one, _MATRIX, np.uint64(0))
    return new


def mt19937_64(seed, count):
    mt = _seed_state(seed)
    blocks = (count + _N - 1) // _N
    out = np.empty(blocks * _N, dtype=np.uint64)
    for b in range(blocks):
        mt = _twist(mt)
        out[b * _N:(b + 1) * _N] = mt
    y = out[:count]
    y = y ^ ((y >> np.uint64(29)) & np.uint64(0x5555555555555555))
    y = y ^ ((y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000))
    y = y ^ ((y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000))
    y = y ^ (y >> np.uint64(43))
    return y


def uniform01(x):
    return (x >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def config4_curves(n, seed=2026, m=50):
    """(loads i32 [n*m], speeds f64 [n*m], offsets i64 [n+1], truth [n][3])."""
    u = uniform01(mt19937_64(seed, n * (3 + m))).reshape(n, 3 + m)
    truth = np.stack([50.0 + 100.0 * u[:, 0], 0.2 * u[:, 1], 0.005 * u[:, 2]], 1)
    L = np.arange(1, m + 1, dtype=np.float64)
    denom = (1.0 + truth[:, 1:2] * (L - 1.0)) + (truth[:, 2:3] * L) * (L - 1.0)
    speeds = (truth[:, 0:1] / denom) * (1.0 + 0.01 * (u[:, 3:] - 0.5))
    loads = np.tile(np.arange(1, m + 1, dtype=np.int32), n)
    offsets = np.arange(0, n * m + 1, m, dtype=np.int64)
    return loads, speeds.reshape(-1), offsets, truth
