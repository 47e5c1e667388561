"""The engine's correctly-rounded sin/cos (csrc/exa_math.h, host build):
the Ziv fast path agrees with the double-double slow path wherever it
accepts, defers rarely, and the whole routine matches glibc (numpy) on all
but the ~0.2% of arguments where glibc itself is not correctly rounded."""

import numpy as np

from oracle import crtrig


def _samples(n=1_000_000, seed=0):
    rng = np.random.default_rng(seed)
    return np.concatenate([
        rng.uniform(-np.pi / 4, np.pi / 4, n),
        rng.integers(-50, 51, n // 10) / 64.0 + rng.uniform(-2.0**-20, 2.0**-20, n // 10),  # table knots
        rng.uniform(-1 / 128, 1 / 128, n // 10),                                          # j = 0
        rng.uniform(-1e-6, 1e-6, n // 20),
    ])


def test_fast_path_equals_slow_path_where_accepted():
    x = _samples()
    s, c, ok = crtrig.sincos_fast(x)
    ss, cc = crtrig.sincos_slow(x)
    assert np.array_equal(s[ok], ss[ok]) and np.array_equal(c[ok], cc[ok])
    u = x[: 1_000_000]
    assert 1.0 - ok[: u.size].mean() < 5e-5  # uniform arguments: the slow path is rare


def test_full_routine_matches_glibc_mostly():
    rng = np.random.default_rng(1)
    x = rng.uniform(-0.8, 0.8, 400_000)
    s, c = crtrig.sincos(x)
    assert (s != np.sin(x)).mean() < 5e-3 and (c != np.cos(x)).mean() < 5e-3
    # out-of-fast-range arguments take the reduction path
    y = rng.uniform(-50, 50, 100_000)
    s2, c2 = crtrig.sincos(y)
    assert (s2 != np.sin(y)).mean() < 5e-3 and (c2 != np.cos(y)).mean() < 5e-3
