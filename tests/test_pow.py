"""The shared deterministic pow (csrc/ef_pow.h): accuracy and IEEE special cases."""

import math

import mpmath as mp
import numpy as np
import pytest

import oracle as O

HOT_EXPONENTS = [1 / 2.4, -1.4, -(0.4 / 2.8), 0.4 / 2.8, 2.8 / 0.4, 2.4, 1.4, (-1.4) * (1 / 2.4)]


@pytest.mark.parametrize("y", HOT_EXPONENTS + [0.5, 3.0, -7.3])
def test_pow_is_within_about_one_ulp(y):
    mp.mp.prec = 120
    rng = np.random.default_rng(11)
    x = np.concatenate([np.exp(rng.uniform(-30, 30, 400)), rng.uniform(0.5, 2.0, 300),
                        1.0 + rng.standard_normal(100) * 1e-9])
    r = O.shared_pow(x, y)
    worst = 0.0
    for xi, ri in zip(x, r):
        ex = mp.power(mp.mpf(float(xi)), mp.mpf(y))
        worst = max(worst, float(abs(mp.mpf(float(ri)) - ex) / math.ulp(float(ex))))
    assert worst < 1.1


def test_pow_special_cases_follow_numpy():
    cases = [(0.0, 2.4), (0.0, -1.4), (-0.0, 3.0), (-0.0, -3.0), (-2.0, 3.0), (-2.0, 2.0), (np.inf, 2.0),
             (np.inf, -2.0), (-np.inf, 3.0), (np.nan, 0.0), (1.0, np.nan), (2.0, np.inf), (0.5, np.inf),
             (2.0, -np.inf), (5e-324, 0.5), (1e308, 1.5), (1e-308, 2.0), (-2.0, 2.4), (np.nan, 2.0)]
    with np.errstate(all="ignore"):
        for x, y in cases:
            a = O.shared_pow(np.array([x]), y)[0]
            b = np.power(x, y)
            if np.isnan(b):
                assert np.isnan(a), (x, y)
            else:
                assert a == b and math.copysign(1, a) == math.copysign(1, b), (x, y, a, b)


def test_pow_is_monotone_on_a_fine_grid():
    x = np.linspace(0.5, 2.0, 200001)
    for y in (2.4, -1.4, 1 / 2.4):
        r = O.shared_pow(x, y)
        d = np.diff(r)
        assert (d >= 0).all() if y > 0 else (d <= 0).all()


def _worst_ulp(x, y):
    mp.mp.prec = 160
    r = O.shared_pow(x, y)
    worst = 0.0
    for xi, ri in zip(x, r):
        ex = mp.power(mp.mpf(float(xi)), mp.mpf(y))
        worst = max(worst, float(abs(mp.mpf(float(ri)) - ex) / math.ulp(float(ex))))
    return worst


@pytest.mark.parametrize("name", ["two_g_over_gm1", "neg_gm1_over_2g"])
def test_specialised_pows_of_gamma_seven_fifths(name):
    """ef_pow7 / ef_powm17 (csrc/ef_pow.h): the two-rarefaction exponents of gamma = 7/5
    (riemann.py:88-100) stay within 0.52 ulp over their whole argument range 2^-100 .. 2^100,
    and the pow is continuous (to an ulp) where it hands over to the general algorithm."""
    from paper_2007_00094_b200.physics import AIR

    y = AIR.two_g_over_gm1 if name == "two_g_over_gm1" else -AIR.gm1_over_2g
    assert abs(y - (7.0 if y > 0 else -1 / 7)) < 2.0 ** -44  # the specialised algorithms apply
    rng = np.random.default_rng(5)
    lim = 100.0 / 7.2 if y > 0 else 100.0  # keep x^7 finite
    x = np.concatenate([np.exp2(rng.uniform(-lim, lim, 3000)), rng.uniform(0.25, 4.0, 3000),
                        1.0 + rng.standard_normal(500) * 1e-6,
                        np.exp2(rng.integers(-99, 100, 200).astype(np.float64)) * (1.0 + 2.0 ** -52)])
    assert _worst_ulp(x, y) < 0.52
    for edge in (2.0 ** -100, 2.0 ** 100):  # hand-over to the general algorithm
        xs = np.array([np.nextafter(edge, 0.0), edge, np.nextafter(edge, np.inf)])
        with np.errstate(all="ignore"):
            r = O.shared_pow(xs, y)
        if np.isfinite(r).all() and (r > 1e-300).all():
            assert _worst_ulp(xs, y) < 0.52
    # an exponent just outside the 2^-44 window takes the general algorithm: same accuracy class
    assert _worst_ulp(x[:500], y + 2.0 ** -40) < 0.52
