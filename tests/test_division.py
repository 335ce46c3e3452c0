"""The CD kernel forms RN(g / nsq) as q0 = RN(g*y), r = RN(g - q0*nsq) (FMA),
q = RN(q0 + r*y) (FMA) with y = RN(1/nsq) precomputed (Markstein's
correction).  Emulated here with exact rationals (each operation rounded
once, as the FMA does) against IEEE division, on random and adversarial
operands (significands near 2, huge/small exponents, integer-valued)."""

from fractions import Fraction as F

import numpy as np


def _markstein(a: float, b: float) -> float:
    y = float(F(1) / F(b))
    q0 = float(F(a) * F(y))
    r = float(F(a) - F(b) * F(q0))
    return float(F(q0) + F(r) * F(y))


def test_markstein_quotient_is_ieee():
    rng = np.random.default_rng(7)
    for trial in range(20_000):
        kind = trial % 4
        if kind == 0:
            a, b = rng.standard_normal(), rng.random() * 2 + 1e-3
        elif kind == 1:
            a, b = rng.standard_normal() * 10.0 ** int(rng.integers(-12, 12)), 1.0 + rng.random() * 1e-3
        elif kind == 2:
            a, b = rng.standard_normal(), float(np.nextafter(2.0, 0)) * (0.5 + rng.random())
        else:
            a = float(rng.integers(-2 ** 53, 2 ** 53)) / 2 ** 40
            b = float(rng.integers(1, 2 ** 53)) / 2 ** 52
        assert _markstein(a, b) == a / b, (a, b)
