"""Exact-rational model of IEEE-754 binary32 round-to-nearest-even arithmetic.

Independent of both the C oracle and the GPU: every operation is computed
exactly with fractions.Fraction and rounded once by `round_f32`, which is a
direct transcription of the IEEE-754 rounding rule (ties to even, gradual
underflow, overflow to infinity).  Used for brute-force pins on tiny inputs.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

_MAX_FINITE = Fraction((2 ** 24 - 1) * 2 ** 104)  # (2 - 2^-23) * 2^127
_OVF = Fraction(2 ** 128) - Fraction(2 ** 103)    # halfway between max finite and 2^128


def round_f32(q: Fraction, neg_zero: bool = False) -> np.float32:
    """Round an exact rational to the nearest binary32, ties to even."""
    if q == 0:
        return np.float32(-0.0) if neg_zero else np.float32(0.0)
    sign = -1 if q < 0 else 1
    a = -q if q < 0 else q
    if a >= _OVF:
        return np.float32(sign * math.inf)
    # exponent e with 2^e <= a < 2^(e+1)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    elif Fraction(2) ** (e + 1) <= a:
        e += 1
    quantum_exp = max(e, -126) - 23
    quantum = Fraction(2) ** quantum_exp
    n = a / quantum
    fl = n.numerator // n.denominator
    rem = n - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    val = Fraction(fl) * quantum
    if val > _MAX_FINITE:
        return np.float32(sign * math.inf)
    return np.float32(sign * float(val))


def F(x) -> Fraction:
    return Fraction(float(np.float32(x)))


def _special(*xs) -> bool:
    return any(not math.isfinite(float(x)) for x in xs)


def add(a, b) -> np.float32:
    a, b = np.float32(a), np.float32(b)
    if _special(a, b):
        with np.errstate(all="ignore"):
            return np.float32(a + b)
    s = F(a) + F(b)
    neg0 = s == 0 and math.copysign(1, a) < 0 and math.copysign(1, b) < 0
    return round_f32(s, neg0)


def sub(a, b) -> np.float32:
    return add(a, -np.float32(b))


def mul(a, b) -> np.float32:
    a, b = np.float32(a), np.float32(b)
    if _special(a, b):
        with np.errstate(all="ignore"):
            return np.float32(a * b)
    p = F(a) * F(b)
    neg0 = p == 0 and (math.copysign(1, a) * math.copysign(1, b)) < 0
    return round_f32(p, neg0)


def fma(a, b, c) -> np.float32:
    a, b, c = np.float32(a), np.float32(b), np.float32(c)
    if _special(a, b, c):
        with np.errstate(all="ignore"):
            return np.float32(np.float64(a) * np.float64(b) + np.float64(c))
    p = F(a) * F(b)
    s = p + F(c)
    if s == 0:
        pneg = p == 0 and (math.copysign(1, a) * math.copysign(1, b)) < 0
        neg0 = (p != 0 and False) or (p == 0 and pneg and math.copysign(1, c) < 0)
        return round_f32(s, neg0)
    return round_f32(s)


def f32_bits(x) -> int:
    return int(np.float32(x).view(np.uint32))


def ulp_f32(x: float) -> float:
    """Spacing of binary32 at |x| (for error bounds)."""
    x = abs(float(x))
    if x < 2.0 ** -126:
        return 2.0 ** -149
    e = math.floor(math.log2(x))
    if 2.0 ** e > x:
        e -= 1
    return 2.0 ** (e - 23)
