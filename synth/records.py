"""Interchange-record codec shared by the tests, the oracle wrapper and bench.py.

Pure format marshalling — no arithmetic of the method lives here.  The record
format is the one declared in include/mps_b200.h:

    int64 exp; uint32 sign; uint32 reserved; uint32 limb[L],  L = ceil(p/32)
    value = (-1)^sign * (sum_k limb[k] 2^(32k)) * 2^(exp - 32L)
    zero: all limbs 0 and exp = INT64_MIN; nonzero: limb[L-1] >= 2^31 and the
    low 32L-p bits are zero (exactly p significant bits).

A complex number is the re record followed by the im record.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

INT64_MIN = -(1 << 63)


def nlimbs(p: int) -> int:
    return (p + 31) // 32


def record_bytes(p: int) -> int:
    return 16 + 4 * nlimbs(p)


def record_dtype(p: int) -> np.dtype:
    return np.dtype([("exp", "<i8"), ("sign", "<u4"), ("res", "<u4"), ("limb", "<u4", (nlimbs(p),))])


def empty(p: int, n: int) -> np.ndarray:
    """n zero records (structured array)."""
    a = np.zeros(n, dtype=record_dtype(p))
    a["exp"] = INT64_MIN
    return a


# --------------------------------------------------------------------- scalar codec
def pack_int_exp(p: int, neg: bool, man: int, exp2: int) -> tuple[int, int, list[int]]:
    """Record fields for (-1)^neg * man * 2^exp2 with man < 2^p (exactly representable)."""
    L = nlimbs(p)
    if man == 0:
        return INT64_MIN, 0, [0] * L
    bc = man.bit_length()
    if bc > p:
        raise ValueError("mantissa has more than p bits")
    M = man << (32 * L - bc)
    e = exp2 + bc
    return e, 1 if neg else 0, [(M >> (32 * k)) & 0xFFFFFFFF for k in range(L)]


def to_fraction(rec) -> Fraction:
    """Exact value of one record (row of a structured array)."""
    e = int(rec["exp"])
    limbs = [int(x) for x in rec["limb"]]
    if e == INT64_MIN or not any(limbs):
        return Fraction(0)
    L = len(limbs)
    M = 0
    for k in reversed(range(L)):
        M = (M << 32) | limbs[k]
    sh = e - 32 * L
    v = Fraction(M) * (Fraction(2) ** sh)
    return -v if int(rec["sign"]) else v


def from_fraction(p: int, v, rec) -> None:
    """Write a value that is EXACTLY representable with p bits (int, Fraction with
    power-of-two denominator, float, or mpmath mpf) into a record row."""
    try:
        import mpmath  # noqa: F401
        if hasattr(v, "_mpf_"):
            s, man, ex, bc = v._mpf_
            if man == 0:
                e, sg, limbs = INT64_MIN, 0, [0] * nlimbs(p)
            else:
                e, sg, limbs = pack_int_exp(p, bool(s), int(man), int(ex))
            rec["exp"], rec["sign"], rec["limb"] = e, sg, limbs
            return
    except ImportError:
        pass
    f = Fraction(v)
    if f == 0:
        rec["exp"], rec["sign"], rec["limb"] = INT64_MIN, 0, [0] * nlimbs(p)
        return
    neg = f < 0
    f = abs(f)
    num, den = f.numerator, f.denominator
    if den & (den - 1):
        raise ValueError("not a dyadic rational")
    exp2 = -(den.bit_length() - 1)
    # strip trailing zero bits of num
    tz = (num & -num).bit_length() - 1
    num >>= tz
    exp2 += tz
    e, sg, limbs = pack_int_exp(p, neg, num, exp2)
    rec["exp"], rec["sign"], rec["limb"] = e, sg, limbs


def to_mpf(rec):
    import mpmath
    e = int(rec["exp"])
    limbs = [int(x) for x in rec["limb"]]
    if e == INT64_MIN or not any(limbs):
        return mpmath.mpf(0)
    L = len(limbs)
    M = 0
    for k in reversed(range(L)):
        M = (M << 32) | limbs[k]
    return exact_mpf(bool(int(rec["sign"])), M, e - 32 * L)


def exact_mpf(neg: bool, man: int, exp2: int):
    """mpmath mpf equal to (-1)^neg * man * 2^exp2 exactly (no rounding to the context)."""
    import mpmath
    from mpmath.libmp import from_man_exp, mpf_neg
    v = from_man_exp(int(man), int(exp2))
    return mpmath.mp.make_mpf(mpf_neg(v) if neg else v)


# --------------------------------------------------------------------- array helpers
def reals_from_values(p: int, values) -> np.ndarray:
    a = empty(p, len(values))
    for i, v in enumerate(values):
        from_fraction(p, v, a[i])
    return a


def cplx_from_values(p: int, values) -> np.ndarray:
    """complex-valued sequence -> 2n records (re, im interleaved)."""
    values = list(values)
    a = empty(p, 2 * len(values))
    for i, v in enumerate(values):
        re, im = (v.real, v.imag) if not isinstance(v, tuple) else v
        from_fraction(p, re, a[2 * i])
        from_fraction(p, im, a[2 * i + 1])
    return a


def to_float64(a: np.ndarray) -> np.ndarray:
    """Approximate float64 view of records (diagnostics / loose checks only)."""
    top = a["limb"][..., -1].astype(np.float64) * 2.0 ** 32 + a["limb"][..., -2].astype(np.float64) \
        if a["limb"].shape[-1] > 1 else a["limb"][..., -1].astype(np.float64)
    L = a["limb"].shape[-1]
    nb = 64 if L > 1 else 32
    e = a["exp"].astype(np.int64)
    zero = (e == INT64_MIN)
    ee = np.where(zero, 0, e - nb).astype(np.float64)
    v = np.ldexp(top, ee.astype(np.int64))
    v = np.where(a["sign"] != 0, -v, v)
    return np.where(zero, 0.0, v)


def cplx_to_complex128(a: np.ndarray) -> np.ndarray:
    f = to_float64(a)
    return f[0::2] + 1j * f[1::2]
