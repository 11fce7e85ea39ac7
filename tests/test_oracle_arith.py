"""Pins for the oracle's multiprecision arithmetic (SURVEY.md §8(c) "Pins", row O1).

* bitwise equality with mpmath (a third-party correctly rounded library,
  round-to-nearest ties-to-even) for + - x / sqrt and complex x at p in {53, 256, 280, 512};
* at p = 53 bitwise equality with IEEE-754 binary64 (numpy) — a hardware special case;
* hand-made edge cases: exact ties, carries through every limb, cancellation, zero.
"""
import random

import mpmath
import numpy as np
import pytest

import oracle
from synth import records as R


def rand_value(rng, p, emin=-300, emax=300):
    """A random exactly-p-bit value with a random exponent (plus some structured ones)."""
    kind = rng.random()
    if kind < 0.05:
        return mpmath.mpf(0)
    if kind < 0.15:  # all-ones mantissa (carry propagation through every limb)
        man = (1 << p) - 1
    elif kind < 0.25:  # power of two
        man = 1 << (p - 1)
    else:
        man = rng.getrandbits(p) | (1 << (p - 1))
    e = rng.randint(emin, emax) - p
    return R.exact_mpf(rng.random() < 0.5, man, e)


def pack(p, vals):
    return R.reals_from_values(p, vals)


def unpack(a):
    return [R.to_mpf(a[i]) for i in range(len(a))]


@pytest.mark.parametrize("p", [53, 256, 280, 512])
@pytest.mark.parametrize("op", ["add", "sub", "mul", "div", "sqrt"])
def test_bitwise_vs_mpmath(p, op):
    rng = random.Random(1000 * p + len(op))
    n = 1500
    a_vals, b_vals = [], []
    for i in range(n):
        a = rand_value(rng, p)
        if op in ("add", "sub") and rng.random() < 0.4:
            # near-cancellation / close exponents / tie-producing shifts
            b = a * R.exact_mpf(False, 1, rng.randint(-p - 3, 3)) if rng.random() < 0.5 else a
            if rng.random() < 0.5:
                b = -b
            with mpmath.workprec(p):
                b = +b
        else:
            b = rand_value(rng, p)
        if op == "div" and b == 0:
            b = mpmath.mpf(3)
        if op == "sqrt":
            a = abs(a)
        a_vals.append(a)
        b_vals.append(b)
    out = oracle.arith(p, op, pack(p, a_vals), pack(p, b_vals))
    got = unpack(out)
    with mpmath.workprec(p):
        for a, b, g in zip(a_vals, b_vals, got):
            if op == "add":
                want = a + b
            elif op == "sub":
                want = a - b
            elif op == "mul":
                want = a * b
            elif op == "div":
                want = a / b
            else:
                want = mpmath.sqrt(a)
            assert g == want, (op, p, a, b, g, want)


def test_exact_ties_round_to_even():
    # at p = 4: 1 + 2^-4 = 1.0001b -> tie -> even (1.000b); 1.001b + 2^-4 -> 1.010b
    p = 8
    cases = [
        (mpmath.mpf(1), mpmath.mpf(2) ** -8, mpmath.mpf(1)),                     # exact tie -> stays even
        (mpmath.mpf(1) + mpmath.mpf(2) ** -7, mpmath.mpf(2) ** -8, mpmath.mpf(1) + mpmath.mpf(2) ** -6),
        (mpmath.mpf(255), mpmath.mpf(1) / 2, mpmath.mpf(256)),                   # tie at carry-out
        (mpmath.mpf(254), mpmath.mpf(1) / 2, mpmath.mpf(254)),
    ]
    for a, b, want in cases:
        out = oracle.arith(p, "add", pack(p, [a]), pack(p, [b]))
        assert unpack(out)[0] == want


@pytest.mark.parametrize("op", ["add", "sub", "mul", "div", "sqrt"])
def test_binary64_special_case(op):
    """At p = 53 the oracle must be IEEE-754 binary64 (round-to-nearest-even)."""
    g = np.random.default_rng(7)
    a = g.standard_normal(4000) * np.exp2(g.integers(-60, 60, 4000))
    b = g.standard_normal(4000) * np.exp2(g.integers(-60, 60, 4000))
    b[:500] = -a[:500] * (1 + np.exp2(-g.integers(1, 52, 500)))  # cancellation
    if op == "sqrt":
        a = np.abs(a)
    want = {"add": a + b, "sub": a - b, "mul": a * b, "div": a / b, "sqrt": np.sqrt(a)}[op]
    out = oracle.arith(53, op, pack(53, a.tolist()), pack(53, b.tolist()))
    got = np.array([float(R.to_fraction(out[i])) for i in range(len(out))])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("p", [256, 280, 512])
def test_complex_mul_one_rounding(p):
    """re = RN(ac - bd), im = RN(ad + bc): equal to mpmath's mpc_mul (exact products, one rounding)."""
    rng = random.Random(p)
    n = 600
    vals = [rand_value(rng, p, -40, 40) for _ in range(4 * n)]
    a = pack(p, vals[: 2 * n])
    b = pack(p, vals[2 * n:])
    out = unpack(oracle.arith(p, "cmul", a, b))
    with mpmath.workprec(p):
        for i in range(n):
            z = mpmath.mpc(vals[2 * i], vals[2 * i + 1]) * mpmath.mpc(vals[2 * n + 2 * i], vals[2 * n + 2 * i + 1])
            assert out[2 * i] == z.real and out[2 * i + 1] == z.imag


def test_fused_multiply_add_single_rounding():
    """fma: RN(a*b + c) with one rounding — compare with the exact rational rounded by mpmath."""
    p = 280
    rng = random.Random(5)
    n = 800
    A = [rand_value(rng, p, -20, 20) for _ in range(n)]
    B = [rand_value(rng, p, -20, 20) for _ in range(n)]
    C = [(-(a * b) * (1 + mpmath.mpf(2) ** -rng.randint(1, 400))) if i % 3 == 0 else rand_value(rng, p, -40, 40)
         for i, (a, b) in enumerate(zip(A, B))]
    with mpmath.workprec(p):
        C = [+c for c in C]
    out = pack(p, C)
    oracle.arith(p, "fma", pack(p, A), pack(p, B), out)
    got = unpack(out)
    for a, b, c, g in zip(A, B, C, got):
        with mpmath.workprec(4 * p + 2000):
            exact = a * b + c  # exact at this precision
        with mpmath.workprec(p):
            assert g == +exact


def test_record_roundtrip_and_zero():
    p = 280
    vals = [mpmath.mpf(0), mpmath.mpf(1), mpmath.mpf(-3) / 8, R.exact_mpf(False, (1 << 280) - 1, -500)]
    out = oracle.arith(p, "round", pack(p, vals))
    assert unpack(out) == vals
    assert out[0]["exp"] == R.INT64_MIN
