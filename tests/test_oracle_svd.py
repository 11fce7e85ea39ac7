"""Pins for the oracle's one-sided Jacobi SVD:
third-party library (mpmath.svd_c), the 2x2 closed form, known-sigma matrices,
the identity sum sigma^2 = ||A||_F^2, reconstruction and orthogonality residuals
(SPEC S:172 tolerance 2^(-p+16))."""
import mpmath
import numpy as np
import pytest

import oracle
from synth import gen
from synth import records as R
from tests.helpers import cplx, reals


def colmajor(A_rows):
    """list-of-rows of mpc -> column-major complex records at (caller's) precision."""
    M, N = len(A_rows), len(A_rows[0])
    return [A_rows[r][c] for c in range(N) for r in range(M)]


def mat_from_records(A, M, N):
    v = cplx(A)
    return [[v[c * M + r] for c in range(N)] for r in range(M)]


@pytest.mark.parametrize("p", [256, 512])
def test_2x2_closed_form(p):
    for seed in range(6):
        A = gen.gaussian_cplx(p, 4, 77, seed)
        sig, X, V, sw = oracle.svd(p, A, 2, 2)
        a = mat_from_records(A, 2, 2)
        with mpmath.workprec(4 * p):
            f2 = sum(abs(a[r][c]) ** 2 for r in range(2) for c in range(2))
            det = a[0][0] * a[1][1] - a[0][1] * a[1][0]
            disc = mpmath.sqrt(f2 ** 2 - 4 * abs(det) ** 2)
            want = sorted([mpmath.sqrt((f2 + disc) / 2), mpmath.sqrt((f2 - disc) / 2)], reverse=True)
            got = sorted(reals(sig), reverse=True)
            err = max(abs(g - w) for g, w in zip(got, want)) / want[0]
        assert err <= mpmath.mpf(2) ** (-p + 8), err


@pytest.mark.parametrize("p,n", [(280, 6), (280, 12), (512, 8)])
def test_vs_mpmath_svd(p, n):
    A = gen.gaussian_cplx(p, n * n, 78, n)
    sig, X, V, sw = oracle.svd(p, A, n, n)
    a = mat_from_records(A, n, n)
    with mpmath.workprec(p + 64):
        want = sorted([mpmath.mpf(x) for x in mpmath.svd_c(mpmath.matrix(a), compute_uv=False)], reverse=True)
        got = sorted(reals(sig), reverse=True)
        err = max(abs(g - w) for g, w in zip(got, want)) / want[0]
    assert err <= mpmath.mpf(2) ** (-p + 16), err
    assert 3 <= sw <= 30


@pytest.mark.parametrize("p", [280])
def test_known_sigma_and_identities(p):
    """A = W diag(s) Z^H with Haar W, Z and s spanning 40 decades (M=10 > N=6)."""
    M, N = 10, 6
    s_true = [mpmath.mpf(10) ** (-8 * k) for k in range(N)]
    W = cplx(gen.haar_unitary(p + 64, M, 79, 0))
    Z = cplx(gen.haar_unitary(p + 64, N, 79, 1))
    with mpmath.workprec(p + 64):
        A = [[mpmath.fsum(W[r * M + b] * s_true[b] * mpmath.conj(Z[c * N + b]) for b in range(N))
              for c in range(N)] for r in range(M)]
    with mpmath.workprec(p):
        Ar = [[mpmath.mpc(+x.real, +x.imag) for x in row] for row in A]
    rec = R.cplx_from_values(p, [(x.real, x.imag) for x in colmajor(Ar)])
    sig, X, V, sw = oracle.svd(p, rec, M, N)
    sg = reals(sig)
    Xm = mat_from_records(X, M, N)
    Vm = mat_from_records(V, N, N)
    with mpmath.workprec(p + 64):
        got = sorted(sg, reverse=True)
        # normwise sigma error against the exact singular values of the ROUNDED A is within
        # ||A - Ar|| + rounding; compare against s_true with the input-rounding allowance
        err = max(abs(g - w) for g, w in zip(got, s_true)) / s_true[0]
        assert err <= mpmath.mpf(2) ** (-p + 16)
        # sum sigma^2 = ||A||_F^2
        f2 = mpmath.fsum(abs(x) ** 2 for row in Ar for x in row)
        assert abs(mpmath.fsum(x ** 2 for x in sg) - f2) / f2 <= mpmath.mpf(2) ** (-p + 16)
        # reconstruction A = X diag(sigma) V^H
        res = max(abs(Ar[r][c] - mpmath.fsum(Xm[r][b] * sg[b] * mpmath.conj(Vm[c][b]) for b in range(N)))
                  for r in range(M) for c in range(N))
        assert res <= mpmath.mpf(2) ** (-p + 16) * s_true[0]
        # V unitary
        vv = max(abs(mpmath.fsum(mpmath.conj(Vm[r][a]) * Vm[r][b] for r in range(N)) - (1 if a == b else 0))
                 for a in range(N) for b in range(N))
        assert vv <= mpmath.mpf(2) ** (-p + 16)


def test_zero_and_rank_deficient():
    p = 256
    # zero matrix -> all sigma 0, converges in one check-only sweep
    A = R.empty(p, 2 * 4 * 3)
    sig, X, V, sw = oracle.svd(p, A, 4, 3)
    assert all(x == 0 for x in reals(sig)) and sw == 1
    # rank one: u v^H
    u = cplx(gen.gaussian_cplx(p, 5, 80, 0))
    v = cplx(gen.gaussian_cplx(p, 4, 80, 1))
    with mpmath.workprec(p):
        rows = [[u[r] * mpmath.conj(v[c]) for c in range(4)] for r in range(5)]
    rec = R.cplx_from_values(p, [(x.real, x.imag) for x in colmajor(rows)])
    sig, X, V, sw = oracle.svd(p, rec, 5, 4)
    sg = sorted(reals(sig), reverse=True)
    with mpmath.workprec(p + 32):
        s0 = mpmath.sqrt(mpmath.fsum(abs(x) ** 2 for x in u)) * mpmath.sqrt(mpmath.fsum(abs(x) ** 2 for x in v))
        assert abs(sg[0] - s0) / s0 <= mpmath.mpf(2) ** (-p + 8)
        assert max(sg[1:]) / s0 <= mpmath.mpf(2) ** (-p + 8)
