"""GPU unit tests of the device multiprecision formats against the oracle:
device mpf ops are faithful at p bits (within 2 ulp of the correctly rounded oracle
result), the fixed-point digit format round-trips, and the Jacobi SVD of given matrices
matches the oracle's singular values (normwise, tau)."""
import random

import mpmath
import numpy as np
import pytest

import oracle
from synth import gen
from synth import records as R
from tests.helpers import reals, tau

pytestmark = pytest.mark.gpu


def _m():
    import paper_1111_3124_b200 as m
    return m


def rand_vals(rng, p, n, emin=-200, emax=200):
    out = []
    for i in range(n):
        man = rng.getrandbits(p) | (1 << (p - 1))
        if i % 17 == 0:
            man = (1 << p) - 1
        out.append(R.exact_mpf(rng.random() < 0.5, man, rng.randint(emin, emax) - p))
    return out


@pytest.mark.parametrize("p", [256, 280, 512])
@pytest.mark.parametrize("op", ["add", "sub", "mul", "div", "sqrt", "fixed"])
def test_mpf_ops_faithful(p, op):
    m = _m()
    rng = random.Random(p * 7 + len(op))
    n = 600
    a = rand_vals(rng, p, n)
    b = rand_vals(rng, p, n, -60, 60)
    if op in ("add", "sub"):
        for i in range(0, n, 5):  # cancellation cases
            b[i] = a[i] * (1 + mpmath.mpf(2) ** -rng.randint(1, p - 2))
            with mpmath.workprec(p):
                b[i] = +b[i]
    if op == "sqrt":
        a = [abs(x) for x in a]
    A = R.reals_from_values(p, a)
    B = R.reals_from_values(p, b)
    got = reals(m.debug_mpf(p, op, A, B))
    if op == "fixed":
        for g, x in zip(got, a):
            assert abs(g - x) <= abs(x) * mpmath.mpf(2) ** (-p + 1)
        return
    want = reals(oracle.arith(p, op, A, B) if op != "sqrt" else oracle.arith(p, "sqrt", A))
    for g, w, x, y in zip(got, want, a, b):
        with mpmath.workprec(4 * p):
            if op in ("add", "sub"):
                scale = max(abs(x), abs(y))  # faithful w.r.t. the operands (cancellation)
            else:
                scale = abs(w)
            assert abs(g - w) <= scale * mpmath.mpf(2) ** (-p + 2), (op, x, y, g, w)


@pytest.mark.parametrize("p,M,N", [(280, 8, 8), (280, 12, 6), (280, 5, 9), (512, 10, 10), (280, 32, 32)])
def test_svd_sigma_parity(p, M, N):
    m = _m()
    batch = 2
    A = np.concatenate([gen.gaussian_cplx(p, M * N, 55, b, M, N) for b in range(batch)])
    sig, sw, rps, rc = m.svd_batch(p, M, N, batch, A)
    assert rc == 0, (sw, rps)
    n = min(M, N)
    for b in range(batch):
        Ab = A[2 * M * N * b: 2 * M * N * (b + 1)]
        if N <= M:
            osig, _, _, osw = oracle.svd(p, Ab, M, N)
        else:  # oracle needs N <= M: use A^H (same singular values)
            from tests.helpers import cplx
            v = cplx(Ab)
            with mpmath.workprec(p):
                vh = [mpmath.conj(v[c * M + r]) for r in range(M) for c in range(N)]
            AH = R.cplx_from_values(p, [(z.real, z.imag) for z in vh])
            osig, _, _, osw = oracle.svd(p, AH, N, M)
        want = sorted(reals(osig), reverse=True)
        got = reals(sig[n * b: n * (b + 1)])
        with mpmath.workprec(2 * p):
            err = max(abs(g - w) for g, w in zip(got, want)) / want[0]
        assert err <= tau(p), (b, err, sw[b], rps[b][:20])


def test_svd_rank_deficient_and_graded():
    """Rank-one and strongly graded (sigma over 60 decades) matrices converge."""
    m = _m()
    p = 280
    M = N = 8
    u = gen.gaussian_cplx(p, M, 56, 0)
    from tests.helpers import cplx
    uv = cplx(u)
    with mpmath.workprec(p):
        rows = [uv[r] * mpmath.conj(uv[c]) for c in range(N) for r in range(M)]
    A = R.cplx_from_values(p, [(z.real, z.imag) for z in rows])
    sig, sw, rps, rc = m.svd_batch(p, M, N, 1, A)
    assert rc == 0
    s = reals(sig)
    with mpmath.workprec(p):
        nrm = mpmath.fsum(abs(x) ** 2 for x in uv)
        assert abs(s[0] - nrm) / nrm <= tau(p)
        assert max(s[1:]) / nrm <= tau(p)
