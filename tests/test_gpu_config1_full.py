"""BASELINE configs[1] at full size (chi = 128 at 280 bits, chi = 64 at 512 bits) in the
benchmark's launch configuration (a full wave of items through the batched update kernels
that bench.py times).  The oracle needs ~330 s per full SVD, so the checks are (SURVEY §8(c) "sampled
outputs, else properties that hold at any size"):
  * sampled oracle values: Theta' of two items (the oracle's contraction, ~4 s each) equals
    the GPU's Theta' elementwise, and sum sigma^2 = ||Theta'||_F^2 to tau;
  * local-unitary invariance: item b + 8 applies U' = (V_A (x) V_B) U (V_A, V_B Haar 2 x 2)
    to the same Gamma_A, Gamma_B, so Theta'' = (V_A (x) 1)(V_B (x) 1) Theta' has the same
    singular values to tau (a general U changes them: it entangles);
  * truncation: k = chi, sigma descending, lambda' = sigma_1..k / ||sigma_1..k|| (sum 1);
  * the kept factors are orthonormal: sampled columns of X (= Gamma_A' with lambda = 1) and
    rows of V^H (= Gamma_B') have Gram matrices I to tau;
  * determinism: tiled copies of an item give bitwise identical outputs."""
import mpmath
import numpy as np
import pytest

import oracle
from synth import gen
from synth import records as R
from tests.helpers import cplx, reals, tau

pytestmark = pytest.mark.gpu

ND = 8
CASES = [(280, 128, 296), (512, 64, 148)]


def local_times(P, Ub, key):
    """(V_A (x) V_B) U rounded to P bits; V_A, V_B Haar 2 x 2 (gate index 2i + j)."""
    VA = cplx(gen.haar_unitary(P + 64, 2, 91, key, 1))
    VB = cplx(gen.haar_unitary(P + 64, 2, 91, key, 2))
    with mpmath.workprec(P + 64):
        u = cplx(Ub)
        out = R.empty(P, 32)
        for x in range(4):
            for y in range(4):
                v = mpmath.fsum(VA[(x >> 1) * 2 + (z >> 1)] * VB[(x & 1) * 2 + (z & 1)] * u[z * 4 + y] for z in range(4))
                with mpmath.workprec(P):
                    R.from_fraction(P, +v.real, out[2 * (x * 4 + y)])
                    R.from_fraction(P, +v.imag, out[2 * (x * 4 + y) + 1])
    return out


def _m():
    import paper_1111_3124_b200 as m
    return m


@pytest.fixture(scope="module", params=CASES, ids=lambda c: f"p{c[0]}_chi{c[1]}")
def run(request):
    P, CHI, BATCH = request.param
    A, B, U = gen.update_batch_inputs(P, CHI, ND)
    U2 = np.concatenate([local_times(P, U[32 * b:32 * (b + 1)], b) for b in range(ND)])
    ne = 2 * CHI * CHI * 2  # records per Gamma (complex)
    A16 = np.concatenate([A, A])
    B16 = np.concatenate([B, B])
    U16 = np.concatenate([U, U2])
    reps = BATCH // (2 * ND) + 1
    Aa = np.tile(A16, reps)[: BATCH * ne]
    Ba = np.tile(B16, reps)[: BATCH * ne]
    Ua = np.tile(U16, reps)[: BATCH * 32]
    out = _m().update_batch(P, CHI, BATCH, Aa, Ba, Ua, chi_max=CHI, thr=2.0 ** -(P // 2))
    return P, CHI, A, B, U, U2, out


def _sig(out, b, CHI):
    N = 2 * CHI
    return reals(out["sigma"][b * N:(b + 1) * N])


def test_truncation_and_order(run):
    P, CHI, _, _, _, _, out = run
    assert (out["k"] == CHI).all()
    assert (out["sweeps"] >= 1).all() and (out["sweeps"] <= 10).all()
    with mpmath.workprec(2 * P):
        for b in (0, 5, 13):
            s = _sig(out, b, CHI)
            assert all(s[i] >= s[i + 1] for i in range(len(s) - 1))
            lam = reals(out["lam"][b * CHI:(b + 1) * CHI])
            assert abs(mpmath.fsum(x * x for x in lam) - 1) <= tau(P)
            nu = mpmath.sqrt(mpmath.fsum(x * x for x in s[:CHI]))
            assert max(abs(lam[i] - s[i] / nu) for i in range(CHI)) <= tau(P)


def test_local_unitary_invariance_and_determinism(run):
    P, CHI, _, _, _, _, out = run
    with mpmath.workprec(2 * P):
        for b in range(ND):
            s1, s2 = _sig(out, b, CHI), _sig(out, b + ND, CHI)
            assert max(abs(x - y) for x, y in zip(s1, s2)) / s1[0] <= tau(P), b
    N = 2 * CHI
    for b in (0, 3):  # item b and its tiled copy b + 2 ND: identical inputs -> identical outputs
        c = b + 2 * ND
        assert out["sigma"][b * N:(b + 1) * N].tobytes() == out["sigma"][c * N:(c + 1) * N].tobytes()
        ne = 2 * 2 * CHI * CHI
        assert out["GL"][b * ne:(b + 1) * ne].tobytes() == out["GL"][c * ne:(c + 1) * ne].tobytes()


def test_sampled_theta_and_norm_vs_oracle(run):
    P, CHI, A, B, U, U2, out = run
    m = _m()
    ne = 2 * CHI * CHI * 2
    for b, Ub in ((0, U[0:32]), (ND + 1, U2[32:64])):
        ib = b % ND
        Ai, Bi = A[ib * ne:(ib + 1) * ne], B[ib * ne:(ib + 1) * ne]
        want = oracle.theta2(P, CHI, CHI, CHI, Ai, Bi, Ub)
        got = m.update_batch(P, CHI, 1, Ai, Bi, Ub, theta=True)["theta"]
        with mpmath.workprec(2 * P):
            w = cplx(want)
            g = cplx(got)
            scale = max(abs(x) for x in w)
            assert max(abs(x - y) for x, y in zip(g, w)) / scale <= tau(P)
            f2 = mpmath.fsum(abs(x) ** 2 for x in w)
            s = _sig(out, b, CHI)
            assert abs(mpmath.fsum(x * x for x in s) - f2) / f2 <= tau(P), b


def test_kept_factors_orthonormal(run):
    P, CHI, _, _, _, _, out = run
    b = 2
    ne = 2 * 2 * CHI * CHI
    GL = cplx(out["GL"][b * ne:(b + 1) * ne])  # [2][chi][chi_max]
    GR = cplx(out["GR"][b * ne:(b + 1) * ne])  # [2][chi_max][chi]
    cols = (0, 1, CHI // 3, 2 * CHI // 3, CHI - 1)
    with mpmath.workprec(2 * P):
        for ci in cols:  # X = Gamma_A' (lambda_l = 1): columns (i, a) -> c orthonormal
            for cj in cols:
                gx = mpmath.fsum(mpmath.conj(GL[(i * CHI + a) * CHI + ci]) * GL[(i * CHI + a) * CHI + cj]
                                 for i in range(2) for a in range(CHI))
                gv = mpmath.fsum(GR[(j * CHI + ci) * CHI + g] * mpmath.conj(GR[(j * CHI + cj) * CHI + g])
                                 for j in range(2) for g in range(CHI))
                e = 1 if ci == cj else 0
                assert abs(gx - e) <= tau(P), (ci, cj)
                assert abs(gv - e) <= tau(P), (ci, cj)
