"""GPU parity of the batched two-site update (BASELINE configs[1] kernel path) against
the oracle, through the C ABI (mps_bench_update_batch).  Tolerances:
tau = 1e-70 (p <= 280) / 1e-140 (p = 512), normwise; bond dimensions exact."""
import mpmath
import numpy as np
import pytest

import oracle
from synth import gen
from synth import records as R
from tests.helpers import cplx, reals, tau

pytestmark = pytest.mark.gpu


def _lib():
    import paper_1111_3124_b200 as m
    return m


def rand_lambda(p, chi, batch, key):
    """positive, descending, normalised Schmidt-like vectors (records)."""
    g = np.random.default_rng(key)
    out = []
    for b in range(batch):
        v = np.sort(np.abs(g.standard_normal(chi)) + 0.05)[::-1]
        v = v / np.linalg.norm(v)
        out.extend(v.tolist())
    return R.reals_from_values(p, out)


def theta_mat(rec, M, N):
    v = cplx(rec)
    return [[v[c * M + r] for c in range(N)] for r in range(M)]


@pytest.mark.parametrize("p,chi", [(280, 4), (280, 9), (512, 8)])
def test_theta_contraction_parity(p, chi):
    """Slice test: Theta' = U (lam_l G_A lam_m G_B lam_r) equals the oracle's."""
    m = _lib()
    batch = 3
    A, B, U = gen.update_batch_inputs(p, chi, batch)
    ll = rand_lambda(p, chi, batch, 1)
    lm = rand_lambda(p, chi, batch, 2)
    lr = rand_lambda(p, chi, batch, 3)
    got = m.update_batch(p, chi, batch, A, B, U, ll, lm, lr, theta=True)["theta"]
    want = oracle.update2_batch(p, batch, chi, chi, chi, chi, 2.0 ** -(p // 2), A, B, U, ll, lm, lr, want_theta=True)["theta"]
    n = 4 * chi * chi
    for b in range(batch):
        g = cplx(got[2 * n * b: 2 * n * (b + 1)])
        w = cplx(want[2 * n * b: 2 * n * (b + 1)])
        with mpmath.workprec(2 * p):
            err = max(abs(x - y) for x, y in zip(g, w)) / max(abs(y) for y in w)
        assert err <= tau(p), (b, err)


def gauge_invariant(GL, GR, lam, ll, lr, chi, k, chi_max, p=600):
    """P = lam_l Gamma_L diag(lam') Gamma_R lam_r  (2chi x 2chi), the truncated normalised Theta'."""
    with mpmath.workprec(2 * p + 64):
        return _gauge(GL, GR, lam, ll, lr, chi, k, chi_max)


def _gauge(GL, GR, lam, ll, lr, chi, k, chi_max):
    gl = cplx(GL)
    gr = cplx(GR)
    lamv = reals(lam)
    llv = reals(ll) if ll is not None else [mpmath.mpf(1)] * chi
    lrv = reals(lr) if lr is not None else [mpmath.mpf(1)] * chi
    P = [[mpmath.mpc(0)] * (2 * chi) for _ in range(2 * chi)]
    for i in range(2):
        for a in range(chi):
            for j in range(2):
                for c in range(chi):
                    s = mpmath.fsum(gl[(i * chi + a) * chi_max + b] * lamv[b] * gr[(j * chi_max + b) * chi + c]
                                    for b in range(k))
                    P[i * chi + a][j * chi + c] = llv[a] * s * lrv[c]
    return P


@pytest.mark.parametrize("p,chi,chi_max", [(280, 4, 4), (280, 8, 5), (512, 6, 6), (280, 16, 16)])
def test_update_parity(p, chi, chi_max):
    m = _lib()
    batch = 2
    A, B, U = gen.update_batch_inputs(p, chi, batch, first=10)
    ll = rand_lambda(p, chi, batch, 4)
    lm = rand_lambda(p, chi, batch, 5)
    lr = rand_lambda(p, chi, batch, 6)
    thr = 2.0 ** -(p // 2)
    got = m.update_batch(p, chi, batch, A, B, U, ll, lm, lr, chi_max=chi_max, thr=thr)
    want = oracle.update2_batch(p, batch, chi, chi, chi, chi_max, thr, A, B, U, ll, lm, lr)
    assert list(got["k"]) == list(want["k"])
    N = 2 * chi
    for b in range(batch):
        k = int(want["k"][b])
        sg = reals(got["sigma"][b * N:(b + 1) * N])
        sw = reals(want["sigma"][b * N:(b + 1) * N])
        with mpmath.workprec(2 * p):
            assert max(abs(x - y) for x, y in zip(sg, sw)) / sw[0] <= tau(p)
            lg = reals(got["lam"][b * chi_max:b * chi_max + k])
            lw = reals(want["lam"][b * chi_max:b * chi_max + k])
            assert max(abs(x - y) for x, y in zip(lg, lw)) <= tau(p)
        ne = 2 * 2 * chi * chi_max
        sl = slice(b * ne, (b + 1) * ne)
        llb = ll[b * chi:(b + 1) * chi]
        lrb = lr[b * chi:(b + 1) * chi]
        Pg = gauge_invariant(got["GL"][sl], got["GR"][sl], got["lam"][b * chi_max:(b + 1) * chi_max], llb, lrb, chi, k, chi_max)
        Pw = gauge_invariant(want["GL"][sl], want["GR"][sl], want["lam"][b * chi_max:(b + 1) * chi_max], llb, lrb, chi, k, chi_max)
        with mpmath.workprec(2 * p):
            d = max(abs(Pg[r][c] - Pw[r][c]) for r in range(N) for c in range(N))
            s = max(abs(Pw[r][c]) for r in range(N) for c in range(N))
            assert d / s <= tau(p), (b, d / s)
        assert 1 <= got["sweeps"][b] <= 40  # R22: the refined basis leaves 1-2 p-bit sweeps
