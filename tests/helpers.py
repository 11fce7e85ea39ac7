"""Comparison helpers for the tests (SURVEY.md §8(c) "Comparison metrics").

Tolerance tau = 1e-70 at p <= 280 and 1e-140 at p = 512 (BASELINE.json north_star),
read NORMWISE (SURVEY §8(c) ledger #12):
  amplitudes      e = ||a - b||_inf / ||b||_inf
  singular values max_j |s^_j - s_j| / s_0, bond dims equal exactly
  local check     P = X_k diag(lambda') V_k^H, ||P^ - P||_max / ||P||_max
"""
from __future__ import annotations

from fractions import Fraction

import mpmath
import numpy as np

from synth import records as R


def tau(p: int) -> float:
    return 1e-140 if p > 280 else 1e-70


def reals(a: np.ndarray):
    return [R.to_mpf(a[i]) for i in range(len(a))]


def cplx(a: np.ndarray):
    v = reals(a)
    return [mpmath.mp.make_mpc((v[2 * i]._mpf_, v[2 * i + 1]._mpf_)) for i in range(len(v) // 2)]


def maxabs(v):
    return max((abs(x) for x in v), default=mpmath.mpf(0))


def normwise_err(got, want):
    """||got - want||_inf / ||want||_inf (complex or real sequences)."""
    with mpmath.workprec(2048):
        d = maxabs([g - w for g, w in zip(got, want)])
        s = maxabs(want)
        return d / s if s else d


def showb(rho, nq: int, digits: int = 8) -> str:
    """SPEC S:343 printer: nonzero entries only, row-major term order,
    '<coeff>|<bra bits>><<ket bits>|' joined by '+', real coefficient when
    |imag| < 10^-(digits+4), else '(re,im)'; 'nonzero' means |x| >= 10^-(digits+4)."""
    thr = mpmath.mpf(10) ** -(digits + 4)
    terms = []
    D = 1 << nq
    for r in range(D):
        for c in range(D):
            x = rho[r][c]
            if abs(x) < thr:
                continue
            if abs(x.imag) < thr:
                coeff = fmt(x.real, digits)
            else:
                coeff = "(" + fmt(x.real, digits) + "," + fmt(x.imag, digits) + ")"
            terms.append(f"{coeff}|{r:0{nq}b}><{c:0{nq}b}|")
    return "+".join(terms)


def fmt(x, digits):
    """d.ddddddde+XX (digits significant digits)."""
    s = mpmath.nstr(mpmath.mpf(x), digits, min_fixed=1, max_fixed=0, strip_zeros=False)
    # mpmath gives e.g. '5.0000000e-1' -> normalise the exponent to two digits with sign
    mant, _, ex = s.partition("e")
    e = int(ex) if ex else 0
    return f"{mant}e{'+' if e >= 0 else '-'}{abs(e):02d}"


def partial_trace_dense(psi, n: int, keep, prec: int = 1200):
    """rho_keep = Tr_{others} |psi><psi| for a dense state (qubit 0 = MSB), at `prec` bits."""
    with mpmath.workprec(prec):
        return _ptrace(psi, n, keep)


def _ptrace(psi, n, keep):
    keep = list(keep)
    k = len(keep)
    others = [q for q in range(n) if q not in keep]
    D = 1 << k
    rho = [[mpmath.mpc(0) for _ in range(D)] for _ in range(D)]
    for r in range(D):
        for c in range(D):
            acc = mpmath.mpc(0)
            for o in range(1 << len(others)):
                def idx(sub):
                    x = 0
                    for t, q in enumerate(keep):
                        if (sub >> (k - 1 - t)) & 1:
                            x |= 1 << (n - 1 - q)
                    for t, q in enumerate(others):
                        if (o >> (len(others) - 1 - t)) & 1:
                            x |= 1 << (n - 1 - q)
                    return x
                acc += psi[idx(r)] * mpmath.conj(psi[idx(c)])
            rho[r][c] = acc
    return rho


def frac(x) -> Fraction:
    return Fraction(x)


def p_sample(p: int, chi: int, k: int, GL, GR, lam, rows, cols, lam_l=None, lam_r=None):
    """Entries (rows x cols) of the gauge-invariant local check P = X_k diag(lambda') V_k^H
    (SURVEY §8(c) "Comparison metrics") of a configs[1] item with lambda_l = lambda_r = 1:
    P[(i,a),(j,c)] = sum_{b<k} GL[i][a][b] lambda'_b GR[j][b][c], row r = i chi + a,
    column j chi + c (GL [2][chi][chi_max], GR [2][chi_max][chi] complex records,
    chi_max = chi).  Each entry summed in mpmath at p + 64 bits, rounded to p bits.
    With lam_l / lam_r (records) the outer Schmidt vectors are multiplied back in,
    P[(i,a),(j,c)] = lambda_l(a) sum_b GL lambda' GR lambda_r(c): the gauge-invariant
    X_k diag(lambda') V_k^H of a window with nontrivial outer bonds (Eq. 1)."""
    from synth import records as R
    gl = cplx(GL)
    gr = cplx(GR)
    lm = reals(lam)
    ll = reals(lam_l) if lam_l is not None else None
    lr = reals(lam_r) if lam_r is not None else None
    out = R.empty(p, 2 * len(rows) * len(cols))
    with mpmath.workprec(p + 64):
        for ri, r in enumerate(rows):
            i, a = divmod(r, chi)
            xl = [gl[(i * chi + a) * chi + b] * lm[b] for b in range(k)]
            for ci, c in enumerate(cols):
                j, cc = divmod(c, chi)
                v = mpmath.fsum(xl[b] * gr[(j * chi + b) * chi + cc] for b in range(k))
                if ll is not None:
                    v *= ll[a]
                if lr is not None:
                    v *= lr[cc]
                with mpmath.workprec(p):
                    R.from_fraction(p, +v.real, out[2 * (ri * len(cols) + ci)])
                    R.from_fraction(p, +v.imag, out[2 * (ri * len(cols) + ci) + 1])
    return out
