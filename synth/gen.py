"""Seeded synthetic workloads (SURVEY.md §8(d) "Synthetic inputs").

Every generator is keyed by integers only, so the oracle side and the CUDA side
receive bit-identical p-bit inputs.  Nothing here implements the method:
  * gaussian_records  — iid N(0, 1/2) reals (complex entries N(0,1/2)+iN(0,1/2)):
                        a float64 normal deviate supplies the top 53 bits, the
                        remaining p-53 mantissa bits are uniform random bits;
  * haar_unitary      — complex Gaussian d x d, modified Gram-Schmidt twice in
                        mpmath at p+32 bits (R's diagonal comes out real-positive,
                        so Q is Haar distributed), rounded to p bits;
  * circuits for BASELINE.json configs 1, 3, 4, 5 (brick-wall layouts).
Seeds: 0x11113124 + config index (0-based, BASELINE order), streams keyed
(seed, layer, position) through numpy SeedSequence.
"""
from __future__ import annotations

import numpy as np

from . import records as R

SEED0 = 0x11113124


def rng(*key) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(k) & 0xFFFFFFFF for k in key])))


def gaussian_records(p: int, n: int, *key, scale_exp: int = 0, sigma: float = 0.7071067811865476) -> np.ndarray:
    """n real records ~ N(0, sigma^2) * 2^scale_exp with p random significant bits."""
    g = rng(*key)
    x = g.standard_normal(n) * sigma
    a = R.empty(p, n)
    L = R.nlimbs(p)
    m, e = np.frexp(np.abs(x))                       # |x| = m 2^e, m in [0.5, 1)
    man53 = np.ldexp(m, 53).astype(np.uint64)        # 53-bit integer mantissa (top bit set)
    limbs = g.integers(0, 1 << 32, size=(n, L), dtype=np.uint64)
    limbs[:, L - 1] = man53 >> np.uint64(21)
    limbs[:, L - 2] = ((man53 & np.uint64((1 << 21) - 1)) << np.uint64(11)) | (limbs[:, L - 2] & np.uint64((1 << 11) - 1))
    drop = 32 * L - p                                # low bits that must be zero
    if drop:
        limbs[:, 0] &= np.uint64((0xFFFFFFFF >> drop) << drop)
    a["limb"] = limbs.astype(np.uint32)
    a["exp"] = e.astype(np.int64) + scale_exp
    a["sign"] = (x < 0).astype(np.uint32)
    zero = x == 0
    if zero.any():
        a["exp"][zero] = R.INT64_MIN
        a["limb"][zero] = 0
    return a


def gaussian_cplx(p: int, n: int, *key, scale_exp: int = 0) -> np.ndarray:
    """n complex records (2n reals, re/im interleaved), entries N(0,1/2) + i N(0,1/2)."""
    return gaussian_records(p, 2 * n, *key, scale_exp=scale_exp)


def haar_unitary(p: int, d: int, *key) -> np.ndarray:
    """d x d Haar unitary (row-major complex records)."""
    import mpmath
    z = gaussian_cplx(p + 32, d * d, *key)
    with mpmath.workprec(p + 32):
        vals = [R.to_mpf(z[i]) for i in range(2 * d * d)]
        Z = [[mpmath.mpc(vals[2 * (r * d + c)], vals[2 * (r * d + c) + 1]) for c in range(d)] for r in range(d)]
        cols = [[Z[r][c] for r in range(d)] for c in range(d)]
        for _ in range(2):  # modified Gram-Schmidt, twice
            for c in range(d):
                v = cols[c]
                for b in range(c):
                    u = cols[b]
                    h = mpmath.fsum(mpmath.conj(u[r]) * v[r] for r in range(d))
                    v = [v[r] - h * u[r] for r in range(d)]
                nrm = mpmath.sqrt(mpmath.fsum(abs(x) ** 2 for x in v))
                cols[c] = [x / nrm for x in v]
    out = R.empty(p, 2 * d * d)
    with mpmath.workprec(p):
        for r in range(d):
            for c in range(d):
                x = cols[c][r]
                R.from_fraction(p, +mpmath.mpf(x.real), out[2 * (r * d + c)])
                R.from_fraction(p, +mpmath.mpf(x.imag), out[2 * (r * d + c) + 1])
    return out


def const_gate(p: int, name: str) -> np.ndarray:
    """Named gates (row-major complex records, p-bit rounded entries)."""
    import mpmath
    with mpmath.workprec(p):
        h = +(1 / mpmath.sqrt(2))
        I2 = [[1, 0], [0, 1]]
        tbl = {
            "I": I2,
            "X": [[0, 1], [1, 0]],
            "Z": [[1, 0], [0, -1]],
            "H": [[h, h], [h, -h]],
            "CNOT": [[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]],
            "SWAP": [[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]],
            "CZ": [[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 1, 0], [0, 0, 0, -1]],
            "I4": [[1 if i == j else 0 for j in range(4)] for i in range(4)],
        }
        m = tbl[name]
        d = len(m)
        out = R.empty(p, 2 * d * d)
        for r in range(d):
            for c in range(d):
                R.from_fraction(p, mpmath.mpf(m[r][c]), out[2 * (r * d + c)])
                R.from_fraction(p, 0, out[2 * (r * d + c) + 1])
    return out


def phase_swap_gate(p: int, m: int) -> np.ndarray:
    """SWAP . diag(1,1,1,e^{2 pi i / 2^(m+2)}) (the nearest-neighbour QFT network gate)."""
    import mpmath
    with mpmath.workprec(p + 32):
        th = 2 * mpmath.pi / mpmath.mpf(2) ** (m + 2)
        c, s = mpmath.cos(th), mpmath.sin(th)
    D = [[(1, 0), (0, 0), (0, 0), (0, 0)], [(0, 0), (1, 0), (0, 0), (0, 0)],
         [(0, 0), (0, 0), (1, 0), (0, 0)], [(0, 0), (0, 0), (0, 0), (c, s)]]
    SW = [0, 2, 1, 3]  # SWAP row permutation: (SWAP.D)[r] = D[SW[r]]
    out = R.empty(p, 32)
    with mpmath.workprec(p):
        for r in range(4):
            for col in range(4):
                re, im = D[SW[r]][col]
                R.from_fraction(p, +mpmath.mpf(re), out[2 * (r * 4 + col)])
                R.from_fraction(p, +mpmath.mpf(im), out[2 * (r * 4 + col) + 1])
    return out


# --------------------------------------------------------------------- circuits
def brickwall(n: int, depth: int, p: int, seed: int, one_site_layer: bool = False):
    """List of (U records, sites) for a brick-wall circuit of Haar U(4) on (s, s+1),
    layer t acting on s = t%2, t%2+2, ...; optionally a Haar U(2) on every qubit
    after each U(4) layer (BASELINE configs[0], [2], [4])."""
    gates = []
    for t in range(depth):
        for s in range(t % 2, n - 1, 2):
            gates.append((haar_unitary(p, 4, seed, t, s), (s, s + 1)))
        if one_site_layer:
            for q in range(n):
                gates.append((haar_unitary(p, 2, seed, t, 1000 + q), (q,)))
    return gates


def triples(n: int, depth: int, p: int, seed: int):
    """Haar U(8) on (o+3j, o+3j+1, o+3j+2), o = t mod 3 (BASELINE configs[3])."""
    gates = []
    for t in range(depth):
        o = t % 3
        s = o
        while s + 2 <= n - 1:
            gates.append((haar_unitary(p, 8, seed, t, s), (s, s + 1, s + 2)))
            s += 3
    return gates


def config_circuit(idx: int, p: int | None = None, depth: int | None = None, chi_max: int | None = None):
    """(n, p, chi_max, thr, gates) for BASELINE.json configs[idx] (idx in 0, 2, 3, 4);
    depth / chi_max override the config's (scaled-down parity runs)."""
    if chi_max is not None:
        n, p_, chi, thr, gates = config_circuit(idx, p, depth)
        return n, p_, chi_max, thr, gates
    seed = SEED0 + idx
    if idx == 0:
        p = p or 280
        return 8, p, 16, 2.0 ** -140, brickwall(8, depth or 8, p, seed)
    if idx == 2:
        p = p or 280
        return 32, p, 64, 1e-60, brickwall(32, depth or 20, p, seed, one_site_layer=True)
    if idx == 3:
        p = p or 280
        return 20, p, 128, 2.0 ** -140, triples(20, depth or 16, p, seed)
    if idx == 4:
        p = p or 512
        return 64, p, 256, 2.0 ** -256, brickwall(64, depth or 40, p, seed)
    raise ValueError(idx)


def update_batch_inputs(p: int, chi: int, batch: int, seed: int = SEED0 + 1, first: int = 0):
    """Configs[1] items first..first+batch-1: Gamma_A, Gamma_B in C^{2 x chi x chi} iid,
    lambda = 1, Haar U(4).  Entry variance chosen so ||Theta||_F ~ 1 (a power-of-two scale,
    SURVEY §8(c) ledger #17): E|Theta_ij|^2 = chi s^4 with s^2 = 2^(2*scale_exp)... we scale
    each Gamma by 2^-e with e = round(log2(4 chi^3)/4)."""
    import math
    e = -int(round(math.log2(4.0 * chi ** 3) / 4.0))
    A = np.concatenate([gaussian_cplx(p, 2 * chi * chi, seed, b, 0, scale_exp=e) for b in range(first, first + batch)])
    B = np.concatenate([gaussian_cplx(p, 2 * chi * chi, seed, b, 1, scale_exp=e) for b in range(first, first + batch)])
    U = np.concatenate([haar_unitary(p, 4, seed, b, 2) for b in range(first, first + batch)])
    return A, B, U


# --------------------------------------------------------------------- graded spectra
def graded_sigma(n: int, decades: float, prec: int):
    """Nominal singular values s_b = 10^(-decades b / (n - 1)), b = 0..n-1 (mpf at prec bits)."""
    import mpmath
    with mpmath.workprec(prec):
        return [mpmath.mpf(10) ** (-mpmath.mpf(decades) * b / max(n - 1, 1)) for b in range(n)]


def householder_isometry(p: int, n: int, k: int, *key, reflections: int = 3):
    """n x k isometry Q = H_1 ... H_r [I_k; 0] (rows of mpc at p + 64 bits), H_t = I - 2 v v^H / |v|^2
    with complex Gaussian v: exactly unitary before rounding, dense and generic after r >= 2."""
    import mpmath
    prec = p + 64
    vs = [cplx_list(gaussian_cplx(prec, n, *key, t), prec) for t in range(reflections)]
    with mpmath.workprec(prec):
        Q = [[mpmath.mpc(1 if r == c else 0) for c in range(k)] for r in range(n)]
        for v in reversed(vs):  # Q <- H_t Q, last reflection first
            nv = mpmath.fsum(abs(x) ** 2 for x in v)
            for c in range(k):
                h = mpmath.fsum(mpmath.conj(v[r]) * Q[r][c] for r in range(n)) * 2 / nv
                for r in range(n):
                    Q[r][c] -= v[r] * h
    return Q


def cplx_list(a: np.ndarray, prec: int):
    import mpmath
    with mpmath.workprec(prec):
        vals = [R.to_mpf(a[i]) for i in range(len(a))]
        return [mpmath.mpc(vals[2 * i], vals[2 * i + 1]) for i in range(len(vals) // 2)]


def _round_cplx(p: int, vals) -> np.ndarray:
    import mpmath
    out = R.empty(p, 2 * len(vals))
    with mpmath.workprec(p):
        for i, z in enumerate(vals):
            R.from_fraction(p, +mpmath.mpf(z.real), out[2 * i])
            R.from_fraction(p, +mpmath.mpf(z.imag), out[2 * i + 1])
    return out


def graded_matrix(p: int, M: int, N: int, decades: float, *key, reflections: int = 3):
    """Column-major M x N (M >= N) complex records of A = W diag(s) Z^H rounded to p bits, with
    W an M x N Householder isometry, Z = H_1 ... H_r an N x N Householder unitary and
    s = graded_sigma(N, decades).  Returns (A, s): the singular values of A are s up to the
    rounding of A (normwise ~2^-p)."""
    import mpmath
    prec = p + 64
    s = graded_sigma(N, decades, prec)
    W = householder_isometry(p, M, N, *key, 0)
    vs = [cplx_list(gaussian_cplx(prec, N, *key, 1, t), prec) for t in range(reflections)]
    with mpmath.workprec(prec):
        A = [[W[r][b] * s[b] for b in range(N)] for r in range(M)]
        for v in vs:  # A <- A H_t for t = 1..r (Z^H = H_r ... H_1, each H Hermitian)
            nv = mpmath.fsum(abs(x) ** 2 for x in v)
            for r in range(M):
                h = mpmath.fsum(A[r][c] * v[c] for c in range(N)) * 2 / nv
                for c in range(N):
                    A[r][c] -= h * mpmath.conj(v[c])
        cm = [A[r][c] for c in range(N) for r in range(M)]
    return _round_cplx(p, cm), s


def graded_update_inputs(p: int, chi: int, decades: float, *key, in_lambda: bool = True):
    """A two-site update input (BASELINE configs[1] layout, [2][chi][chi] complex records) whose
    Theta = Gamma_A diag(lambda_m) Gamma_B is W diag(s) Z^H: W, Z 2chi x chi Householder isometries,
    s = graded_sigma(chi, decades); Gamma_A^i(a, b) = W[i chi + a][b], Gamma_B^j(b, c) =
    conj(Z[j chi + c][b]).  in_lambda: s is the middle Schmidt vector lambda_m (returned as
    records); else s is folded into Gamma_A and lambda_m is None (all ones).
    Returns (A, B, lam_m or None, s)."""
    import mpmath
    s = graded_sigma(chi, decades, p + 64)
    W = householder_isometry(p, 2 * chi, chi, *key, 0)
    Z = householder_isometry(p, 2 * chi, chi, *key, 1)
    with mpmath.workprec(p + 64):
        GA = [W[i * chi + a][b] * (1 if in_lambda else s[b]) for i in range(2) for a in range(chi) for b in range(chi)]
        GB = [mpmath.conj(Z[j * chi + c][b]) for j in range(2) for b in range(chi) for c in range(chi)]
    lam = None
    if in_lambda:
        lam = R.empty(p, chi)
        with mpmath.workprec(p):
            for b in range(chi):
                R.from_fraction(p, +s[b], lam[b])
    return _round_cplx(p, GA), _round_cplx(p, GB), lam, s


def schmidt_profile(chi: int, decades: float, prec: int):
    """A unit-norm Schmidt vector with a graded profile: graded_sigma(chi, decades) / its 2-norm
    (descending, sum of squares 1 to the rounding of prec bits)."""
    import mpmath
    s = graded_sigma(chi, decades, prec)
    with mpmath.workprec(prec):
        nrm = mpmath.sqrt(mpmath.fsum(x * x for x in s))
        return [x / nrm for x in s]


def canonical_update_inputs(p: int, chi: int, dec_l: float, dec_m: float, dec_r: float, *key):
    """One two-site gate input as it meets a gate deep inside a saturated configs[4] circuit
    (BASELINE configs[4]: chi_l = chi_m = chi_r = chi): a Vidal canonical window (Eq. 1,
    P:240-247) with graded unit-norm Schmidt vectors lambda_l, lambda_m, lambda_r
    (schmidt_profile with dec_l, dec_m, dec_r decades) and
      Gamma_A^i(a, b) = W[i chi + a][b] / lambda_l(a)     (lambda_l Gamma_A left-normalised),
      Gamma_B^j(b, c) = conj(Z[j chi + c][b]) / lambda_r(c) (Gamma_B lambda_r right-normalised),
    W, Z 2chi x chi Householder isometries at p + 64 bits, so Theta = lambda_l Gamma_A lambda_m
    Gamma_B lambda_r = W diag(lambda_m) Z^H before the gate, and a seeded Haar U(4).  The gate
    mixes the physical indices, so Theta' = U Theta has 2chi generic graded singular values and
    truncation to chi_max = chi drops half of them.  Nothing here computes the update.
    Returns (A, B, lam_l, lam_m, lam_r, U) as p-bit records."""
    import mpmath
    prec = p + 64
    ll = schmidt_profile(chi, dec_l, prec)
    lm = schmidt_profile(chi, dec_m, prec)
    lr = schmidt_profile(chi, dec_r, prec)
    W = householder_isometry(p, 2 * chi, chi, *key, 0)
    Z = householder_isometry(p, 2 * chi, chi, *key, 1)
    with mpmath.workprec(prec):
        GA = [W[i * chi + a][b] / ll[a] for i in range(2) for a in range(chi) for b in range(chi)]
        GB = [mpmath.conj(Z[j * chi + c][b]) / lr[c] for j in range(2) for b in range(chi) for c in range(chi)]
    lams = []
    for v in (ll, lm, lr):
        r = R.empty(p, chi)
        with mpmath.workprec(p):
            for b in range(chi):
                R.from_fraction(p, +v[b], r[b])
        lams.append(r)
    U = haar_unitary(p, 4, *key, 2)
    return (_round_cplx(p, GA), _round_cplx(p, GB), *lams, U)
