"""Pins for the oracle's MPS gate update, queries and dense simulator
(SURVEY.md §8(c) "Pins"): brute-force dense state vector (n <= 12), GHZ and QFT
closed forms, echo circuits, the paper's §3.2 printed output,
Eckart-Young truncation identity, norm preservation, Schmidt form (Eq. 2)."""
import mpmath
import numpy as np
import pytest

import oracle
from synth import gen
from synth import records as R
from tests.helpers import cplx, fmt, normwise_err, partial_trace_dense, reals, showb, tau

GOLDEN = [l.rstrip("\n") for l in open(__file__.replace("test_oracle_tebd.py", "golden/qc_simple_example.txt"))
          if not l.startswith("#")]


def dense_of(gates, n, p):
    d = oracle.OracleDense(n, p)
    for U, s in gates:
        d.apply(U, s)
    return cplx(d.state())


def mps_of(gates, n, p, chi, thr):
    m = oracle.OracleMPS(n, p, chi, thr)
    for U, s in gates:
        m.apply(U, s)
    return m


def test_paper_golden_qc_simple_example():
    """§3.2: 256 bits, H(0), CNOT(0,2) (span 3 -> U(8) embedding), printed at 8 digits."""
    p = 256
    m = oracle.OracleMPS(3, p, 8, 2.0 ** -128)
    psi = cplx(m.to_dense())
    rho = partial_trace_dense(psi, 3, [0, 1, 2])
    assert showb(rho, 3) == GOLDEN[0]
    m.apply(gen.const_gate(p, "H"), [0])
    m.apply(gen.const_gate(p, "CNOT"), [0, 2])
    psi = cplx(m.to_dense())
    rho = partial_trace_dense(psi, 3, [0, 2])
    assert showb(rho, 2) == GOLDEN[1]
    # bond dims 2,2 with V = [1/sqrt2, 1/sqrt2]
    assert m.bond_dims() == [2, 2]
    with mpmath.workprec(p):
        for b in range(2):
            for v in reals(m.schmidt(b)):
                assert abs(v - 1 / mpmath.sqrt(2)) <= mpmath.mpf(2) ** (-p + 4)


def test_dense_closed_forms_ghz_qft():
    p = 280
    n = 5
    H, CX = gen.const_gate(p, "H"), gen.const_gate(p, "CNOT")
    ghz = [(H, (0,))] + [(CX, (s, s + 1)) for s in range(n - 1)]
    psi = dense_of(ghz, n, p)
    with mpmath.workprec(p):
        want = [0] * (1 << n)
        want[0] = want[-1] = 1 / mpmath.sqrt(2)
    assert normwise_err(psi, want) <= tau(p)
    # nearest-neighbour QFT network on basis input x: amp(y) = 2^(-n/2) e^{2 pi i x y / 2^n}
    n = 4
    for x in (0, 1, 6, 13):
        gates = []
        for q in range(n):
            if (x >> (n - 1 - q)) & 1:
                gates.append((gen.const_gate(p, "X"), (q,)))
        for j in range(n):
            gates.append((H, (0,)))
            for mm in range(n - 1 - j):
                gates.append((gen.phase_swap_gate(p, mm), (mm, mm + 1)))
        psi = dense_of(gates, n, p)
        with mpmath.workprec(p + 32):
            want = [mpmath.expjpi(mpmath.mpf(2 * x * y) / 2 ** n) / mpmath.sqrt(2 ** n) for y in range(1 << n)]
        assert normwise_err(psi, want) <= tau(p)


def test_mps_vs_dense_config1():
    """BASELINE configs[0]: n=8, depth 8 Haar U(4) brick-wall, chi_max=16 (never binds),
    280 bits — all 256 amplitudes against the dense 2^8 state vector."""
    n, p, chi, thr, gates = gen.config_circuit(0)
    m = mps_of(gates, n, p, chi, thr)
    assert normwise_err(cplx(m.to_dense()), dense_of(gates, n, p)) <= tau(p)
    assert m.bond_dims() == [2, 4, 8, 16, 8, 4, 2]
    # norm preservation (non-truncating run)
    with mpmath.workprec(p):
        assert abs(reals(m.norm2())[0] - 1) <= mpmath.mpf(2) ** (-p + 20)
    # Schmidt form (Eq. 2): eigenvalues of rho_{0..s} = lambda_s^2, checked via sum lambda^2 = 1
    for b in range(n - 1):
        lam = reals(m.schmidt(b))
        with mpmath.workprec(p):
            assert abs(mpmath.fsum(x ** 2 for x in lam) - 1) <= mpmath.mpf(2) ** (-p + 16)
            assert all(lam[i] >= lam[i + 1] for i in range(len(lam) - 1))


@pytest.mark.parametrize("p", [256, 512])
def test_mps_vs_dense_mixed_gates(p):
    """U(2), U(4), U(8) and span-3 two-qubit gates on n=6 vs the dense simulator."""
    n = 6
    gates = [(gen.haar_unitary(p, 2, 91, 0, q), (q,)) for q in range(n)]
    gates += [(gen.haar_unitary(p, 4, 91, 1, s), (s, s + 1)) for s in (0, 2, 4)]
    gates += [(gen.haar_unitary(p, 8, 91, 2, 1), (1, 2, 3))]
    gates += [(gen.haar_unitary(p, 4, 91, 3, 2), (2, 4))]
    gates += [(gen.haar_unitary(p, 4, 91, 4, s), (s, s + 1)) for s in (1, 3)]
    gates += [(gen.haar_unitary(p, 8, 91, 5, 3), (3, 4, 5))]
    thr = 2.0 ** -(p // 2)
    m = mps_of(gates, n, p, 64, thr)
    assert normwise_err(cplx(m.to_dense()), dense_of(gates, n, p)) <= tau(p)


def test_schmidt_values_equal_dense_spectrum():
    """Eq. 2: V_s are the square roots of the eigenvalues of rho_{0..s}."""
    p = 256
    n = 5
    gates = gen.brickwall(n, 4, p, 92)
    m = mps_of(gates, n, p, 32, 2.0 ** -128)
    psi = dense_of(gates, n, p)
    for s in range(n - 1):
        # reshape psi to 2^(s+1) x 2^(n-s-1) and take its singular values
        rows = 1 << (s + 1)
        cols = 1 << (n - s - 1)
        with mpmath.workprec(p + 64):
            Mx = mpmath.matrix([[psi[r * cols + c] for c in range(cols)] for r in range(rows)])
            sv = sorted([x for x in mpmath.svd_c(Mx, compute_uv=False)], reverse=True)
            lam = reals(m.schmidt(s))
            assert len(lam) == sum(1 for x in sv if x > mpmath.mpf(2) ** (-p // 2))
            for a, b in zip(lam, sv):
                assert abs(a - b) <= tau(p)


def test_ghz_mps_n10():
    p = 280
    n = 10
    H, CX = gen.const_gate(p, "H"), gen.const_gate(p, "CNOT")
    m = oracle.OracleMPS(n, p, 4, 2.0 ** -140)
    m.apply(H, [0])
    for s in range(n - 1):
        m.apply(CX, [s, s + 1])
    assert m.bond_dims() == [2] * (n - 1)
    with mpmath.workprec(p):
        for b in range(n - 1):
            for v in reals(m.schmidt(b)):
                assert abs(v - 1 / mpmath.sqrt(2)) <= tau(p)
        for bits, want in (([0] * n, 1 / mpmath.sqrt(2)), ([1] * n, 1 / mpmath.sqrt(2)), ([1] + [0] * (n - 1), 0)):
            a = cplx(m.amplitude(bits))[0]
            assert abs(a - want) <= tau(p)


def test_qft_mps_rank_one():
    """QFT of a basis state through the MPS: chi stays 1 (rank-1 Theta), amplitudes closed form."""
    p = 280
    n = 6
    x = 0b101101
    m = oracle.OracleMPS(n, p, 8, 2.0 ** -140)
    for q in range(n):
        if (x >> (n - 1 - q)) & 1:
            m.apply(gen.const_gate(p, "X"), [q])
    for j in range(n):
        m.apply(gen.const_gate(p, "H"), [0])
        for mm in range(n - 1 - j):
            m.apply(gen.phase_swap_gate(p, mm), [mm, mm + 1])
    assert m.bond_dims() == [1] * (n - 1)
    with mpmath.workprec(p + 32):
        want = [mpmath.expjpi(mpmath.mpf(2 * x * y) / 2 ** n) / mpmath.sqrt(2 ** n) for y in range(1 << n)]
    assert normwise_err(cplx(m.to_dense()), want) <= tau(p)


def test_echo_returns_to_zero_state():
    """Depth-d Haar brick-wall then its inverse: |0...0> exactly (chi_max >= 2^d)."""
    p = 280
    n, d = 8, 3
    gates = gen.brickwall(n, d, p, 93)
    m = oracle.OracleMPS(n, p, 8, 2.0 ** -140)
    for U, s in gates:
        m.apply(U, s)
    for U, s in reversed(gates):
        u = cplx(U)
        D = 1 << len(s)
        with mpmath.workprec(p):
            Uh = [mpmath.conj(u[c * D + r]) for r in range(D) for c in range(D)]
        m.apply(R.cplx_from_values(p, [(z.real, z.imag) for z in Uh]), s)
    a = cplx(m.amplitude([0] * n))[0]
    assert abs(a - 1) <= tau(p)
    assert m.bond_dims() == [1] * (n - 1)


def test_truncation_eckart_young_and_renorm():
    """Sum of dropped sigma^2 = ||Theta' - X_k S_k V_k^H||_F^2; kept lambda renormalised."""
    p = 256
    chi = 4
    A, B, U = gen.update_batch_inputs(p, chi, 1)
    out = oracle.update2_batch(p, 1, chi, chi, chi, chi, 2.0 ** -128, A, B, U, want_theta=True)
    k = int(out["k"][0])
    assert k == chi
    sig = reals(out["sigma"])
    lam = reals(out["lam"][:k])
    with mpmath.workprec(p):
        nu = mpmath.sqrt(mpmath.fsum(s ** 2 for s in sig[:k]))
        for a, s in zip(lam, sig):
            assert abs(a - s / nu) <= mpmath.mpf(2) ** (-p + 4)
        assert abs(mpmath.fsum(x ** 2 for x in lam) - 1) <= mpmath.mpf(2) ** (-p + 8)
    # sum sigma^2 = ||Theta'||_F^2
    th = cplx(out["theta"])
    with mpmath.workprec(p + 32):
        f2 = mpmath.fsum(abs(z) ** 2 for z in th)
        assert abs(mpmath.fsum(s ** 2 for s in sig) - f2) / f2 <= mpmath.mpf(2) ** (-p + 16)
    # Eckart-Young: the kept factors are the best rank-k approximation, so the residual of
    # X_k S_k V_k^H = nu Gamma_A' diag(lambda') Gamma_B' (lambda_l = lambda_r = 1) carries
    # exactly the dropped weight; keeping any other k columns would leave more.  Theta' is
    # column-major 2chi x 2chi (rows (i, a), columns (j, c)).
    N = 2 * chi
    GL = cplx(out["GL"])  # [2][chi][chi_max]
    GR = cplx(out["GR"])  # [2][chi_max][chi]
    with mpmath.workprec(2 * p):
        res2 = mpmath.mpf(0)
        for c in range(N):
            j, g = divmod(c, chi)
            for r in range(N):
                i, a = divmod(r, chi)
                approx = nu * mpmath.fsum(GL[(i * chi + a) * chi + b] * lam[b] * GR[(j * chi + b) * chi + g]
                                          for b in range(k))
                res2 += abs(th[c * N + r] - approx) ** 2
        dropped = mpmath.fsum(s ** 2 for s in sig[k:])
        assert dropped > mpmath.mpf(2) ** -20 * f2  # the cut removes real weight
        assert abs(res2 - dropped) <= mpmath.mpf(2) ** (-p + 16) * f2, (res2, dropped)
        # and it is the SMALLEST possible residual: the dropped sigma are the N - k smallest
        assert min(sig[:k]) >= max(sig[k:])


def test_expectation_vs_dense():
    p = 256
    n = 5
    gates = gen.brickwall(n, 3, p, 94)
    m = mps_of(gates, n, p, 32, 2.0 ** -128)
    psi = dense_of(gates, n, p)
    O = gen.haar_unitary(p, 4, 94, 99)  # any matrix works for <psi|O|psi>
    val, raw = m.expect(O, [2, 3])
    o = cplx(O)
    with mpmath.workprec(p + 32):
        acc = mpmath.mpc(0)
        for x in range(1 << n):
            bx = (x >> 1) & 3  # qubits 2,3 of n=5 -> bits 2,1
            for yp in range(4):
                y = (x & ~(3 << 1)) | (yp << 1)
                acc += mpmath.conj(psi[x]) * o[bx * 4 + yp] * psi[y]
        got = cplx(val)[0]
        assert abs(got - acc) <= tau(p)


def test_errors():
    p = 256
    m = oracle.OracleMPS(4, p, 4, 2.0 ** -128)
    bad = gen.const_gate(p, "H").copy()
    bad["exp"][0] += 1  # entry doubled -> not unitary
    with pytest.raises(oracle.OracleError) as e:
        m.apply(bad, [1])
    assert e.value.rc == -2
    with pytest.raises(oracle.OracleError) as e:
        m.apply(gen.const_gate(p, "CNOT"), [2, 2])  # repeated qubit
    assert e.value.rc == -1
    with pytest.raises(oracle.OracleError) as e:
        m.apply(gen.const_gate(p, "CNOT"), [0, 4])  # out of range
    assert e.value.rc == -1
    with pytest.raises(oracle.OracleError):
        oracle.OracleMPS(0, p, 4, 1e-10)


# ---------------------------------------------------------------- general placement (R18)
def routed_circuit(p, n, seed):
    """Gates on chosen qubits in any order and at any distance (P:331-333 applyU on chosen
    qubits; the n factor of O(g n m^3)): reversed pairs, spans 3..n, U(8) on
    scattered and permuted triples, mixed with local gates."""
    g = []
    g += [(gen.haar_unitary(p, 2, seed, 0, q), (q,)) for q in range(n)]
    g += [(gen.haar_unitary(p, 4, seed, 1, 0), (3, 0))]          # reversed, span 4
    g += [(gen.haar_unitary(p, 4, seed, 2, 0), (1, n - 1))]      # long range
    g += [(gen.haar_unitary(p, 4, seed, 3, 0), (5, 4))]          # reversed adjacent
    g += [(gen.haar_unitary(p, 4, seed, 4, 0), (4, 2))]          # reversed span 3 (U(8) embedding)
    g += [(gen.haar_unitary(p, 8, seed, 5, 0), (0, 3, n - 1))]   # scattered triple
    g += [(gen.haar_unitary(p, 8, seed, 6, 0), (4, 1, 2))]       # permuted, not consecutive
    g += [(gen.haar_unitary(p, 8, seed, 7, 0), (3, 2, 4))]       # permuted consecutive
    g += [(gen.const_gate(p, "CNOT"), (n - 1, 1))]
    return g


@pytest.mark.parametrize("p", [256, 512])
def test_general_placement_vs_dense(p):
    """Routed / reordered gates on the oracle MPS (no truncation) equal the dense simulator,
    which applies every gate directly on its qubits (a different code path)."""
    n = 7
    gates = routed_circuit(p, n, 93)
    m = mps_of(gates, n, p, 128, 2.0 ** -(p // 2))
    assert normwise_err(cplx(m.to_dense()), dense_of(gates, n, p)) <= tau(p)


def test_general_placement_reversed_equals_permuted():
    """U on (b, a) equals (SWAP U SWAP) on (a, b), up to rounding."""
    p, n = 256, 4
    U = gen.haar_unitary(p, 4, 94, 0, 0)
    perm = [0, 2, 1, 3]  # W = SWAP U SWAP (exact entry permutation)
    W = np.empty_like(U)
    for x in range(4):
        for y in range(4):
            W[2 * (4 * x + y)] = U[2 * (4 * perm[x] + perm[y])]
            W[2 * (4 * x + y) + 1] = U[2 * (4 * perm[x] + perm[y]) + 1]
    pre = [(gen.haar_unitary(p, 2, 94, 1, q), (q,)) for q in range(n)]
    a = mps_of(pre + [(U, (2, 0))], n, p, 16, 2.0 ** -64)
    b = mps_of(pre + [(W, (0, 2))], n, p, 16, 2.0 ** -64)
    assert normwise_err(cplx(a.to_dense()), cplx(b.to_dense())) <= tau(p)


def test_theta2_is_the_updates_contraction():
    """orc_theta2 (contraction + gate only, used for full-size samples) equals the Theta' the
    oracle's full update computes."""
    p, chi = 256, 3
    A, B, U = gen.update_batch_inputs(p, chi, 1)
    want = oracle.update2_batch(p, 1, chi, chi, chi, chi, 2.0 ** -128, A, B, U, want_theta=True)["theta"]
    got = oracle.theta2(p, chi, chi, chi, A, B, U)
    assert got.tobytes() == want.tobytes()
