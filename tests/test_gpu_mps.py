"""GPU MPS state (mps_init / mps_apply_gate / queries) against the oracle and the paper:
BASELINE configs[0] end to end vs the dense 2^8 state vector, U(2)/U(4)/U(8)/span-3 gates
vs dense, the §3.2 golden output, GHZ / QFT / echo closed forms, norm and expectation
values, a truncating run vs the oracle MPS, and the error contract."""
import mpmath
import numpy as np
import pytest

import oracle
from synth import gen
from synth import records as R
from tests.helpers import cplx, normwise_err, partial_trace_dense, reals, showb, tau

pytestmark = pytest.mark.gpu

GOLDEN = [l.rstrip("\n") for l in open(__file__.replace("test_gpu_mps.py", "golden/qc_simple_example.txt"))
          if not l.startswith("#")]


def M():
    import paper_1111_3124_b200 as m
    return m


def dense_of(gates, n, p):
    d = oracle.OracleDense(n, p)
    for U, s in gates:
        d.apply(U, s)
    return cplx(d.state())


def test_config1_vs_dense():
    n, p, chi, thr, gates = gen.config_circuit(0)
    st = M().MPS(n, p, chi, thr)
    for U, s in gates:
        st.apply(U, s)
    assert normwise_err(cplx(st.to_dense()), dense_of(gates, n, p)) <= tau(p)
    om = oracle.OracleMPS(n, p, chi, thr)
    for U, s in gates:
        om.apply(U, s)
    assert st.bond_dims() == om.bond_dims() == [2, 4, 8, 16, 8, 4, 2]
    with mpmath.workprec(2 * p):
        for b in range(n - 1):
            g, w = reals(st.schmidt(b)), reals(om.schmidt(b))
            assert max(abs(x - y) for x, y in zip(g, w)) <= tau(p)
        assert abs(reals(st.norm2())[0] - 1) <= mpmath.mpf(2) ** (-p + 20)


def test_layer_equals_sequential():
    n, p, chi, thr, gates = gen.config_circuit(0, depth=4)
    a = M().MPS(n, p, chi, thr)
    b = M().MPS(n, p, chi, thr)
    for U, s in gates:
        a.apply(U, s)
    layers = {}
    for i, (U, s) in enumerate(gates):
        layers.setdefault(s[0] % 2 if True else 0, [])
    # rebuild the brick-wall layers in order
    t, cur = 0, []
    for U, s in gates:
        if cur and s[0] < cur[-1][1][0]:
            b.apply_layer(cur)
            cur = []
        cur.append((U, s))
    b.apply_layer(cur)
    assert a.bond_dims() == b.bond_dims()
    x, y = cplx(a.to_dense()), cplx(b.to_dense())
    assert normwise_err(x, y) == 0  # same kernels, same per-gate decomposition: bitwise


@pytest.mark.parametrize("p", [256, 512])
def test_mixed_gates_vs_dense(p):
    n = 6
    gates = [(gen.haar_unitary(p, 2, 91, 0, q), (q,)) for q in range(n)]
    gates += [(gen.haar_unitary(p, 4, 91, 1, s), (s, s + 1)) for s in (0, 2, 4)]
    gates += [(gen.haar_unitary(p, 8, 91, 2, 1), (1, 2, 3))]
    gates += [(gen.haar_unitary(p, 4, 91, 3, 2), (2, 4))]
    gates += [(gen.haar_unitary(p, 4, 91, 4, s), (s, s + 1)) for s in (1, 3)]
    gates += [(gen.haar_unitary(p, 8, 91, 5, 3), (3, 4, 5))]
    st = M().MPS(n, p, 64, 2.0 ** -(p // 2))
    for U, s in gates:
        st.apply(U, s)
    assert normwise_err(cplx(st.to_dense()), dense_of(gates, n, p)) <= tau(p)


def test_paper_golden_on_gpu():
    p = 256
    st = M().MPS(3, p, 8, 2.0 ** -128)
    rho = partial_trace_dense(cplx(st.to_dense()), 3, [0, 1, 2])
    assert showb(rho, 3) == GOLDEN[0]
    st.apply(gen.const_gate(p, "H"), [0])
    st.apply(gen.const_gate(p, "CNOT"), [0, 2])
    rho = partial_trace_dense(cplx(st.to_dense()), 3, [0, 2])
    assert showb(rho, 2) == GOLDEN[1]
    assert st.bond_dims() == [2, 2]


@pytest.mark.parametrize("n", [10, 40])
def test_ghz(n):
    p = 280
    st = M().MPS(n, p, 4, 2.0 ** -140)
    st.apply(gen.const_gate(p, "H"), [0])
    for s in range(n - 1):
        st.apply(gen.const_gate(p, "CNOT"), [s, s + 1])
    assert st.bond_dims() == [2] * (n - 1)
    with mpmath.workprec(2 * p):
        for bits, want in (([0] * n, 1 / mpmath.sqrt(2)), ([1] * n, 1 / mpmath.sqrt(2)), ([1] + [0] * (n - 1), 0)):
            assert abs(cplx(st.amplitude(bits))[0] - want) <= tau(p)
        for b in range(n - 1):
            for v in reals(st.schmidt(b)):
                assert abs(v - 1 / mpmath.sqrt(2)) <= tau(p)


def test_qft_and_echo():
    p = 280
    n = 6
    x = 0b101101
    st = M().MPS(n, p, 8, 2.0 ** -140)
    for q in range(n):
        if (x >> (n - 1 - q)) & 1:
            st.apply(gen.const_gate(p, "X"), [q])
    for j in range(n):
        st.apply(gen.const_gate(p, "H"), [0])
        for mm in range(n - 1 - j):
            st.apply(gen.phase_swap_gate(p, mm), [mm, mm + 1])
    assert st.bond_dims() == [1] * (n - 1)
    with mpmath.workprec(p + 32):
        want = [mpmath.expjpi(mpmath.mpf(2 * x * y) / 2 ** n) / mpmath.sqrt(2 ** n) for y in range(1 << n)]
    assert normwise_err(cplx(st.to_dense()), want) <= tau(p)
    # echo
    n, d = 8, 3
    gates = gen.brickwall(n, d, p, 93)
    st = M().MPS(n, p, 8, 2.0 ** -140)
    for U, s in gates:
        st.apply(U, s)
    for U, s in reversed(gates):
        u = cplx(U)
        D = 1 << len(s)
        with mpmath.workprec(p):
            Uh = [mpmath.conj(u[c * D + r]) for r in range(D) for c in range(D)]
        st.apply(R.cplx_from_values(p, [(z.real, z.imag) for z in Uh]), s)
    with mpmath.workprec(2 * p):
        assert abs(cplx(st.amplitude([0] * n))[0] - 1) <= tau(p)
    assert st.bond_dims() == [1] * (n - 1)


def test_truncating_run_vs_oracle_mps():
    """chi_max binds (configs[2]-like, small): lambda on every bond and sampled amplitudes."""
    p = 280
    n, chi, thr = 10, 6, 1e-60
    gates = gen.brickwall(n, 6, p, 95, one_site_layer=True)
    st = M().MPS(n, p, chi, thr)
    om = oracle.OracleMPS(n, p, chi, thr)
    for U, s in gates:
        st.apply(U, s)
        om.apply(U, s)
    assert st.bond_dims() == om.bond_dims()
    with mpmath.workprec(2 * p):
        for b in range(n - 1):
            g, w = reals(st.schmidt(b)), reals(om.schmidt(b))
            assert max(abs(x - y) for x, y in zip(g, w)) <= tau(p)
    rng = np.random.default_rng(3)
    amps_g, amps_w = [], []
    for _ in range(12):
        bits = rng.integers(0, 2, n).tolist()
        amps_g.append(cplx(st.amplitude(bits))[0])
        amps_w.append(cplx(om.amplitude(bits))[0])
    amps_g.append(cplx(st.amplitude([0] * n))[0])
    amps_w.append(cplx(om.amplitude([0] * n))[0])
    with mpmath.workprec(2 * p):
        e = max(abs(a - b) for a, b in zip(amps_g, amps_w)) / max(max(abs(b) for b in amps_w), mpmath.mpf(2) ** (-n / 2))
    assert e <= tau(p)
    # norm of the stored (truncated) tensors agrees with the oracle's
    with mpmath.workprec(2 * p):
        assert abs(reals(st.norm2())[0] - reals(om.norm2())[0]) <= tau(p)


def test_expectation_vs_oracle():
    p = 256
    n = 5
    gates = gen.brickwall(n, 3, p, 94)
    st = M().MPS(n, p, 32, 2.0 ** -128)
    om = oracle.OracleMPS(n, p, 32, 2.0 ** -128)
    for U, s in gates:
        st.apply(U, s)
        om.apply(U, s)
    for sites, d in (([2, 3], 4), ([1], 2), ([0, 1, 2], 8)):
        O = gen.haar_unitary(p, d, 94, 99, d)
        g = cplx(st.expect(O, sites))[0]
        w = cplx(om.expect(O, sites)[0])[0]
        with mpmath.workprec(2 * p):
            assert abs(g - w) <= tau(p), (sites, g, w)


def test_error_contract():
    m = M()
    p = 256
    st = m.MPS(4, p, 4, 2.0 ** -128)
    bad = gen.const_gate(p, "H").copy()
    bad["exp"][0] += 1
    with pytest.raises(m.MpsError) as e:
        st.apply(bad, [1])
    assert e.value.rc == -2
    with pytest.raises(m.MpsError) as e:
        st.apply(gen.const_gate(p, "CNOT"), [2, 2])  # repeated qubit
    assert e.value.rc == -1
    with pytest.raises(m.MpsError) as e:
        st.apply(gen.const_gate(p, "CNOT"), [0, 4])  # out of range
    assert e.value.rc == -1
    with pytest.raises(m.MpsError) as e:
        st.apply_layer([(gen.const_gate(p, "CNOT"), (0, 1)), (gen.const_gate(p, "CNOT"), (1, 2))])
    assert e.value.rc == -5
    with pytest.raises(m.MpsError):
        m.MPS(0, p, 4)
    # the failed calls had no side effects
    assert st.bond_dims() == [1, 1, 1]


def rho_of(rec, k):
    v = cplx(rec)
    D = 1 << k
    return [[v[r * D + c] for c in range(D)] for r in range(D)]


def test_paper_golden_via_gpu_rdo():
    """§3.2 end to end on the GPU path: RDO_block(0,2) of |000>, then RDO({0,2}) after
    H(0), CNOT(0,2), printed at 8 digits."""
    p = 256
    st = M().MPS(3, p, 8, 2.0 ** -128)
    assert showb(rho_of(st.rdo([0, 1, 2]), 3), 3) == GOLDEN[0]
    st.apply(gen.const_gate(p, "H"), [0])
    st.apply(gen.const_gate(p, "CNOT"), [0, 2])
    assert showb(rho_of(st.rdo([0, 2]), 2), 2) == GOLDEN[1]


def test_rdo_vs_dense_partial_trace():
    p = 280
    n = 7
    gates = gen.brickwall(n, 4, p, 96, one_site_layer=True)
    st = M().MPS(n, p, 16, 2.0 ** -140)
    for U, s in gates:
        st.apply(U, s)
    psi = dense_of(gates, n, p)
    for keep in ([2], [0, 6], [1, 3, 4], [0, 1, 2, 3]):
        got = rho_of(st.rdo(keep), len(keep))
        want = partial_trace_dense(psi, n, keep)
        with mpmath.workprec(2 * p):
            tr = mpmath.fsum(want[i][i] for i in range(1 << len(keep)))
            err = max(abs(got[r][c] - want[r][c] / tr) for r in range(1 << len(keep)) for c in range(1 << len(keep)))
        assert err <= tau(p), (keep, err)


@pytest.mark.parametrize("p", [280, 512])
def test_general_placement_vs_oracle_and_dense(p):
    """Gates on chosen qubits in any order / at any distance (R18: reordering + exact SWAP
    routing) on the GPU MPS: equal to the dense simulator and to the oracle MPS, whose
    routing is implemented independently."""
    from tests.test_oracle_tebd import routed_circuit
    n = 7
    gates = routed_circuit(p, n, 95)
    st = M().MPS(n, p, 128, 2.0 ** -(p // 2))
    om = oracle.OracleMPS(n, p, 128, 2.0 ** -(p // 2))
    for U, s in gates:
        st.apply(U, s)
        om.apply(U, s)
    assert st.bond_dims() == om.bond_dims()
    want = dense_of(gates, n, p)
    assert normwise_err(cplx(st.to_dense()), want) <= tau(p)
    assert normwise_err(cplx(st.to_dense()), cplx(om.to_dense())) <= tau(p)
    # the same gates as disjoint layers (routed gates run one by one inside the layer)
    st2 = M().MPS(n, p, 128, 2.0 ** -(p // 2))
    layers = [[g] for g in gates[n:]]
    st2.apply_layer(gates[:n])
    for l in layers:
        st2.apply_layer(l)
    assert normwise_err(cplx(st2.to_dense()), want) <= tau(p)
