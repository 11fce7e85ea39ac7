"""configs[4]-shaped pins at n = 64, 512 bits (cfg5 end-to-end parity is
pinned by closed forms): GHZ, the nearest-neighbour QFT of a basis state (2080 gates,
amp(y) = 2^-32 e^{2 pi i x y / 2^64}), and a depth-4 Haar echo (exactly |0...0>)."""
import mpmath
import numpy as np
import pytest

from synth import gen
from synth import records as R
from tests.helpers import cplx, tau

pytestmark = pytest.mark.gpu
N, P = 64, 512


def M():
    import paper_1111_3124_b200 as m
    return m


def test_ghz_64_512bit():
    st = M().MPS(N, P, 4, 2.0 ** -256)
    st.apply(gen.const_gate(P, "H"), [0])
    for s in range(N - 1):
        st.apply(gen.const_gate(P, "CNOT"), [s, s + 1])
    assert st.bond_dims() == [2] * (N - 1)
    with mpmath.workprec(2 * P):
        for bits, want in (([0] * N, 1 / mpmath.sqrt(2)), ([1] * N, 1 / mpmath.sqrt(2)), ([0] * 32 + [1] * 32, 0)):
            assert abs(cplx(st.amplitude(bits))[0] - want) <= tau(P)


def test_qft_basis_state_64_512bit():
    x = 0x9E3779B97F4A7C15  # basis input
    st = M().MPS(N, P, 4, 2.0 ** -256)
    X = gen.const_gate(P, "X")
    H = gen.const_gate(P, "H")
    for q in range(N):
        if (x >> (N - 1 - q)) & 1:
            st.apply(X, [q])
    phase = [gen.phase_swap_gate(P, mm) for mm in range(N - 1)]
    for j in range(N):
        st.apply(H, [0])
        for mm in range(N - 1 - j):
            st.apply(phase[mm], [mm, mm + 1])
    assert max(st.bond_dims()) == 1
    rng = np.random.default_rng(11)
    ys = [0, 1, (1 << 64) - 1] + [int(v) for v in rng.integers(0, 1 << 62, 5)]
    for y in ys:
        bits = [(y >> (N - 1 - q)) & 1 for q in range(N)]
        got = cplx(st.amplitude(bits))[0]
        with mpmath.workprec(P + 64):
            want = mpmath.expjpi(mpmath.mpf(2 * ((x * y) % (1 << 64))) / mpmath.mpf(2) ** 64) / mpmath.mpf(2) ** 32
            assert abs(got - want) <= tau(P) * mpmath.mpf(2) ** -32, (y, got, want)


def test_echo_64_512bit():
    d = 4
    gates = gen.brickwall(N, d, P, 4444)
    st = M().MPS(N, P, 16, 2.0 ** -256)
    t, cur = None, []
    layers = []
    for U, s in gates:
        if cur and s[0] < cur[-1][1][0]:
            layers.append(cur)
            cur = []
        cur.append((U, s))
    layers.append(cur)
    for layer in layers:
        st.apply_layer(layer)
    assert max(st.bond_dims()) == 2 ** (d // 2) * 2 or max(st.bond_dims()) <= 16
    for layer in reversed(layers):
        inv = []
        for U, s in layer:
            u = cplx(U)
            D = 1 << len(s)
            with mpmath.workprec(P):
                Uh = [mpmath.conj(u[c * D + r]) for r in range(D) for c in range(D)]
            inv.append((R.cplx_from_values(P, [(z.real, z.imag) for z in Uh]), s))
        st.apply_layer(inv)
    with mpmath.workprec(2 * P):
        assert abs(cplx(st.amplitude([0] * N))[0] - 1) <= tau(P)
    assert st.bond_dims() == [1] * (N - 1)
