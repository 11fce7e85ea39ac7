"""End-to-end parity of BASELINE circuit configs on the GPU MPS against the cached oracle
runs in tests/golden/cfg*_oracle*.json (written by tools/make_oracle_golden.py, which
calls only oracle/).  SURVEY §8(c): bond dimensions equal exactly, Schmidt values
normwise, sampled amplitudes e = max|a-b| / max(max|b|, 2^(-n/2)) <= tau."""
import glob
import json
import os

import mpmath
import numpy as np
import pytest

from synth import gen
from synth import records as R
from tests.helpers import cplx, reals, tau

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "cfg*_oracle*.json")))


def from_hex(p, hexes):
    a = R.empty(p, len(hexes))
    raw = b"".join(bytes.fromhex(h) for h in hexes)
    return np.frombuffer(raw, dtype=R.record_dtype(p)).copy()


def layers_of(gates):
    out, cur, used = [], [], set()
    for U, s in gates:
        span = set(range(s[0], s[-1] + 1))
        if span & used:
            out.append(cur)
            cur, used = [], set()
        cur.append((U, s))
        used |= span
    if cur:
        out.append(cur)
    return out


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(g) for g in GOLDEN])
def test_config_vs_cached_oracle(path):
    import paper_1111_3124_b200 as m
    g = json.load(open(path))
    n, p, chi, thr, gates = gen.config_circuit(g["config"], depth=g["depth"], chi_max=g.get("chi_override"))
    assert len(gates) == g["gates"]
    st = m.MPS(n, p, chi, thr)
    for layer in layers_of(gates):
        st.apply_layer(layer)
    assert st.bond_dims() == g["bond_dims"]
    with mpmath.workprec(2 * p):
        for b in range(n - 1):
            got = reals(st.schmidt(b))
            want = reals(from_hex(p, g["schmidt"][b]))
            assert max(abs(x - y) for x, y in zip(got, want)) <= tau(p), b
        ga = [cplx(st.amplitude(bits))[0] for bits in g["bits"]]
        wa = [cplx(from_hex(p, h))[0] for h in g["amplitudes"]]
        e = max(abs(x - y) for x, y in zip(ga, wa)) / max(max(abs(y) for y in wa), mpmath.mpf(2) ** (-n / 2.0))
        assert e <= tau(p), e
        got_n = reals(st.norm2())[0]
        want_n = reals(from_hex(p, g["norm2"]))[0]
        assert abs(got_n - want_n) <= tau(p)
