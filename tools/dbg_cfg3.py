"""Amplitude / Schmidt errors of a cached-oracle config run (max over bits), for comparing
builds — development tool.  usage: dbg_cfg3.py golden.json"""
import json
import sys
import mpmath
sys.path.append('.')
import paper_1111_3124_b200 as m
from synth import gen
from tests.helpers import cplx, reals
from tests.test_gpu_configs import from_hex, layers_of
g = json.load(open(sys.argv[1]))
n, p, chi, thr, gates = gen.config_circuit(g["config"], depth=g["depth"], chi_max=g.get("chi_override"))
st = m.MPS(n, p, chi, thr)
for layer in layers_of(gates):
    st.apply_layer(layer)
print(m.__file__, st.bond_dims() == g["bond_dims"])
with mpmath.workprec(2 * p):
    es = max(max(abs(x - y) for x, y in zip(reals(st.schmidt(b)), reals(from_hex(p, g["schmidt"][b])))) for b in range(n - 1))
    ga = [cplx(st.amplitude(bits))[0] for bits in g["bits"]]
    wa = [cplx(from_hex(p, h))[0] for h in g["amplitudes"]]
    e = max(abs(x - y) for x, y in zip(ga, wa)) / max(max(abs(y) for y in wa), mpmath.mpf(2) ** (-n / 2.0))
    print("schmidt", mpmath.nstr(es, 3), "amplitudes", mpmath.nstr(e, 3))
