"""The routed circuit up to gate `upto` on the oracle, loaded into the GPU state, then the
next gate on both — development tool."""
import sys
import mpmath
sys.path.append('.')
import oracle
import paper_1111_3124_b200 as M
from tests.test_oracle_tebd import routed_circuit
from tests.helpers import cplx, normwise_err, reals
p = int(sys.argv[1]) if len(sys.argv) > 1 else 512
upto = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n = 7
g = routed_circuit(p, n, 95)
om = oracle.OracleMPS(n, p, 128, 2.0 ** -(p // 2))
for U, s in g[:upto]:
    om.apply(U, s)
st = M.MPS(n, p, 128, 2.0 ** -(p // 2))
for b in range(n - 1):
    st.set_schmidt(b, om.schmidt(b))
for s in range(n):
    G, ml, mr = om.get_site(s)
    st.set_site(s, G, ml, mr)
with mpmath.workprec(2 * p):
    print("loaded", mpmath.nstr(normwise_err(cplx(st.to_dense()), cplx(om.to_dense())), 3))
    for b in range(n - 1):
        print(" lam", b, [mpmath.nstr(x, 3) for x in reals(om.schmidt(b))])
    U, s = g[upto]
    st.apply(U, s)
    om.apply(U, s)
    print("gate", s, st.bond_dims(), om.bond_dims())
    for b in range(n - 1):
        a, w = reals(st.schmidt(b)), reals(om.schmidt(b))
        print("  bond", b, mpmath.nstr(max(abs(x - y) for x, y in zip(a, w)), 3), [mpmath.nstr(x, 3) for x in w])
    print("  amplitudes", mpmath.nstr(normwise_err(cplx(st.to_dense()), cplx(om.to_dense())), 3))
    print("  norm2", mpmath.nstr(reals(st.norm2())[0] - 1, 3), mpmath.nstr(reals(om.norm2())[0] - 1, 3))

# gauge-fixed site comparison: phases fixed per bond index from the oracle's largest entry
def site(m, s):
    G, ml, mr = m.get_site(s)
    v = cplx(G)
    return [[[v[(i * ml + a) * mr + b] for b in range(mr)] for a in range(ml)] for i in range(2)], ml, mr

with mpmath.workprec(2 * p):
    S = {s: (site(st, s), site(om, s)) for s in (2, 3, 4)}
    # bond 3 phases from site 4 rows b; bond 2 phases from site 2 columns a
    (g4, ml4, mr4), (o4, _, _) = S[4]
    ph3 = []
    for b in range(ml4):
        i, c = max(((i, c) for i in range(2) for c in range(mr4)), key=lambda t: abs(o4[t[0]][b][t[1]]))
        ph3.append(g4[i][b][c] / o4[i][b][c])
    e4 = max(abs(g4[i][b][c] / ph3[b] - o4[i][b][c]) for i in range(2) for b in range(ml4) for c in range(mr4))
    (g2, ml2, mr2), (o2, _, _) = S[2]
    ph2 = []
    for b in range(mr2):
        i, a = max(((i, a) for i in range(2) for a in range(ml2)), key=lambda t: abs(o2[t[0]][t[1]][b]))
        ph2.append(g2[i][a][b] / o2[i][a][b])
    e2 = max(abs(g2[i][a][b] / ph2[b] - o2[i][a][b]) for i in range(2) for a in range(ml2) for b in range(mr2))
    (g3, ml3, mr3), (o3, _, _) = S[3]
    e3 = max(abs(g3[i][a][b] * ph2[a] / ph3[b] - o3[i][a][b]) for i in range(2) for a in range(ml3) for b in range(mr3))
    print("gauge-fixed site errors: G2", mpmath.nstr(e2, 3), "G3", mpmath.nstr(e3, 3), "G4", mpmath.nstr(e4, 3))
    print("phase moduli", [mpmath.nstr(abs(x) - 1, 3) for x in ph2 + ph3])
