"""Three-site update accuracy: the same input state loaded into GPU and oracle, one U(8)
gate, then Schmidt vectors and amplitudes compared — development tool."""
import sys
import mpmath
sys.path.append('.')
import oracle
import paper_1111_3124_b200 as M
from synth import gen
from tests.helpers import cplx, normwise_err, reals
p = int(sys.argv[1]) if len(sys.argv) > 1 else 280
n = 7
seed = 96
g = [(gen.haar_unitary(p, 2, seed, 0, q), (q,)) for q in range(n)]
g += [(gen.haar_unitary(p, 4, seed, 1, s), (s, s + 1)) for s in (0, 2, 4)]
g += [(gen.haar_unitary(p, 4, seed, 2, s), (s, s + 1)) for s in (1, 3, 5)]
om = oracle.OracleMPS(n, p, 128, 2.0 ** -(p // 2))
for U, s in g:
    om.apply(U, s)
st = M.MPS(n, p, 128, 2.0 ** -(p // 2))
for b in range(n - 1):
    pass
# load the oracle state into the GPU state (exact copy of the records)
dims = om.bond_dims()
for b in range(n - 1):
    st.set_schmidt(b, om.schmidt(b))
for s in range(n):
    G, ml, mr = om.get_site(s)
    st.set_site(s, G, ml, mr)
with mpmath.workprec(2 * p):
    e0 = normwise_err(cplx(st.to_dense()), cplx(om.to_dense()))
    print("loaded state diff", mpmath.nstr(e0, 3))
    U8 = gen.haar_unitary(p, 8, seed, 9, 1)
    for name, U, sites in (("U4 (3,4)", gen.haar_unitary(p, 4, seed, 11, 2), (3, 4)), ("U8 (1,2,3)", U8, (1, 2, 3)), ("U4 (2,4)", gen.haar_unitary(p, 4, seed, 10, 2), (2, 4))):
        st.apply(U, sites)
        om.apply(U, sites)
        print(name, st.bond_dims(), om.bond_dims())
        for b in range(n - 1):
            a, w = reals(st.schmidt(b)), reals(om.schmidt(b))
            print("  bond", b, mpmath.nstr(max(abs(x - y) for x, y in zip(a, w)), 3))
        print("  amplitudes", mpmath.nstr(normwise_err(cplx(st.to_dense()), cplx(om.to_dense())), 3))
