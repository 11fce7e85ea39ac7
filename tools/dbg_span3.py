"""Accuracy of span-3 / U(8) gates (GPU and oracle vs dense) on small circuits — development tool."""
import sys
import mpmath
sys.path.append('.')
import oracle
import paper_1111_3124_b200 as M
from synth import gen
from tests.helpers import cplx, normwise_err
p = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = 7
for seed in range(96, 100):
    g = [(gen.haar_unitary(p, 2, seed, 0, q), (q,)) for q in range(n)]
    g += [(gen.haar_unitary(p, 4, seed, 1, s), (s, s + 1)) for s in (0, 2, 4)]
    g += [(gen.haar_unitary(p, 4, seed, 2, s), (s, s + 1)) for s in (1, 3, 5)]
    g += [(gen.haar_unitary(p, 4, seed, 3, 2), (2, 4))]
    g += [(gen.haar_unitary(p, 8, seed, 4, 1), (1, 2, 3))]
    st = M.MPS(n, p, 128, 2.0 ** -(p // 2))
    om = oracle.OracleMPS(n, p, 128, 2.0 ** -(p // 2))
    d = oracle.OracleDense(n, p)
    out = []
    for U, s in g:
        st.apply(U, s); om.apply(U, s); d.apply(U, s)
        if len(s) > 1 and (len(s) == 3 or s[1] - s[0] == 2):
            want = cplx(d.state())
            out.append((s, mpmath.nstr(normwise_err(cplx(st.to_dense()), want), 3), mpmath.nstr(normwise_err(cplx(om.to_dense()), want), 3)))
    print(seed, st.bond_dims(), out, flush=True)
