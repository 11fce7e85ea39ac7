"""Per-gate error of the routed circuit (GPU and oracle vs dense) — development tool."""
import sys
import mpmath
sys.path.insert(0, '.')
import oracle
import paper_1111_3124_b200 as M
from tests.test_oracle_tebd import routed_circuit
from tests.helpers import cplx, normwise_err
p = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = 7
g = routed_circuit(p, n, 95)
st = M.MPS(n, p, 128, 2.0 ** -(p // 2))
om = oracle.OracleMPS(n, p, 128, 2.0 ** -(p // 2))
d = oracle.OracleDense(n, p)
for U, s in g:
    st.apply(U, s)
    om.apply(U, s)
    d.apply(U, s)
    want = cplx(d.state())
    print(s, st.bond_dims(), mpmath.nstr(normwise_err(cplx(st.to_dense()), want), 4),
          mpmath.nstr(normwise_err(cplx(om.to_dense()), want), 4), flush=True)
