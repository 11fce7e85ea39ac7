import sys, numpy as np, mpmath
sys.path.insert(0, '/root/repo')
import paper_1111_3124_b200 as m
import oracle
from synth import gen, records as R
from tests.helpers import cplx, reals
P = 512; N = 8; x = 0b10011101
om = oracle.OracleMPS(N, P, 4, 2.0 ** -(P//2))
gates = []
for q in range(N):
    if (x >> (N - 1 - q)) & 1: gates.append((gen.const_gate(P, "X"), [q]))
gates.append((gen.const_gate(P, "H"), [0]))
for mm in range(2):
    gates.append((gen.phase_swap_gate(P, mm), [mm, mm + 1]))
for U, s in gates: om.apply(U, s)
A, _, _ = om.get_site(2); B, _, _ = om.get_site(3)
U = gen.phase_swap_gate(P, 2)
print("A", R.cplx_to_complex128(A), "B", R.cplx_to_complex128(B))
th_g = m.update_batch(P, 1, 1, A, B, U, theta=True)["theta"]
th_w = oracle.update2_batch(P, 1, 1, 1, 1, 1, 2.0**-256, A, B, U, want_theta=True)["theta"]
with mpmath.workprec(2*P):
    print("theta gpu", [complex(z) for z in cplx(th_g)])
    print("theta err", [float(abs(a-b)) for a, b in zip(cplx(th_g), cplx(th_w))])
sig, sw, rps, rc = m.svd_batch(P, 2, 2, 1, th_w)
print("svd(oracle theta) rc", rc, sw, rps[0][:6], [float(v) for v in reals(sig)])
sig, sw, rps, rc = m.svd_batch(P, 2, 2, 1, th_g)
print("svd(gpu theta) rc", rc, sw, rps[0][:6], [float(v) for v in reals(sig)])
for PP in (280, 512):
    T = th_w if PP == 512 else None
print("U", R.cplx_to_complex128(U))
# probe debug mpf ops on the U entries
for op in ("fixed", "copy"):
    out = m.debug_mpf(P, op, U)
    with mpmath.workprec(2*P):
        print(op, [float(abs(a-b)) for a, b in zip(reals(out), reals(U))])
