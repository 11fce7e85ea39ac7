import sys, numpy as np, mpmath
sys.path.insert(0, '/root/repo')
import paper_1111_3124_b200 as m
import oracle
from synth import gen, records as R
from tests.helpers import cplx, reals
P = int(sys.argv[1]); N = int(sys.argv[2]); d = int(sys.argv[3])
thr = 2.0 ** -(P // 2)
gates = gen.brickwall(N, d, P, 4444)
inv = []
for U, s in reversed(gates):
    u = cplx(U); D = 1 << len(s)
    with mpmath.workprec(P):
        Uh = [mpmath.conj(u[c * D + r]) for r in range(D) for c in range(D)]
    inv.append((R.cplx_from_values(P, [(z.real, z.imag) for z in Uh]), s))
st = m.MPS(N, P, 16, thr)
for g, (U, s) in enumerate(gates + inv):
    q = s[0]
    GL, a1, b1 = st.get_site(q); GR, a2, b2 = st.get_site(q + 1)
    ll = reals(st.schmidt(q - 1)) if q > 0 else [mpmath.mpf(1)]
    lm = reals(st.schmidt(q)); lr = reals(st.schmidt(q + 1)) if q + 1 < N - 1 else [mpmath.mpf(1)]
    try:
        st.apply(U, s)
    except Exception as e:
        print("fail gate", g, s, e, "dims", a1, b1, b2)
        Uc = cplx(U); gl = cplx(GL); gr = cplx(GR); cl, cm, cr = a1, b1, b2
        with mpmath.workprec(2 * P):
            Th = {}
            for i in range(2):
                for a in range(cl):
                    for j in range(2):
                        for c in range(cr):
                            Th[(i, a, j, c)] = mpmath.fsum(ll[a] * gl[(i * cl + a) * cm + b] * lm[b] * gr[(j * cm + b) * cr + c] * lr[c] for b in range(cm))
            vals = []
            for j in range(2):
                for c in range(cr):
                    for i in range(2):
                        for a in range(cl):
                            vals.append(mpmath.fsum(Uc[(2 * i + j) * 4 + 2 * ip + jp] * Th[(ip, a, jp, c)] for ip in range(2) for jp in range(2)))
        with mpmath.workprec(P):
            rec = R.cplx_from_values(P, [(+z.real, +z.imag) for z in vals])
        Mr, Nc = 2 * cl, 2 * cr
        sig, sw, rps, rc = m.svd_batch(P, Mr, Nc, 1, rec)
        print("gpu svd rc", rc, sw, rps[0][:20], [float(v) for v in reals(sig)])
        if Nc <= Mr:
            osig, _, _, osw = oracle.svd(P, rec, Mr, Nc)
            print("oracle sweeps", osw, sorted([float(v) for v in reals(osig)], reverse=True))
        np.save('/root/repo/gpurun_out/echo_fail_%d.npy' % P, rec)
        break
else:
    print("ok", st.bond_dims())
