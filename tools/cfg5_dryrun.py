"""Dry run of tests/test_gpu_cfg5_golden.py without goldens: the configs[4]-shaped windows through both
GPU paths (one mps_apply_layer of a 64-site 512-bit state, and mps_bench_update_batch), compared
with each other (k, lambda', the gauge-invariant P on a seeded grid).  GPU only; no oracle call.
  python tools/cfg5_dryrun.py [item ...]"""
import os, sys, time
import mpmath
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1111_3124_b200 as m  # noqa: E402
import make_cfg5_golden as mk  # noqa: E402  (the input recipe only)
from tests.helpers import p_sample, reals, tau  # noqa: E402

items = [int(x) for x in sys.argv[1:]] or [0, 3]
p, chi = 512, 256
t0 = time.time()
inp = {i: mk.inputs(i) for i in items}
print(f"inputs of {items}: {time.time() - t0:.1f} s", flush=True)
st = m.MPS(64, p, chi, 2.0 ** -256)
gates = []
for i in items:
    A, B, ll, lm, lr, U = inp[i]
    s = mk.ITEMS[i][1]
    st.set_schmidt(s - 1, ll); st.set_schmidt(s, lm); st.set_schmidt(s + 1, lr)
    st.set_site(s, A, chi, chi); st.set_site(s + 1, B, chi, chi)
    gates.append((U, (s, s + 1)))
t0 = time.time()
st.apply_layer(gates); st.sync()
print(f"mps_apply_layer of {len(gates)} gates: {time.time() - t0:.1f} s", flush=True)
for i in items:
    A, B, ll, lm, lr, U = inp[i]
    s = mk.ITEMS[i][1]
    lam = st.schmidt(s)
    GL, ml, mr = st.get_site(s)
    GR, ml2, mr2 = st.get_site(s + 1)
    t0 = time.time()
    out = m.update_batch(p, chi, 1, A, B, U, lam_l=ll, lam_m=lm, lam_r=lr, chi_max=chi, thr=2.0 ** -256)
    dt = time.time() - t0
    k = int(out["k"][0])
    rows, cols = mk.grid(i)
    with mpmath.workprec(2 * p):
        l1, l2 = reals(lam[:k]), reals(out["lam"][:k])
        e_l = max(abs(x - y) for x, y in zip(l1, l2)) / l2[0]
        P1 = reals(p_sample(p, chi, len(lam), GL, GR, lam, rows, cols, lam_l=ll, lam_r=lr))
        P2 = reals(p_sample(p, chi, k, out["GL"], out["GR"], out["lam"], rows, cols, lam_l=ll, lam_r=lr))
        pm = max(abs(x) for x in P2)
        e_p = max(abs(x - y) for x, y in zip(P1, P2)) / pm
    print(f"item {i}: k layer {len(lam)} batch {k} (dims {ml},{mr},{ml2},{mr2}), update_batch {dt:.1f} s, sweeps {int(out['sweeps'][0])}, "
          f"lambda diff {float(e_l):.2e}, P diff {float(e_p):.2e} (tau {float(tau(p)):.1e})", flush=True)
st.close()
