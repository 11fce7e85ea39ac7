"""A/B of two builds / switches on a configs[4] prefix (no oracle data exists at chi = 256, 512 bits): run
the first `depth` layers, dump every Schmidt vector; `cmp` compares two dumps normwise.
  python tools/cfg4_ab.py run <depth> <out.json>;  python tools/cfg4_ab.py cmp <a.json> <b.json>"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import gen, records as R  # noqa: E402


def layers_of(gates):
    out, cur, used = [], [], set()
    for U, s in gates:
        span = set(range(s[0], s[-1] + 1))
        if span & used:
            out.append(cur); cur, used = [], set()
        cur.append((U, s)); used |= span
    if cur:
        out.append(cur)
    return out


if sys.argv[1] == "run":
    import paper_1111_3124_b200 as m
    depth, out = int(sys.argv[2]), sys.argv[3]
    n, p, chi, thr, gates = gen.config_circuit(4, depth=depth)
    st = m.MPS(n, p, chi, thr)
    t0 = time.time()
    for layer in layers_of(gates):
        st.apply_layer(layer)
    st.sync()
    dt = time.time() - t0
    json.dump({"p": p, "seconds": dt, "dims": st.bond_dims(),
               "schmidt": [bytes(st.schmidt(b).tobytes()).hex() for b in range(n - 1)]}, open(out, "w"))
    print(f"depth {depth}: {dt:.1f} s, max bond {max(st.bond_dims())}")
else:
    import mpmath
    from tests.helpers import reals, tau
    a, b = json.load(open(sys.argv[2])), json.load(open(sys.argv[3]))
    p = a["p"]
    assert a["dims"] == b["dims"], "bond dimensions differ"
    worst = 0
    with mpmath.workprec(2 * p):
        for x, y in zip(a["schmidt"], b["schmidt"]):
            ra = reals(np.frombuffer(bytes.fromhex(x), dtype=R.record_dtype(p)))
            rb = reals(np.frombuffer(bytes.fromhex(y), dtype=R.record_dtype(p)))
            worst = max(worst, max(abs(u - v) for u, v in zip(ra, rb)))
        print(f"seconds {a['seconds']:.1f} vs {b['seconds']:.1f}; max bond {max(a['dims'])}; "
              f"max |lambda_a - lambda_b| = {float(worst):.3e} (tau {float(tau(p)):.1e})")
