import json, sys, os
import numpy as np, mpmath
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import records as R
from tests.helpers import reals
a, b = json.load(open(sys.argv[1])), json.load(open(sys.argv[2]))
p = a["p"]
with mpmath.workprec(2 * p):
    for la, lb in zip(a["layers"], b["layers"]):
        worst = (0, None)
        for bond, (x, y) in enumerate(zip(la["schmidt"], lb["schmidt"])):
            ra = reals(np.frombuffer(bytes.fromhex(x), dtype=R.record_dtype(p)))
            rb = reals(np.frombuffer(bytes.fromhex(y), dtype=R.record_dtype(p)))
            if len(ra) != len(rb):
                print("layer", la["layer"], "bond", bond, "dims differ", len(ra), len(rb)); continue
            d = [(abs(u - v), i) for i, (u, v) in enumerate(zip(ra, rb))]
            if d:
                e, i = max(d)
                if e > worst[0]: worst = (e, (bond, i, len(ra), float(ra[i]), float(rb[i])))
        print("layer", la["layer"], "sites", la["sites"], "dims", la["dims"], "worst diff %.3e" % float(worst[0]), worst[1])
