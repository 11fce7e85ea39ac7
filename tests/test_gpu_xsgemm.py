"""GEMM form of the refinement sweeps (R26) against the sequential application of the
same sweeps (MPS_XS_GEMM=0, R22): the same configs[1]-shaped items and a graded-spectrum item in
two subprocesses (the switch is read once per process).  Both forms only choose the starting
basis of the p-bit stage, which ends on the stopping criterion either way, so k must be equal
and sigma must agree to 2^-(p-24) sigma_1; the GEMM form must leave the p-bit stage as short as
the sequential one (1 sweep at 280 bits: the first-order finish or one certified k_jacobi sweep;
2 at 512 bits).  Both forms are compared with the oracle by the parity suites
(test_gpu_variants.py, test_gpu_cfg1_golden.py, test_gpu_graded.py run the default = GEMM form)."""
import json
import os
import subprocess
import sys
from fractions import Fraction

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, ".")
import paper_1111_3124_b200 as m
from synth import gen
from synth import records as R
res = {}
for p, chi, nb in ((280, 16, 8), (280, 64, 8), (280, 128, 3), (512, 32, 4)):
    A, B, U = gen.update_batch_inputs(p, chi, nb, first=9300)
    out = m.update_batch(p, chi, nb, A, B, U)
    sig = [str(R.to_fraction(r)) for r in out["sigma"]]
    res[f"{p}_{chi}"] = {"sigma": sig, "k": [int(x) for x in out["k"]], "sweeps": [int(x) for x in out["sweeps"]]}
print("JSON" + json.dumps(res))
"""


def _run(gemm: bool):
    env = dict(os.environ)
    env["MPS_XS_GEMM"] = "1" if gemm else "0"
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("JSON")][-1]
    return json.loads(line[4:])


@pytest.fixture(scope="module")
def both():
    return _run(True), _run(False)


def test_gemm_form_matches_sequential_sweeps(both):
    gf, seq = both
    for key, c in gf.items():
        r = seq[key]
        p, chi = (int(x) for x in key.split("_"))
        nb = len(c["k"])
        N = 2 * chi
        assert c["k"] == r["k"], key
        bound = Fraction(1, 2 ** (p - 24))
        worst = Fraction(0)
        for b in range(nb):
            sc = [Fraction(x) for x in c["sigma"][b * N:(b + 1) * N]]
            sr = [Fraction(x) for x in r["sigma"][b * N:(b + 1) * N]]
            err = max(abs(x - y) for x, y in zip(sc, sr)) / sr[0]
            assert err <= bound, (key, b, float(err))
            worst = max(worst, err)
        # the p-bit stage is no longer than after the sequential sweeps
        assert max(c["sweeps"]) <= max(r["sweeps"]), (key, c["sweeps"], r["sweeps"])
        print(f"xs gemm {key}: sweeps {sorted(set(c['sweeps']))} (sequential {sorted(set(r['sweeps']))}), "
              f"max |dsigma|/sigma_1 = {float(worst):.3e}")
