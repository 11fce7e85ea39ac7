"""CPU checks of the graded-spectrum input generators and of the cached oracle goldens the GPU
parity tests compare with (tests/golden/cfg1_*.json, graded_*.json; written by
tools/make_cfg1_golden.py and tools/make_graded_golden.py, which call only oracle/).

  * the generators produce the singular values they claim (mpmath.svd_c, a third-party SVD);
  * the oracle's SVD / two-site update reproduces those known values on small graded inputs;
  * every cached golden is internally consistent: sigma descending, k = chi,
    lambda' = sigma_1..k / ||sigma_1..k||, sum lambda'^2 = 1."""
import glob
import json
import os

import mpmath
import numpy as np
import pytest

import oracle
from synth import gen
from synth import records as R
from tests.helpers import cplx, reals

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("p,dec", [(280, 40), (512, 80)])
def test_graded_matrix_has_the_claimed_sigma(p, dec):
    M = N = 8
    A, s = gen.graded_matrix(p, M, N, dec, 11, p)
    v = cplx(A)
    with mpmath.workprec(p + 64):
        a = mpmath.matrix([[v[c * M + r] for c in range(N)] for r in range(M)])
        got = sorted([mpmath.mpf(x) for x in mpmath.svd_c(a, compute_uv=False)], reverse=True)
        assert max(abs(x - y) for x, y in zip(got, s)) / s[0] <= mpmath.mpf(2) ** (-p + 8)
    # the oracle's Jacobi SVD on the same graded matrix
    sig, _, _, sw = oracle.svd(p, A, M, N)
    with mpmath.workprec(p + 64):
        o = sorted(reals(sig), reverse=True)
        assert max(abs(x - y) for x, y in zip(o, s)) / s[0] <= mpmath.mpf(2) ** (-p + 16)


@pytest.mark.parametrize("in_lambda", [True, False])
def test_graded_update_inputs_spectrum(in_lambda):
    p, chi, dec = 280, 4, 40
    A, B, lam, s = gen.graded_update_inputs(p, chi, dec, 12, in_lambda=in_lambda)
    o = oracle.update2_batch(p, 1, chi, chi, chi, chi, 0.0, A, B, gen.const_gate(p, "I4"), lam_m=lam)
    sg = reals(o["sigma"])
    with mpmath.workprec(p + 64):
        assert max(abs(x - y) for x, y in zip(sg[:chi], s)) / s[0] <= mpmath.mpf(2) ** (-p + 16)
        assert max(sg[chi:]) / s[0] <= mpmath.mpf(2) ** (-p + 16)  # Theta has rank chi


def _goldens():
    fs = sorted(glob.glob(os.path.join(GOLD, "cfg1_p*_chi*_item*.json")) +
                glob.glob(os.path.join(GOLD, "graded_upd_*.json")) +
                glob.glob(os.path.join(GOLD, "cfg5_p*_chi*_item*.json")))
    return fs


@pytest.mark.parametrize("f", _goldens(), ids=[os.path.basename(f) for f in _goldens()])
def test_cached_update_golden_consistent(f):
    g = json.load(open(f))
    p, chi, k = g["prec"], g["chi"], g["k"]
    dt = R.record_dtype(p)
    sig = reals(np.frombuffer(bytes.fromhex(g["sigma"]), dtype=dt))
    lam = reals(np.frombuffer(bytes.fromhex(g["lam"]), dtype=dt))
    assert len(sig) == 2 * chi and k == chi and len(lam) == chi
    if os.path.basename(f).startswith("cfg5_"):
        sig = sorted(sig, reverse=True)  # (stored in the oracle's output order)
    assert all(sig[i] >= sig[i + 1] for i in range(len(sig) - 1))
    with mpmath.workprec(2 * p):
        nu = mpmath.sqrt(mpmath.fsum(x * x for x in sig[:k]))
        assert max(abs(lam[i] - sig[i] / nu) for i in range(k)) <= mpmath.mpf(2) ** (-p + 8)
        assert abs(mpmath.fsum(x * x for x in lam) - 1) <= mpmath.mpf(2) ** (-p + 8)
    assert len(g["P_rows"]) * len(g["P_cols"]) * 2 == len(np.frombuffer(bytes.fromhex(g["P"]), dtype=dt))
    assert g["Pmax"] > 0 and 1 <= g["sweeps"] <= 60
