"""Graded spectra on the GPU against cached ORACLE runs and the known singular values
(VERDICT r01 "What's weak" 2: no GPU test fed a known graded spectrum).

Inputs (synth.gen, seeded): A = W diag(s) Z^H with Householder isometries W, Z and
s_b = 10^(-decades b / (N - 1)), 60 decades at 280 bits and 120 at 512 bits.  One-sided
Jacobi SVD, truncation and split (P:258-263,
P:272-273), tolerance tau normwise (§8(c) ledger #12):

  * mps_svd_batch (the p-bit Jacobi kernel alone, N = 64, 128): sigma vs the oracle's and vs s;
  * the full two-site update through mps_bench_update_batch (contraction, binary64
    preconditioner R19, Newton-Schulz, p-bit Jacobi with the certified stop R21, V recovery
    or accumulation R16, truncation, split) with Theta = W diag(s) Z^H:
      "lam": s is the middle Schmidt vector (the V-recovery decision predicts a wide spectrum
             and accumulates V),
      "gam": s is folded into Gamma_A and lambda_m = 1 (the prediction says narrow, the
             device check of sigma_1 / sigma_k must catch it and re-run with accumulated V);
    sigma, k, lambda' and the gauge-invariant P = X_k diag(lambda') V_k^H vs the oracle.
"""
import glob
import json
import os

import mpmath
import numpy as np
import pytest

from synth import gen
from synth import records as R
from tests.helpers import p_sample, reals, tau

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _m():
    import paper_1111_3124_b200 as m
    return m


def recs(p, h):
    return np.frombuffer(bytes.fromhex(h), dtype=R.record_dtype(p)).copy()


SVD = [json.load(open(f)) for f in sorted(glob.glob(os.path.join(GOLD, "graded_svd_p*_N*.json")))]
UPD = [json.load(open(f)) for f in sorted(glob.glob(os.path.join(GOLD, "graded_upd_p*_chi*.json")))]


@pytest.mark.skipif(not SVD, reason="no cached graded SVD")
@pytest.mark.parametrize("g", SVD, ids=[f"p{g['prec']}_N{g['N']}" for g in SVD])
def test_graded_svd_vs_oracle_and_known_sigma(g):
    p, N = g["prec"], g["N"]
    A, s = gen.graded_matrix(p, N, N, g["decades"], *g["key"])
    sig, sw, rps, rc = _m().svd_batch(p, N, N, 2, np.concatenate([A, A]))
    assert rc == 0, sw
    assert sig[:N].tobytes() == sig[N:].tobytes()
    with mpmath.workprec(2 * p):
        got = reals(sig[:N])  # descending (mps_svd_batch)
        want = sorted(reals(recs(p, g["sigma"])), reverse=True)  # the oracle's SVD keeps column order
        e_or = max(abs(x - y) for x, y in zip(got, want)) / want[0]
        e_kn = max(abs(x - y) for x, y in zip(got, s)) / s[0]
    print(f"graded svd p={p} N={N}: vs oracle {float(e_or):.2e}, vs known {float(e_kn):.2e}, "
          f"GPU sweeps {sw[0]}, oracle sweeps {g['sweeps']}")
    assert e_or <= tau(p)
    assert e_kn <= tau(p)


@pytest.mark.skipif(not UPD, reason="no cached graded updates")
@pytest.mark.parametrize("g", UPD, ids=[f"p{g['prec']}_chi{g['chi']}_{'lam' if g['in_lambda'] else 'gam'}" for g in UPD])
def test_graded_update_vs_oracle(g):
    p, chi = g["prec"], g["chi"]
    A, B, lam, s = gen.graded_update_inputs(p, chi, g["decades"], *g["key"], in_lambda=g["in_lambda"])
    U = gen.const_gate(p, "I4")
    # the oracle's thr = 0 keeps every sigma >= 0; the GPU ABI reads thr <= 0 as its default
    # 2^-ceil(p/2), so pass a threshold below every nonzero sigma instead (k = chi_max either way)
    out = _m().update_batch(p, chi, 1, A, B, U, lam_m=lam, chi_max=chi, thr=2.0 ** -1000)
    k = int(out["k"][0])
    assert k == g["k"] == chi
    with mpmath.workprec(2 * p):
        got, want = reals(out["sigma"]), reals(recs(p, g["sigma"]))
        e_s = max(abs(x - y) for x, y in zip(got, want)) / want[0]
        e_kn = max(abs(x - y) for x, y in zip(got[:chi], s)) / s[0]
        lg, lw = reals(out["lam"]), reals(recs(p, g["lam"]))
        e_l = max(abs(x - y) for x, y in zip(lg, lw)) / lw[0]
        Pg = reals(p_sample(p, chi, k, out["GL"], out["GR"], out["lam"], g["P_rows"], g["P_cols"]))
        Pw = reals(recs(p, g["P"]))
        e_p = max(abs(x - y) for x, y in zip(Pg, Pw)) / mpmath.mpf(g["Pmax"])
    print(f"graded update p={p} chi={chi} {'lam' if g['in_lambda'] else 'gam'}: sigma {float(e_s):.2e} "
          f"(known {float(e_kn):.2e}) lambda {float(e_l):.2e} P {float(e_p):.2e}; GPU sweeps {out['sweeps'][0]}")
    for e in (e_s, e_kn, e_l, e_p):
        assert e <= tau(p)
