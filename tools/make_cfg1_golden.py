"""Cache the ORACLE's two-site updates of BASELINE configs[1] items (calls only oracle/ and synth/).

    python tools/make_cfg1_golden.py --prec 280 --chi 128 --item 0 [--item 1 ...]

One item per process (the oracle's update of one item is single-threaded; run several
processes side by side).  Item i is `synth.gen.update_batch_inputs(p, chi, 1, first=i)`,
i.e. the same seeded item bench.py places at batch positions i, i + 128, ... on rank 0,
with the bench's truncation (chi_max = chi, thr = 0: k = chi, SURVEY §8(d) cfg2 "truncate
to k = chi").  Writes tests/golden/cfg1_p{p}_chi{chi}_item{i}.json:

  sigma   all 2chi singular values (descending), exact p-bit records (hex of the bytes)
  k, lam  kept count and the renormalised Schmidt vector lambda'
  P       the gauge-invariant local check of SURVEY §8(c) "Comparison metrics",
          P = X_k diag(lambda') V_k^H = Gamma_A' diag(lambda') Gamma_B' (lambda_l = lambda_r = 1),
          on a seeded grid of 32 rows x 32 columns of the 2chi x 2chi matrix, each entry the
          sum over b < k evaluated in mpmath at p + 64 bits and rounded to p bits
  Pmax    ||P||_max over ALL entries (binary64, from the oracle's factors: a scale only)
  sweeps  the oracle's sweep count (its textbook cyclic Jacobi, final check-only sweep included)
  seconds wall time of the oracle update on one core
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import gen  # noqa: E402
from synth import records as R  # noqa: E402
from tests.helpers import p_sample  # noqa: E402

NGRID = 32


def grid(chi: int, item: int):
    """Seeded rows / columns of P (first and last always included)."""
    N = 2 * chi
    g = gen.rng(gen.SEED0 + 1, item, 0x9A1D)
    rows = sorted(set([0, N - 1] + g.choice(N, NGRID - 2, replace=False).tolist()))
    cols = sorted(set([0, N - 1] + g.choice(N, NGRID - 2, replace=False).tolist()))
    return rows[:NGRID], cols[:NGRID]


def pmax(chi, GL, GR, lam):
    gl = R.cplx_to_complex128(GL).reshape(2 * chi, chi)
    gr = R.cplx_to_complex128(GR).reshape(2, chi, chi).transpose(1, 0, 2).reshape(chi, 2 * chi)
    lm = R.to_float64(lam)
    return float(np.abs((gl * lm[None, :]) @ gr).max())


def hexa(a: np.ndarray) -> str:
    return a.tobytes().hex()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prec", type=int, required=True)
    ap.add_argument("--chi", type=int, required=True)
    ap.add_argument("--item", type=int, action="append", required=True)
    ap.add_argument("--outdir", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    p, chi = a.prec, a.chi
    for it in a.item:
        A, B, U = gen.update_batch_inputs(p, chi, 1, first=it)
        t0 = time.time()
        o = oracle.update2_batch(p, 1, chi, chi, chi, chi, 0.0, A, B, U, nthreads=1)
        secs = time.time() - t0
        k = int(o["k"][0])
        rows, cols = grid(chi, it)
        P = p_sample(p, chi, k, o["GL"], o["GR"], o["lam"], rows, cols)
        res = {
            "what": "oracle two-site update of one BASELINE configs[1] item (tools/make_cfg1_golden.py, oracle/ only)",
            "prec": p, "chi": chi, "item": it, "chi_max": chi, "thr": 0.0,
            "sigma": hexa(o["sigma"]), "k": k, "lam": hexa(o["lam"]), "sweeps": int(o["sweeps"][0]),
            "P_rows": rows, "P_cols": cols, "P": hexa(P), "Pmax": pmax(chi, o["GL"], o["GR"], o["lam"]),
            "seconds": secs, "threads": 1, "cpu": platform.processor() or platform.machine(),
        }
        out = os.path.join(a.outdir, f"cfg1_p{p}_chi{chi}_item{it}.json")
        with open(out, "w") as f:
            json.dump(res, f)
        print("wrote", out, f"{secs:.0f}s sweeps {res['sweeps']}", flush=True)


if __name__ == "__main__":
    main()
