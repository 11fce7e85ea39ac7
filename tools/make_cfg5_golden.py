"""Cache the ORACLE's two-site updates of configs[4]-shaped gates (calls only oracle/ and synth/).

    python tools/make_cfg5_golden.py --item 0 [--item 1 ...]

SURVEY §8(c) "cfg5 end-to-end": the whole configs[4] circuit (n = 64, depth 40, chi_max 256,
512 bits) is out of the oracle's reach (~1.1e3 core-hours), so it is pinned per gate.  The
inputs of a deep gate cannot be dumped from the GPU run (no oracle input may come from the
CUDA path), so each sampled gate is a seeded synthetic window of the same shape and structure
(`synth.gen.canonical_update_inputs`, R25): chi_l = chi_m = chi_r = 256 (every bond
from site 9 to 54 is saturated at 256 in configs[4]), Vidal canonical Gamma tensors, graded
unit-norm Schmidt vectors over 6-16 decades, a Haar U(4); configs[4]'s chi_max = 256 and
threshold 2^-256, so the 512 singular values of Theta' are cut to 256.

ITEMS[i] = (layer, first site, dec_l, dec_m, dec_r): the four disjoint windows of one odd
layer (sites 15-16 and 31-32 cross the block edges of the 8-sites-per-GPU sharding).  Writes
tests/golden/cfg5_p512_chi256_item{i}.json: sigma (all 512, oracle order), k, lambda', P on a
seeded 32 x 32 grid with lambda_l, lambda_r multiplied back in (tests.helpers.p_sample), Pmax,
the oracle's sweep count and wall time (one core).
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

P, CHI, THR = 512, 256, 2.0 ** -256
LAYER = 21
ITEMS = [(LAYER, 15, 6, 10, 6), (LAYER, 19, 8, 12, 8), (LAYER, 27, 6, 14, 6), (LAYER, 31, 8, 16, 8)]
NGRID = 32


def key(i: int):
    layer, site = ITEMS[i][:2]
    return (gen.SEED0 + 4, layer, site)


def inputs(i: int, chi: int = CHI):
    _, _, dl, dm, dr = ITEMS[i]
    return gen.canonical_update_inputs(P, chi, dl, dm, dr, *key(i))


def grid(i: int, chi: int = CHI):
    N = 2 * chi
    g = gen.rng(*key(i), 0x9A1D)
    rows = sorted(set([0, N - 1] + g.choice(N, NGRID - 2, replace=False).tolist()))
    cols = sorted(set([0, N - 1] + g.choice(N, NGRID - 2, replace=False).tolist()))
    return rows[:NGRID], cols[:NGRID]


def pmax(GL, GR, lam, lam_l, lam_r, chi: int = CHI):
    gl = R.cplx_to_complex128(GL).reshape(2, chi, chi) * R.to_float64(lam_l)[None, :, None]
    gr = R.cplx_to_complex128(GR).reshape(2, chi, chi) * R.to_float64(lam_r)[None, None, :]
    gl = gl.reshape(2 * chi, chi)
    gr = gr.transpose(1, 0, 2).reshape(chi, 2 * chi)
    return float(np.abs((gl * R.to_float64(lam)[None, :]) @ gr).max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--item", type=int, action="append", required=True)
    ap.add_argument("--outdir", default=os.path.join(ROOT, "tests", "golden"))
    ap.add_argument("--chi", type=int, default=CHI,
                    help="bond dimension of the window (configs[4] saturates at 256: ~5 h per item on one core; "
                         "128 is the half-size stand-in, ~45 min)")
    a = ap.parse_args()
    chi = a.chi
    for it in a.item:
        A, B, ll, lm, lr, U = inputs(it, chi)
        t0 = time.time()
        o = oracle.update2_batch(P, 1, chi, chi, chi, chi, THR, A, B, U, lam_l=ll, lam_m=lm, lam_r=lr, nthreads=1)
        secs = time.time() - t0
        k = int(o["k"][0])
        rows, cols = grid(it, chi)
        Ps = p_sample(P, chi, k, o["GL"], o["GR"], o["lam"], rows, cols, lam_l=ll, lam_r=lr)
        res = {
            "what": "oracle two-site update of a configs[4]-shaped gate (tools/make_cfg5_golden.py, oracle/ only)",
            "prec": P, "chi": chi, "item": it, "chi_max": chi, "thr": THR, "spec": list(ITEMS[it]),
            "key": list(key(it)),
            "sigma": o["sigma"].tobytes().hex(), "k": k, "lam": o["lam"].tobytes().hex(),
            "sweeps": int(o["sweeps"][0]), "P_rows": rows, "P_cols": cols, "P": Ps.tobytes().hex(),
            "Pmax": pmax(o["GL"], o["GR"], o["lam"], ll, lr, chi),
            "seconds": secs, "threads": 1, "cpu": platform.processor() or platform.machine(),
        }
        out = os.path.join(a.outdir, f"cfg5_p{P}_chi{chi}_item{it}.json")
        with open(out, "w") as f:
            json.dump(res, f)
        print("wrote", out, f"{secs:.0f}s sweeps {res['sweeps']} k {k}", flush=True)


if __name__ == "__main__":
    main()
