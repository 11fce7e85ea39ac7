"""BASELINE configs[1] at the benchmark's sizes and launch configuration against cached ORACLE
updates (SURVEY §8(c) "cfg2 items: compare sigma and P"; VERDICT r01 "Next round" item 1).

tests/golden/cfg1_p{p}_chi{chi}_item{i}.json hold the oracle's complete two-site update of
seeded item i (tools/make_cfg1_golden.py, oracle/ only: its textbook cyclic Jacobi from
Theta', accumulated V).  Here the same items run inside a full bench-shaped batch through
mps_update_batch_device, the entry bench.py times (1024 items at chi <= 128, one wave of 296
at chi = 256; 128 distinct seeded items tiled, so item i sits at positions i, i + 128, ...;
chi_max = chi, thr = 0; the cluster size is chosen by the library as in the bench).
Compared (tau = 1e-70 at 280 bits, 1e-140 at 512, normwise, SURVEY §8(c) ledger #12):
  * k exactly; all 2chi singular values: max_j |s^_j - s_j| / s_0 <= tau  (PAPER.md:69-70 SVD);
  * lambda' = sigma_1..k / ||sigma_1..k|| (P:272-273 truncation, S:338 renormalisation);
  * the gauge-invariant P = X_k diag(lambda') V_k^H on the cached 32 x 32 grid of entries:
    max |P^ - P| / ||P||_max <= tau  (P:258-263 split into site tensors);
  * the tiled copies of the item in the same launch are bitwise equal to it.
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
ND = 128  # distinct seeded items (bench.py --distinct)


def batch_of(chi):
    return 1024 if chi <= 128 else 296


def cases():
    out = {}
    for f in sorted(glob.glob(os.path.join(GOLD, "cfg1_p*_chi*_item*.json"))):
        g = json.load(open(f))
        out.setdefault((g["prec"], g["chi"]), []).append(g)
    return sorted(out.items())


def recs(p, hexstr):
    return np.frombuffer(bytes.fromhex(hexstr), dtype=R.record_dtype(p)).copy()


def run_bench_batch(p, chi, batch, items):
    """One mps_update_batch_device launch of the bench's batch; host copies of the outputs of
    the positions of `items` and of their first tiled copy."""
    import torch

    import paper_1111_3124_b200 as m
    dev = torch.device("cuda", 0)
    A, B, U = gen.update_batch_inputs(p, chi, ND)
    reps = (batch + ND - 1) // ND
    A = np.tile(A, reps)[: batch * 4 * chi * chi]
    B = np.tile(B, reps)[: batch * 4 * chi * chi]
    U = np.tile(U, reps)[: batch * 32]
    rb = R.record_bytes(p)
    tA = torch.from_numpy(A.view(np.uint8)).to(dev)
    tB = torch.from_numpy(B.view(np.uint8)).to(dev)
    tU = torch.from_numpy(U.view(np.uint8)).to(dev)
    del A, B
    sig = torch.empty(batch * 2 * chi * rb, dtype=torch.uint8, device=dev)
    kk = torch.empty(batch, dtype=torch.int32, device=dev)
    Ao = torch.empty(batch * 4 * chi * chi * rb, dtype=torch.uint8, device=dev)
    Bo = torch.empty_like(Ao)
    lam = torch.empty(batch * chi * rb, dtype=torch.uint8, device=dev)
    sw = torch.empty(batch, dtype=torch.int32, device=dev)
    ws = torch.empty(m.update_batch_workspace(p, chi, batch), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev)
    m.update_batch_device(p, chi, chi, batch, 0.0, tA, tB, tU, sig, kk, Ao, Bo, lam, sw, ws, stream=st.cuda_stream)
    torch.cuda.synchronize(dev)
    del ws, tA, tB, tU
    dt = R.record_dtype(p)
    N = 2 * chi
    ne = 4 * chi * chi
    out = {"k": kk.cpu().numpy(), "sweeps": sw.cpu().numpy()}
    for b in sorted(set(items) | {i + ND for i in items if i + ND < batch}):
        out[b] = dict(
            sigma=np.frombuffer(sig[b * N * rb:(b + 1) * N * rb].cpu().numpy().tobytes(), dtype=dt).copy(),
            lam=np.frombuffer(lam[b * chi * rb:(b + 1) * chi * rb].cpu().numpy().tobytes(), dtype=dt).copy(),
            GL=np.frombuffer(Ao[b * ne * rb:(b + 1) * ne * rb].cpu().numpy().tobytes(), dtype=dt).copy(),
            GR=np.frombuffer(Bo[b * ne * rb:(b + 1) * ne * rb].cpu().numpy().tobytes(), dtype=dt).copy())
    del sig, Ao, Bo, lam
    torch.cuda.empty_cache()
    return out


CASES = cases()


@pytest.mark.skipif(not CASES, reason="no cached configs[1] oracle updates")
@pytest.mark.parametrize("key,golds", CASES, ids=[f"p{k[0]}_chi{k[1]}" for k, _ in CASES])
def test_bench_batch_vs_cached_oracle(key, golds):
    p, chi = key
    batch = batch_of(chi)
    items = [g["item"] for g in golds]
    assert max(items) < ND
    out = run_bench_batch(p, chi, batch, items)
    assert (out["k"] == chi).all()
    t = tau(p)
    for g in golds:
        i = g["item"]
        got = out[i]
        # tiled copy in the same launch: bitwise equal
        if i + ND < batch:
            for f in ("sigma", "lam", "GL", "GR"):
                assert got[f].tobytes() == out[i + ND][f].tobytes(), (i, f)
        assert g["k"] == chi
        with mpmath.workprec(2 * p):
            sw, sg = reals(recs(p, g["sigma"])), reals(got["sigma"])
            es = max(abs(x - y) for x, y in zip(sg, sw)) / sw[0]
            lw, lg = reals(recs(p, g["lam"])), reals(got["lam"])
            el = max(abs(x - y) for x, y in zip(lg, lw)) / lw[0]
            Pw = reals(recs(p, g["P"]))
            Pg = reals(p_sample(p, chi, chi, got["GL"], got["GR"], got["lam"], g["P_rows"], g["P_cols"]))
            ep = max(abs(x - y) for x, y in zip(Pg, Pw)) / mpmath.mpf(g["Pmax"])
        print(f"p={p} chi={chi} item {i}: sigma {float(es):.2e} lambda {float(el):.2e} P {float(ep):.2e} "
              f"(tau {t:.0e}); GPU sweeps {out['sweeps'][i]}, oracle sweeps {g['sweeps']}")
        assert es <= t, (i, es)
        assert el <= t, (i, el)
        assert ep <= t, (i, ep)
