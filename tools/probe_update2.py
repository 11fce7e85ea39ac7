"""Timing probe of the device batch path (mps_update_batch_device) — development tool."""
import argparse
import json
import time

import numpy as np
import torch

import paper_1111_3124_b200 as m
from synth import gen
from synth import records as R

ap = argparse.ArgumentParser()
ap.add_argument("--chi", type=int, nargs="+", default=[32, 64, 128])
ap.add_argument("--prec", type=int, default=280)
ap.add_argument("--batch", type=int, default=148)
ap.add_argument("--distinct", type=int, default=16)
args = ap.parse_args()

res = []
for chi in args.chi:
    p = args.prec
    nd = min(args.distinct, args.batch)
    A, B, U = gen.update_batch_inputs(p, chi, nd)
    reps = (args.batch + nd - 1) // nd
    A = np.tile(A, reps)[: args.batch * 4 * chi * chi]
    B = np.tile(B, reps)[: args.batch * 4 * chi * chi]
    U = np.tile(U, reps)[: args.batch * 32]
    dev = torch.device("cuda:0")
    tA = torch.from_numpy(A.view(np.uint8)).to(dev)
    tB = torch.from_numpy(B.view(np.uint8)).to(dev)
    tU = torch.from_numpy(U.view(np.uint8)).to(dev)
    rb = R.record_bytes(p)
    batch = args.batch
    sig = torch.empty(batch * 2 * chi * rb, dtype=torch.uint8, device=dev)
    k = torch.empty(batch, dtype=torch.int32, device=dev)
    Ao = torch.empty(batch * 2 * chi * chi * 2 * rb, dtype=torch.uint8, device=dev)
    Bo = torch.empty_like(Ao)
    lam = torch.empty(batch * chi * rb, dtype=torch.uint8, device=dev)
    sw = torch.empty(batch, dtype=torch.int32, device=dev)
    ws = torch.empty(m.update_batch_workspace(p, chi, batch), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    torch.cuda.synchronize()
    t0 = time.time()
    m.update_batch_device(p, chi, chi, batch, 0.0, tA, tB, tU, sig, k, Ao, Bo, lam, sw, ws, stream=st)
    torch.cuda.synchronize()
    dt = time.time() - t0
    sweeps = sw.cpu().numpy()
    S = float(sweeps.mean())
    n = 2 * chi
    real_mults = 16 * chi ** 3 + 64 * chi ** 2 + (S - 1) * n * (n - 1) / 2 * (20 * n + 12 * n) + n * (n - 1) / 2 * 8 * n
    L = 9 if p <= 288 else 16
    limb_macs = real_mults * (((p + 31) // 32) ** 2)
    r = dict(chi=chi, p=p, batch=batch, seconds=dt, items_per_s=batch / dt, sweeps_mean=S,
             limb_mac_per_s=limb_macs * batch / dt, frac_of_imadwide=limb_macs * batch / dt / 7.30e12)
    print(json.dumps(r), flush=True)
    res.append(r)
