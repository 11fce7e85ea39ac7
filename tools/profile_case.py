"""One batched two-site update (device path) for ncu captures: python tools/profile_case.py CHI PREC BATCH"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_3124_b200 as m  # noqa: E402
from synth import gen  # noqa: E402
from synth import records as R  # noqa: E402

chi, p, batch = (int(x) for x in sys.argv[1:4])
nd = min(16, batch)
A, B, U = gen.update_batch_inputs(p, chi, nd)
reps = (batch + nd - 1) // nd
A = np.tile(A, reps)[: batch * 4 * chi * chi]
B = np.tile(B, reps)[: batch * 4 * chi * chi]
U = np.tile(U, reps)[: batch * 32]
dev = torch.device("cuda:0")
t = {k: torch.from_numpy(v.view(np.uint8)).to(dev) for k, v in (("A", A), ("B", B), ("U", U))}
rb = R.record_bytes(p)
sig = torch.empty(batch * 2 * chi * rb, dtype=torch.uint8, device=dev)
k = torch.empty(batch, dtype=torch.int32, device=dev)
Ao = torch.empty(batch * 4 * chi * chi * rb, dtype=torch.uint8, device=dev)
Bo = torch.empty_like(Ao)
lam = torch.empty(batch * chi * rb, dtype=torch.uint8, device=dev)
sw = torch.empty(batch, dtype=torch.int32, device=dev)
ws = torch.empty(m.update_batch_workspace(p, chi, batch), dtype=torch.uint8, device=dev)
m.update_batch_device(p, chi, chi, batch, 0.0, t["A"], t["B"], t["U"], sig, k, Ao, Bo, lam, sw, ws,
                      stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("sweeps", sw.cpu().numpy().mean(), "k", int(k.cpu().numpy().min()))
