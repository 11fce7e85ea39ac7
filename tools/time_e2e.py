"""Time the end-to-end call (mps_bench_update_batch, pinned host buffers) a few times; MPS_E2E_CHUNK selects the chunking.
   python tools/time_e2e.py [chi] [p] [batch] [reps]"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_3124_b200 as m  # noqa: E402
from synth import gen  # noqa: E402

chi = int(sys.argv[1]) if len(sys.argv) > 1 else 128
p = int(sys.argv[2]) if len(sys.argv) > 2 else 280
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
nd = min(batch, 128)
A0, B0, U0 = gen.update_batch_inputs(p, chi, nd)
rep = (batch + nd - 1) // nd
A = np.tile(A0, rep)[: batch * 4 * chi * chi]
B = np.tile(B0, rep)[: batch * 4 * chi * chi]
U = np.tile(U0, rep)[: batch * 32]
def pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).pin_memory().numpy().view(a.dtype)
pA, pB, pU = pinned(A), pinned(B), pinned(U)
rdt = A.dtype
ob = {"sigma": pinned(np.empty(batch * 2 * chi, rdt)), "k": pinned(np.zeros(batch, np.int32)),
      "GL": pinned(np.empty(batch * 4 * chi * chi, rdt)), "GR": pinned(np.empty(batch * 4 * chi * chi, rdt)),
      "lam": pinned(np.empty(batch * chi, rdt)), "sweeps": pinned(np.zeros(batch, np.int32))}
m.update_batch(p, chi, batch, pA, pB, pU, out_buffers=ob)
for _ in range(reps):
    t0 = time.perf_counter()
    m.update_batch(p, chi, batch, pA, pB, pU, out_buffers=ob)
    dt = time.perf_counter() - t0
    print(f"chunk={os.environ.get('MPS_E2E_CHUNK', 'default')} e2e {dt:.3f} s = {batch / dt:.1f} updates/s", flush=True)
