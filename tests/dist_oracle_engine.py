"""Test-only engines for the sharded driver (paper_1111_3124_b200/dist.py) on CPU ranks over
gloo: the same engine interface as dist.CudaEngine, backed by the ORACLE's full-length MPS
(oracle.OracleMPS: get_site / set_site / schmidt / set_schmidt / apply_layer), with host
torch tensors as transport buffers.  The product never uses it."""
import numpy as np
import torch

import oracle
from synth import records as R


class OracleEngine:
    def __init__(self, n, p, chi_max, thr):
        self.torch = torch
        self.device = None
        self.n, self.p = n, p
        self.m = oracle.OracleMPS(n, p, chi_max, thr)
        self.dt = R.record_dtype(p)

    def _rec(self, buf):
        return np.frombuffer(buf.numpy().tobytes(), dtype=self.dt).copy()

    def bond_dims(self):
        return self.m.bond_dims()

    def apply_layer(self, gates):
        if gates:
            self.m.apply_layer(gates, nthreads=1)

    def export_site(self, q, out):
        G, ml, mr = self.m.get_site(q)
        out.copy_(torch.from_numpy(G.view(np.uint8).copy()))

    def import_site(self, q, buf, ml, mr):
        self.m.set_site(q, self._rec(buf), ml, mr)

    def export_schmidt(self, b, out):
        lam = self.m.schmidt(b)
        out[: lam.nbytes].copy_(torch.from_numpy(lam.view(np.uint8).copy()))
        return len(lam)

    def import_schmidt(self, b, buf, m):
        self.m.set_schmidt(b, self._rec(buf)[:m])

    def amplitude(self, bits):
        return self.m.amplitude(bits)
