"""Test-only block engine backed by the ORACLE (oracle.update2_batch) so that the sharded
driver's exchange protocol (paper_1111_3124_b200/dist.py) can run on CPU ranks over gloo.
It implements the CudaBlockEngine interface; the product never uses it."""
import mpmath
import numpy as np
import torch

import oracle
from synth import records as R


class OracleBlockEngine:
    def __init__(self, n_total, lo, hi, p, chi_max, thr):
        self.torch = torch
        self.device = None
        self.n, self.lo, self.p, self.chi_max, self.thr = hi - lo, lo, p, chi_max, thr
        self.has_l, self.has_r = lo > 0, hi < n_total
        one = R.reals_from_values(p, [1])
        site = R.cplx_from_values(p, [(1, 0), (0, 0)])
        self.G = [site.copy() for _ in range(self.n)]
        self.lam = [one.copy() for _ in range(self.n - 1)]
        self.m = [1] * (self.n - 1)
        self.lam_el, self.lam_er = one.copy(), one.copy()
        self.m_el = self.m_er = 1

    def dl(self, s):
        return (self.m_el if self.has_l else 1) if s == 0 else self.m[s - 1]

    def dr(self, s):
        return (self.m_er if self.has_r else 1) if s == self.n - 1 else self.m[s]

    def lamL(self, s):
        return self.lam[s - 1] if s > 0 else (self.lam_el if self.has_l else None)

    def lamR(self, s):
        return self.lam[s] if s < self.n - 1 else (self.lam_er if self.has_r else None)

    def dims(self):
        return self.dl(0), self.dr(self.n - 1)

    def _update(self, U, GL, GR, dl, dm, dr, lamL, lamM, lamR):
        o = oracle.update2_batch(self.p, 1, dl, dm, dr, self.chi_max, self.thr, GL, GR, U, lamL, lamM, lamR, nthreads=1)
        k = int(o["k"][0])
        gl = o["GL"].reshape(2 * dl, self.chi_max, 2)[:, :k].reshape(-1)
        gr = o["GR"].reshape(2, self.chi_max, dr * 2)[:, :k].reshape(-1)
        return gl.copy(), gr.copy(), o["lam"][:k].copy(), k

    def apply_layer(self, gates):
        for U, s in gates:
            assert len(s) == 2 and s[1] == s[0] + 1, "test engine: two-site gates only"
            q = s[0]
            gl, gr, lam, k = self._update(U, self.G[q], self.G[q + 1], self.dl(q), self.m[q], self.dr(q + 1),
                                          self.lamL(q), self.lam[q], self.lamR(q + 1))
            self.G[q], self.G[q + 1], self.lam[q], self.m[q] = gl, gr, lam, k

    def to_transport(self, x):
        return torch.from_numpy(np.ascontiguousarray(x).view(np.uint8).copy())

    def _from(self, t):
        return np.frombuffer(t.numpy().tobytes(), dtype=R.record_dtype(self.p)).copy()

    def export_first(self):
        lam = self.lamR(0)
        return (self.to_transport(self.G[0]), self.to_transport(lam) if lam is not None else torch.empty(0, dtype=torch.uint8),
                self.dl(0), self.dr(0))

    def boundary_apply(self, U, G_halo, m_h, lam_h):
        q = self.n - 1
        gl, gr, lam, k = self._update(U, self.G[q], self._from(G_halo), self.dl(q), self.m_er, m_h,
                                      self.lamL(q), self.lam_er, self._from(lam_h) if lam_h is not None else None)
        self.G[q], self.lam_er, self.m_er = gl, lam, k
        return self.to_transport(gr), self.to_transport(lam), k

    def import_first(self, G0, lam_mid, k):
        self.G[0], self.lam_el, self.m_el = self._from(G0), self._from(lam_mid), k

    def amplitude_block(self, bits, v_in):
        """partial Eq. 1 chain in mpmath at 2p+64 bits, rounded to p-bit records"""
        from tests.helpers import cplx, reals
        with mpmath.workprec(2 * self.p + 64):
            v = cplx(v_in) if v_in is not None else [mpmath.mpc(1)]
            for s in range(self.n):
                dl, dr = self.dl(s), self.dr(s)
                lam = reals(self.lamL(s)) if self.lamL(s) is not None else [mpmath.mpf(1)] * dl
                g = cplx(self.G[s])
                b = bits[s]
                v = [mpmath.fsum(v[a] * lam[a] * g[(b * dl + a) * dr + c] for a in range(dl)) for c in range(dr)]
        with mpmath.workprec(self.p):
            return R.cplx_from_values(self.p, [(+x.real, +x.imag) for x in v])
