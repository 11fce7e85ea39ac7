"""Site-sharded MPS across GPUs (BASELINE north_star "sites are sharded in
contiguous blocks per GPU ... gates that cross a shard boundary exchange bond tensors by
NCCL send/recv over NVLink").

SPMD: every rank makes the same calls with the same (global) arguments.  Rank r owns the
contiguous global sites [lo_r, hi_r) in a block state (include/mps_b200.h, mps_init_block);
the Schmidt vector of each block-edge bond is mirrored on both neighbours.  Per layer:

  1. a rank whose first site takes part in a gate on its left edge exports that site and the
     Schmidt vector right of it and sends them to rank r-1 (isend/irecv pairs);
  2. every rank applies its interior gates (one batched launch per kernel class) and, for a
     gate on its right edge (hi-1, hi), the boundary update with the received halo;
  3. the updated halo site and the new shared Schmidt vector go back to rank r+1, which
     imports them.

The exchange uses torch.distributed point-to-point (NCCL over NVLink for CUDA tensors, gloo
for the CPU tests); the arithmetic runs in the CUDA kernels of the block engine.  Amplitudes
chain the partial vectors rank to rank and the last rank broadcasts the value.
"""
from __future__ import annotations

import ctypes

import numpy as np


def block_range(n: int, world: int, rank: int):
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


# ------------------------------------------------------------------ CUDA block engine
class CudaBlockEngine:
    """One block state on the current CUDA device (the product engine)."""

    def __init__(self, n_total: int, lo: int, hi: int, p: int, chi_max: int, thr: float):
        import torch

        from . import _chk, _p, lib
        self.torch, self._chk, self._p, self.L = torch, _chk, _p, lib()
        L = self.L
        L.mps_init_block.argtypes = [ctypes.POINTER(ctypes.c_void_p)] + [ctypes.c_int] * 5 + [ctypes.c_double]
        L.mps_block_export_first.argtypes = [ctypes.c_void_p] * 5
        L.mps_block_boundary_apply.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] + [ctypes.c_void_p] * 4
        L.mps_block_import_first.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int]
        L.mps_amplitude_block.argtypes = [ctypes.c_void_p] * 4
        L.mps_block_dims.argtypes = [ctypes.c_void_p] * 5
        h = ctypes.c_void_p()
        _chk(L.mps_init_block(ctypes.byref(h), n_total, lo, hi, p, chi_max, thr), "mps_init_block")
        self.h = h
        self.n, self.lo, self.p, self.chi_max = hi - lo, lo, p, chi_max
        self.rb = int(L.mps_record_bytes(p))
        self.device = torch.device("cuda", torch.cuda.current_device())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.mps_free(self.h)
            self.h = None

    def dims(self):
        a = [ctypes.c_int(0) for _ in range(4)]
        self._chk(self.L.mps_block_dims(self.h, *[ctypes.byref(x) for x in a]))
        return a[2].value, a[3].value

    def apply_layer(self, gates):
        n = len(gates)
        if not n:
            return
        ptrs = (ctypes.c_void_p * n)(*[U.ctypes.data for U, _ in gates])
        flat = [q for _, s in gates for q in s]
        sf = (ctypes.c_int * len(flat))(*flat)
        ks = (ctypes.c_int * n)(*[len(s) for _, s in gates])
        self._chk(self.L.mps_apply_layer(self.h, n, ptrs, sf, ks), "mps_apply_layer")

    def export_first(self):
        t = self.torch
        ml, mr = ctypes.c_int(0), ctypes.c_int(0)
        cap = 2 * self.chi_max * self.chi_max * 2 * self.rb
        G = t.empty(cap, dtype=t.uint8, device=self.device)
        lam = t.empty(self.chi_max * self.rb, dtype=t.uint8, device=self.device)
        self._chk(self.L.mps_block_export_first(self.h, self._p(G), self._p(lam), ctypes.byref(ml), ctypes.byref(mr)))
        return G[: 4 * ml.value * mr.value * self.rb], lam[: mr.value * self.rb], ml.value, mr.value

    def boundary_apply(self, U, G_halo, m_h, lam_h):
        t = self.torch
        k = ctypes.c_int(0)
        Gout = t.empty(2 * self.chi_max * m_h * 2 * self.rb, dtype=t.uint8, device=self.device)
        lam_mid = t.empty(self.chi_max * self.rb, dtype=t.uint8, device=self.device)
        self._chk(self.L.mps_block_boundary_apply(self.h, self._p(U), self._p(G_halo), m_h,
                                                  self._p(lam_h) if lam_h is not None else None,
                                                  self._p(Gout), self._p(lam_mid), ctypes.byref(k)),
                  "mps_block_boundary_apply")
        kk = k.value
        return Gout[: 4 * kk * m_h * self.rb], lam_mid[: kk * self.rb], kk

    def import_first(self, G0, lam_mid, k):
        self._chk(self.L.mps_block_import_first(self.h, self._p(G0), self._p(lam_mid), k), "mps_block_import_first")

    def amplitude_block(self, bits_local, v_in):
        from synth import records as R
        ml, mr = self.dims()
        b = np.asarray(bits_local, np.uint8)
        out = R.empty(self.p, 2 * mr)
        vin = v_in if v_in is not None else None
        self._chk(self.L.mps_amplitude_block(self.h, b.ctypes.data_as(ctypes.c_void_p),
                                             vin.ctypes.data_as(ctypes.c_void_p) if vin is not None else None,
                                             out.ctypes.data_as(ctypes.c_void_p)), "mps_amplitude_block")
        return out

    def to_transport(self, x):
        """numpy record array -> tensor on the engine's device (for NCCL)."""
        return self.torch.from_numpy(np.ascontiguousarray(x).view(np.uint8)).to(self.device)


# ------------------------------------------------------------------ SPMD driver
class ShardedMPS:
    """An n-qubit MPS sharded over the ranks of a torch.distributed group."""

    def __init__(self, n: int, p: int, chi_max: int, thr: float = 0.0, engine_factory=None, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.n, self.p = n, p
        if self.world > n:
            raise ValueError("more ranks than sites")
        self.bounds = [block_range(n, self.world, r) for r in range(self.world)]
        self.lo, self.hi = self.bounds[self.rank]
        factory = engine_factory or CudaBlockEngine
        self.engine = factory(n, self.lo, self.hi, p, chi_max, thr)

    # -- point-to-point helpers: variable-size uint8 payloads with an int64 header
    def _send(self, tensors, dst, ints=()):
        t = self.engine.torch
        hdr = t.tensor([len(x) for x in tensors] + list(ints), dtype=t.int64, device=tensors[0].device)
        keep = [hdr] + [x.contiguous() for x in tensors]
        self._keep = getattr(self, "_keep", []) + keep  # buffers must outlive the isends
        reqs = [self.dist.isend(hdr, dst, group=self.group)]
        for x in keep[1:]:
            if len(x):
                reqs.append(self.dist.isend(x, dst, group=self.group))
        return reqs

    def _recv(self, n_t, src, n_ints, device):
        t = self.engine.torch
        hdr = t.empty(n_t + n_ints, dtype=t.int64, device=device)
        self.dist.recv(hdr, src, group=self.group)
        out = []
        for i in range(n_t):
            x = t.empty(int(hdr[i].item()), dtype=t.uint8, device=device)
            if len(x):
                self.dist.recv(x, src, group=self.group)
            out.append(x)
        return out, [int(v) for v in hdr[n_t:].tolist()]

    def apply_layer(self, gates):
        """gates: list of (U records, global sites), pairwise disjoint."""
        lo, hi = self.lo, self.hi
        local, right_edge, left_edge = [], None, None
        for U, s in gates:
            s = list(s)
            if lo <= s[0] and s[-1] < hi:
                local.append((U, [q - lo for q in s]))
            elif s[0] < hi <= s[-1] and s[0] >= lo:
                if len(s) != 2 or s[1] != s[0] + 1:
                    raise NotImplementedError("only adjacent two-site gates may cross a block edge")
                right_edge = U
            elif s[0] < lo <= s[-1] and s[-1] < hi:
                if len(s) != 2 or s[1] != s[0] + 1:
                    raise NotImplementedError("only adjacent two-site gates may cross a block edge")
                left_edge = True
        dev = getattr(self.engine, "device", None)
        reqs = []
        # 1. halos to the left neighbour
        if left_edge:
            G, lam, ml, mr = self.engine.export_first()
            reqs += self._send([G, lam], self.rank - 1, ints=(mr,))
        halo = None
        if right_edge is not None:
            (G, lam), (mh,) = self._recv(2, self.rank + 1, 1, dev)
            halo = (G, lam if len(lam) else None, mh)
        for r in reqs:
            r.wait()
        # 2. interior gates (batched) and the right-edge gate
        self.engine.apply_layer(local)
        reqs = []
        if halo is not None:
            G, lam, mh = halo
            Gout, lam_mid, k = self.engine.boundary_apply(right_edge, G, mh, lam)
            reqs += self._send([Gout, lam_mid], self.rank + 1, ints=(k,))
        # 3. the left neighbour returns our new first site and shared Schmidt vector
        if left_edge:
            (G0, lam_mid), (k,) = self._recv(2, self.rank - 1, 1, dev)
            self.engine.import_first(G0, lam_mid, k)
        for r in reqs:
            r.wait()
        self._keep = []

    def amplitude(self, bits):
        """Eq. 1 amplitude (complex records) of global bit string `bits`, on every rank."""
        from synth import records as R
        t = self.engine.torch
        v_in = None
        if self.rank > 0:
            (v,), _ = self._recv(1, self.rank - 1, 0, getattr(self.engine, "device", None))
            v_in = np.frombuffer(v.cpu().numpy().tobytes(), dtype=R.record_dtype(self.p)).copy()
        v_out = self.engine.amplitude_block(list(bits[self.lo:self.hi]), v_in)
        if self.rank < self.world - 1:
            for r in self._send([self.engine.to_transport(v_out)], self.rank + 1):
                r.wait()
        # broadcast the amplitude from the last rank
        buf = self.engine.to_transport(v_out) if self.rank == self.world - 1 else \
            t.empty(2 * R.record_bytes(self.p), dtype=t.uint8, device=getattr(self.engine, "device", None))
        if self.world > 1:
            self.dist.broadcast(buf, self.world - 1, group=self.group)
        return np.frombuffer(buf.cpu().numpy().tobytes(), dtype=R.record_dtype(self.p)).copy()
