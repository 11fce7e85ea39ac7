"""Site-sharded MPS across GPUs (BASELINE north_star "sites are sharded in
contiguous blocks per GPU ... disjoint gates within a brick-wall layer run concurrently, and
gates that cross a shard boundary exchange bond tensors by NCCL send/recv over NVLink").

SPMD: every rank makes the same calls with the same (global) arguments.  Rank r OWNS the
contiguous global sites [lo_r, hi_r) (block_range).  A gate updates only the site tensors
of its window and the Schmidt vectors between them (§3.1: "we have only
to update Q_s, V_s, Q_{s+1}"), so a layer of disjoint gates is independent work that any
rank can do.  Per layer (ShardedMPS.apply_layer):

  0. plan: every gate gets an executing rank, identically on all ranks, from the replicated
     bond dimensions: gates are taken in decreasing order of their predicted cost (the
     Jacobi work N^2 (20M + 12N) of SURVEY §8(d)) and given to the least loaded
     rank, the owner of the window's first site when it is within 5% of that (LPT; §8(e)
     computes E(8) ~ 0.74 with owner-computes and ~0.98 with LPT on configs[4]);
  1. migrate in: owners send the window's site tensors to the executing rank when it is
     another (one batched NCCL send/recv group per layer, sizes known from the replicated
     dims: no size headers, no host round trips);
  2. compute: each rank applies its gates as ONE mps_apply_layer call (the batched kernels
     of the single-GPU engine; a gate's arithmetic does not depend on which other gates
     share its batch, so results are bitwise independent of the placement and of N);
  3. the new Schmidt vectors and bond dimensions of the layer's windows reach every rank in
     one all-reduce (each slot written by its executing rank only, zeros elsewhere: exact);
  4. migrate out: executing ranks send updated site tensors back to their owners.

Every rank holds a full-length state whose Schmidt vectors and bond dimensions are always
current (replicated, O(n chi) records) and whose site tensors are current on the sites it
owns (plus, transiently, the windows it executes).  Queries gather the site tensors on
rank 0 and broadcast the value.  Transport: torch.distributed point-to-point and all-reduce
(NCCL over NVLink on GPUs; gloo with host staging for the CPU tests and for several ranks
sharing one GPU).
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


# ------------------------------------------------------------------ full-state CUDA engine
class CudaEngine:
    """A full-length MPS state on the current CUDA device (mps_init) with device-buffer
    export / import of site tensors and Schmidt vectors (the product engine of ShardedMPS)."""

    def __init__(self, n: int, p: int, chi_max: int, thr: float):
        import torch

        from . import MPS, _chk, _p, lib
        self.torch, self._chk, self._p, self.L = torch, _chk, _p, lib()
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.current_stream(self.device)
        self.mps = MPS(n, p, chi_max, thr, stream=self.stream.cuda_stream)
        self.n, self.p, self.chi_max = n, p, chi_max
        self.rb = int(self.L.mps_record_bytes(p))

    def empty(self, nbytes: int):
        return self.torch.empty(nbytes, dtype=self.torch.uint8, device=self.device)

    def bond_dims(self):
        return self.mps.bond_dims()

    def apply_layer(self, gates):
        if gates:
            self.mps.apply_layer(gates)

    def export_site(self, q: int, out):
        ml, mr = ctypes.c_int(0), ctypes.c_int(0)
        self._chk(self.L.mps_get_site(self.mps.h, q, self._p(out), ctypes.byref(ml), ctypes.byref(mr)),
                  "mps_get_site")

    def import_site(self, q: int, buf, ml: int, mr: int):
        self._chk(self.L.mps_set_site(self.mps.h, q, self._p(buf), ml, mr), "mps_set_site")

    def export_schmidt(self, b: int, out):
        m = ctypes.c_int(0)
        self._chk(self.L.mps_schmidt(self.mps.h, b, self._p(out), ctypes.byref(m)), "mps_schmidt")
        return m.value

    def import_schmidt(self, b: int, buf, m: int):
        self._chk(self.L.mps_set_schmidt(self.mps.h, b, self._p(buf), m), "mps_set_schmidt")

    def amplitude(self, bits):
        return self.mps.amplitude(bits)

    def norm2(self):
        return self.mps.norm2()


# ------------------------------------------------------------------ planning (host, replicated)
def bond_cap(b: int, n: int, chi_max: int) -> int:
    """Capacity of bond b: the Schmidt rank bound min(2^(b+1), 2^(n-b-1)), capped at chi_max
    (the same rule as the library's store, state.cu gcap)."""
    e = min(b + 1, n - b - 1)
    return min(chi_max, 1 << min(e, 30))


def window(sites):
    return min(sites), max(sites)


def svd_cost(rows: int, cols: int) -> float:
    """Real p-bit multiplies per Jacobi sweep of a rows x cols matrix:
    N(N-1)/2 pairs x (20M + 12N), M >= N."""
    M, N = max(rows, cols), min(rows, cols)
    return N * (N - 1) / 2.0 * (20 * M + 12 * N)


def gate_cost(sites, dims, n: int, chi_max: int) -> float:
    """Predicted cost of a gate from the current bond dims (O(m^3) per update)."""
    lo, hi = window(sites)
    dl = dims[lo - 1] if lo > 0 else 1
    dr = dims[hi] if hi < n - 1 else 1
    span = hi - lo + 1
    if span == 1:
        return 1.0
    if span == 2:
        return svd_cost(2 * dl, 2 * dr)
    if span == 3 and len(sites) == 3 and list(sites) == [lo, lo + 1, lo + 2] or (span == 3 and len(sites) == 2):
        k1 = min(chi_max, 4 * dl, 2 * dr)
        return svd_cost(4 * dl, 2 * dr) + svd_cost(2 * dl, 2 * k1)
    big = max([dl, dr] + [dims[b] for b in range(lo, hi)])
    return (2 * (span - 2) + 1) * svd_cost(2 * big, 2 * big)  # SWAP-routed (R18)


def plan_layer(gates, dims, n: int, chi_max: int, bounds, lpt: bool = True, small: float = 1e-3):
    """Executing rank of every gate (identical on all ranks: a pure function of its inputs)
    and the predicted load per rank."""
    world = len(bounds)
    owner = [next(r for r, (a, b) in enumerate(bounds) if a <= window(s)[0] < b) for _, s in gates]
    cost = [gate_cost(s, dims, n, chi_max) for _, s in gates]
    loads = [0.0] * world
    ex = list(owner)
    if not gates:
        return ex, loads
    cmax = max(cost)
    for g in sorted(range(len(gates)), key=lambda g: (-cost[g], g)):
        o = owner[g]
        r = o
        if lpt and cost[g] >= small * cmax:
            best = min(range(world), key=lambda x: (loads[x], x))
            if loads[o] > loads[best] + 0.05 * cost[g]:
                r = best
        ex[g] = r
        loads[r] += cost[g]
    return ex, loads


# ------------------------------------------------------------------ SPMD driver
class ShardedMPS:
    """An n-qubit MPS sharded over the ranks of a torch.distributed group (module docstring)."""

    def __init__(self, n: int, p: int, chi_max: int, thr: float = 0.0, engine_factory=None, group=None,
                 lpt: bool = True, host_transport=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.n, self.p, self.chi_max, self.lpt = n, p, chi_max, lpt
        if self.world > n:
            raise ValueError("more ranks than sites")
        self.bounds = [block_range(n, self.world, r) for r in range(self.world)]
        self.lo, self.hi = self.bounds[self.rank]
        self.engine = (engine_factory or CudaEngine)(n, p, chi_max, thr)
        from synth import records as R
        self.rb = R.record_bytes(p)
        self.cb = 2 * self.rb
        self.dims = [1] * (n - 1)
        dev = getattr(self.engine, "device", None)
        backend = dist.get_backend(group) if dist.is_initialized() else "none"
        # gloo moves host tensors only: stage device buffers through the host
        self.host = (backend != "nccl") if host_transport is None else host_transport
        self.dev = dev
        self.stats = {"layers": 0, "migrated_bytes": 0, "loads": [0.0] * self.world, "moved_gates": 0}
        if self.world > 1:  # set up the communicator before the first point-to-point batch
            t = torch.zeros(1, dtype=torch.int32, device=dev if not self.host else None)
            dist.all_reduce(t, group=group)

    # ------------------------------------------------------------ transport
    def owner(self, q: int) -> int:
        return next(r for r, (a, b) in enumerate(self.bounds) if a <= q < b)

    def _peer(self, r: int) -> int:
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def _buf(self, nbytes: int):
        t = self.torch
        if self.dev is None:
            return t.empty(nbytes, dtype=t.uint8)
        return t.empty(nbytes, dtype=t.uint8, device=self.dev)

    def _p2p(self, sends, recvs):
        """sends: [(tensor, peer)], recvs: [(tensor, peer)] -> one batched group; recv tensors
        are filled in place when this returns."""
        if not sends and not recvs:
            return
        dist, t = self.dist, self.torch
        stage = self.host and self.dev is not None
        s_t = [(x.cpu() if stage else x, r) for x, r in sends]
        r_t = [(t.empty(x.numel(), dtype=x.dtype) if stage else x, r) for x, r in recvs]
        ops = [dist.P2POp(dist.isend, x, self._peer(r), group=self.group) for x, r in s_t] + \
              [dist.P2POp(dist.irecv, x, self._peer(r), group=self.group) for x, r in r_t]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        if stage:
            for (dst, _), (src, _) in zip(recvs, r_t):
                dst.copy_(src)

    def _allreduce_sum(self, x):
        if self.world == 1:
            return x
        if self.host and self.dev is not None:
            y = x.cpu()
            self.dist.all_reduce(y, group=self.group)
            x.copy_(y)
        else:
            self.dist.all_reduce(x, group=self.group)
        return x

    # ------------------------------------------------------------ layers
    def site_bytes(self, q: int) -> int:
        dl = self.dims[q - 1] if q > 0 else 1
        dr = self.dims[q] if q < self.n - 1 else 1
        return 2 * dl * dr * self.cb

    def _dl_dr(self, q):
        return (self.dims[q - 1] if q > 0 else 1), (self.dims[q] if q < self.n - 1 else 1)

    def _move_sites(self, moves):
        """moves: [(site, src rank, dst rank)] with the current dims; dst imports."""
        sends, recvs, imports = [], [], []
        for q, src, dst in moves:
            nb = self.site_bytes(q)
            if self.rank == src:
                b = self._buf(nb)
                self.engine.export_site(q, b)
                sends.append((b, dst))
            elif self.rank == dst:
                b = self._buf(nb)
                recvs.append((b, src))
                imports.append((q, b))
            self.stats["migrated_bytes"] += nb
        self._p2p(sends, recvs)
        for q, b in imports:
            dl, dr = self._dl_dr(q)
            self.engine.import_site(q, b, dl, dr)

    def apply_layer(self, gates):
        """gates: list of (U records, global sites); the windows [min, max] must be disjoint."""
        n = self.n
        ex, loads = plan_layer(gates, self.dims, n, self.chi_max, self.bounds, self.lpt) if self.world > 1 \
            else ([0] * len(gates), [0.0])
        for r in range(self.world):
            self.stats["loads"][r] += loads[r]
        self.stats["layers"] += 1
        # 1. migrate in
        moves = []
        for g, (_, s) in enumerate(gates):
            lo, hi = window(s)
            for q in range(lo, hi + 1):
                if self.owner(q) != ex[g]:
                    moves.append((q, self.owner(q), ex[g]))
            self.stats["moved_gates"] += int(any(self.owner(q) != ex[g] for q in range(lo, hi + 1)))
        self._move_sites(moves)
        # 2. compute: this rank's gates in one batched call
        mine = [(U, list(s)) for g, (U, s) in enumerate(gates) if ex[g] == self.rank]
        self.engine.apply_layer(mine)
        if self.world == 1:
            self.dims = self.engine.bond_dims()
            return
        # 3. new Schmidt vectors and dims of every window bond, to every rank (one all-reduce each)
        bonds = [(b, g) for g, (_, s) in enumerate(gates) for b in range(window(s)[0], window(s)[1])]
        caps = [bond_cap(b, n, self.chi_max) for b, _ in bonds]
        offs = [0]
        for c in caps:
            offs.append(offs[-1] + c * self.rb)
        t = self.torch
        lam = self._buf(max(offs[-1], 4))
        lam.zero_()
        dimv = t.zeros(max(len(bonds), 1), dtype=t.int32, device=self.dev if not self.host else None)
        for i, (b, g) in enumerate(bonds):
            if ex[g] == self.rank:
                dimv[i] = self.engine.export_schmidt(b, lam[offs[i]:offs[i + 1]])
        if len(bonds):
            self._allreduce_sum(lam.view(t.int32) if lam.numel() % 4 == 0 else lam)
            self._allreduce_sum(dimv)
            dv = dimv.tolist()  # one host synchronisation per layer
            for i, (b, g) in enumerate(bonds):
                self.dims[b] = int(dv[i])
                if ex[g] != self.rank:
                    self.engine.import_schmidt(b, lam[offs[i]:offs[i] + dv[i] * self.rb], int(dv[i]))
        # 4. migrate out (updated sites back to their owners)
        back = []
        for g, (_, s) in enumerate(gates):
            lo, hi = window(s)
            for q in range(lo, hi + 1):
                if self.owner(q) != ex[g]:
                    back.append((q, ex[g], self.owner(q)))
        self._move_sites(back)

    # ------------------------------------------------------------ queries
    def gather(self, root: int = 0):
        """Site tensors of every rank to `root` (queries)."""
        self._move_sites([(q, self.owner(q), root) for q in range(self.n) if self.owner(q) != root])

    def amplitude(self, bits):
        """Eq. 1 amplitude (complex records) of the global bit string, on every rank."""
        from synth import records as R
        self.gather(0)
        t = self.torch
        if self.rank == 0:
            a = self.engine.amplitude(bits)
            buf = t.from_numpy(a.view(np.uint8).copy())
        else:
            buf = t.zeros(2 * self.rb, dtype=t.uint8)
        if self.world > 1:
            dev_buf = buf if (self.host or self.dev is None) else buf.to(self.dev)
            self.dist.broadcast(dev_buf, self._peer(0), group=self.group)
            buf = dev_buf.cpu()
        return np.frombuffer(buf.numpy().tobytes(), dtype=R.record_dtype(self.p)).copy()

    def schmidt(self, b: int):
        """Schmidt vector of bond b (replicated on every rank)."""
        from synth import records as R
        out = np.zeros(self.dims[b] * self.rb, np.uint8)
        buf = self._buf(self.dims[b] * self.rb)
        self.engine.export_schmidt(b, buf)
        out[:] = buf.cpu().numpy()
        return out.view(R.record_dtype(self.p))
