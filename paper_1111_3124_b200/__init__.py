"""Python binding of libmps_b200.so (include/mps_b200.h) — argument marshalling only.

Every step of the gate update runs in the sm_100a kernels behind the C ABI; this
module converts numpy record arrays / torch device tensors to pointers and raises
on error statuses.  There is no CPU fallback: if the CUDA library is missing or no
CUDA device is present, calls fail loudly (MpsError / ImportError).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("MPS_B200_SO") or os.path.join(_HERE, "libmps_b200.so")  # env: dev A/B builds

STATUS = {0: "MPS_OK", -1: "MPS_EINVAL", -2: "MPS_ENOTUNITARY", -3: "MPS_ENOCONV", -4: "MPS_EZEROBOND",
          -5: "MPS_EOVERLAP", -6: "MPS_EUNSUPPORTED", -7: "MPS_ENOMEM", -8: "MPS_ECUDA", -9: "MPS_ENCCL",
          -10: "MPS_ETOOBIG"}

# every symbol include/mps_b200.h declares
EXPORTS = ["mps_profile_counts", "mps_profile_counts_n", "mps_rdo", "mps_init_block", "mps_block_dims", "mps_block_export_first", "mps_block_boundary_apply",
           "mps_block_import_first", "mps_amplitude_block", "mps_record_bytes", "mps_strerror", "mps_max_chi", "mps_init", "mps_free", "mps_set_stream",
           "mps_apply_gate", "mps_apply_layer", "mps_amplitude", "mps_expect", "mps_norm2", "mps_to_dense",
           "mps_sync", "mps_n_qubits", "mps_bond_dims", "mps_schmidt", "mps_get_site", "mps_set_schmidt",
           "mps_set_site", "mps_stats", "mps_bench_update_batch", "mps_update_batch_workspace",
           "mps_update_batch_device", "mps_last_launch_count", "mps_profile_enable", "mps_profile_query",
           "mps_svd_batch", "mps_debug_mpf"]


class MpsError(RuntimeError):
    def __init__(self, rc: int, what: str = ""):
        super().__init__(f"{STATUS.get(rc, rc)}{': ' + what if what else ''}")
        self.rc = rc


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise ImportError(f"{_SO} not built: run python -c 'import __graft_entry__ as g; g.build()'")
        L = ctypes.CDLL(_SO)
        vp, ci, cd, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
        L.mps_record_bytes.restype = sz
        L.mps_strerror.restype = ctypes.c_char_p
        L.mps_update_batch_workspace.restype = sz
        L.mps_update_batch_workspace.argtypes = [ci, ci, ci]
        L.mps_bench_update_batch.argtypes = [ci, ci, ci, ci, cd] + [vp] * 6 + [vp, vp, vp, vp, vp, vp, vp, vp]
        L.mps_update_batch_device.argtypes = [ci, ci, ci, ci, cd] + [vp] * 6 + [vp] * 8
        L.mps_profile_enable.argtypes = [ci]
        L.mps_profile_query.argtypes = [ci, vp, vp]
        L.mps_svd_batch.argtypes = [ci, ci, ci, ci, vp, vp, vp, vp]
        L.mps_debug_mpf.argtypes = [ci, ci, ci, vp, vp, vp]
        if hasattr(L, "mps_init"):
            L.mps_init.argtypes = [ctypes.POINTER(vp), ci, ci, ci, cd]
            L.mps_free.argtypes = [vp]
            L.mps_set_stream.argtypes = [vp, vp]
            L.mps_apply_gate.argtypes = [vp, vp, vp, ci]
            L.mps_apply_layer.argtypes = [vp, ci, vp, vp, vp]
            L.mps_amplitude.argtypes = [vp, vp, vp]
            L.mps_expect.argtypes = [vp, vp, vp, ci, vp]
            L.mps_norm2.argtypes = [vp, vp]
            L.mps_to_dense.argtypes = [vp, vp]
            L.mps_sync.argtypes = [vp]
            L.mps_n_qubits.argtypes = [vp]
            L.mps_bond_dims.argtypes = [vp, vp]
            L.mps_schmidt.argtypes = [vp, ci, vp, vp]
            L.mps_get_site.argtypes = [vp, ci, vp, vp, vp]
            L.mps_set_schmidt.argtypes = [vp, ci, vp, ci]
            L.mps_set_site.argtypes = [vp, ci, vp, ci, ci]
            L.mps_stats.argtypes = [vp, vp, sz]
        _lib = L
    return _lib


def _chk(rc: int, what: str = ""):
    if rc != 0:
        raise MpsError(rc, what)


def _p(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    if hasattr(a, "data_ptr"):  # torch tensor
        return ctypes.c_void_p(a.data_ptr())
    return a


def record_bytes(p: int) -> int:
    return int(lib().mps_record_bytes(p))


def _empty(p, n):
    from synth import records as R  # record dtype helper (format only)
    return R.empty(p, n)


def update_batch(p: int, chi: int, batch: int, A, B, U, lam_l=None, lam_m=None, lam_r=None, chi_max: int | None = None,
                 thr: float = 0.0, theta: bool = False, stream=None, out_buffers=None):
    """Batched two-site update through mps_bench_update_batch (host records in/out).
    out_buffers: optional dict of preallocated (e.g. pinned) output arrays with the keys and
    shapes this function returns (sigma, k, GL, GR, lam, sweeps)."""
    chi_max = chi_max or chi
    out = {}
    if theta:
        th = _empty(p, batch * 2 * 4 * chi * chi)
        rc = lib().mps_bench_update_batch(p, chi, chi_max, batch, thr, _p(A), _p(B), _p(lam_l), _p(lam_m), _p(lam_r),
                                          _p(U), None, None, None, None, None, None, _p(th), stream)
        _chk(rc, "mps_bench_update_batch")
        return {"theta": th}
    ob = out_buffers or {}
    sig = ob.get("sigma", None)
    sig = _empty(p, batch * 2 * chi) if sig is None else sig
    k = ob.get("k", None)
    k = np.zeros(batch, np.int32) if k is None else k
    Ao = ob.get("GL", None)
    Ao = _empty(p, batch * 2 * 2 * chi * chi_max) if Ao is None else Ao
    Bo = ob.get("GR", None)
    Bo = _empty(p, batch * 2 * 2 * chi_max * chi) if Bo is None else Bo
    lam = ob.get("lam", None)
    lam = _empty(p, batch * chi_max) if lam is None else lam
    sw = ob.get("sweeps", None)
    sw = np.zeros(batch, np.int32) if sw is None else sw
    rc = lib().mps_bench_update_batch(p, chi, chi_max, batch, thr, _p(A), _p(B), _p(lam_l), _p(lam_m), _p(lam_r),
                                      _p(U), _p(sig), _p(k), _p(Ao), _p(Bo), _p(lam), _p(sw), None, stream)
    _chk(rc, "mps_bench_update_batch")
    out.update(sigma=sig, k=k, GL=Ao, GR=Bo, lam=lam, sweeps=sw)
    return out


def update_batch_workspace(p: int, chi: int, batch: int) -> int:
    return int(lib().mps_update_batch_workspace(p, chi, batch))


def update_batch_device(p, chi, chi_max, batch, thr, dA, dB, dU, dsigma, dk, dA_out, dB_out, dlam, dsweeps, dws,
                        stream=None, dlam_l=None, dlam_m=None, dlam_r=None):
    """Same on torch CUDA tensors (no host copies)."""
    rc = lib().mps_update_batch_device(p, chi, chi_max, batch, thr, _p(dA), _p(dB), _p(dlam_l), _p(dlam_m),
                                       _p(dlam_r), _p(dU), _p(dsigma), _p(dk), _p(dA_out), _p(dB_out), _p(dlam),
                                       _p(dsweeps), _p(dws), stream)
    _chk(rc, "mps_update_batch_device")


def last_launch_count() -> int:
    return int(lib().mps_last_launch_count())


def svd_batch(p: int, M: int, N: int, batch: int, A):
    """sigma (descending), sweeps, rotations per sweep of column-major M x N matrices."""
    n = min(M, N)
    sig = _empty(p, batch * n)
    sw = np.zeros(batch, np.int32)
    rps = np.zeros(batch * 64, np.int32)
    rc = lib().mps_svd_batch(p, M, N, batch, _p(A), _p(sig), _p(sw), _p(rps))
    if rc not in (0, -3):
        _chk(rc, "mps_svd_batch")
    return sig, sw, rps.reshape(batch, 64), rc


def debug_mpf(p: int, op: str, a, b=None):
    ops = {"add": 0, "sub": 1, "mul": 2, "div": 3, "sqrt": 4, "rsqrt": 5, "recip": 6, "copy": 7, "fixed": 8}
    out = _empty(p, len(a))
    _chk(lib().mps_debug_mpf(p, ops[op], len(a), _p(a), _p(b), _p(out)), "mps_debug_mpf")
    return out


PROF_JACOBI, PROF_CONTRACT, PROF_FINALIZE, PROF_PRECOND, PROF_RECOVER = 0, 1, 2, 3, 4
PROF_JDB, PROF_XS, PROF_TCMMA, PROF_JSP = 5, 6, 7, 8  # binary64 block Jacobi, refinement sweeps, k_tc_mma, binary32 block Jacobi + hand-over (inside the above)
CNT_JDB_DFMA, CNT_TC_MAC, CNT_JSP_FFMA = 6, 7, 8  # profile_counts(): algorithmic DFMA / FFMA of the block Jacobi phases, int8 MACs of k_tc_mma


def profile_enable(on: bool = True):
    _chk(lib().mps_profile_enable(1 if on else 0))


def profile_counts(n: int = 5):
    out = (ctypes.c_longlong * n)()
    _chk(lib().mps_profile_counts_n(out, n))
    return list(out)


def profile_query(which: int):
    ms = ctypes.c_double(0)
    n = ctypes.c_int(0)
    _chk(lib().mps_profile_query(which, ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


class MPS:
    """The on-device MPS state (mps_init ... mps_free).  Records in / out are synth.records arrays."""

    def __init__(self, n: int, p: int, chi_max: int, thr: float = 0.0, stream=None):
        self.n, self.p = n, p
        h = ctypes.c_void_p()
        _chk(lib().mps_init(ctypes.byref(h), n, p, chi_max, thr), "mps_init")
        self.h = h
        if stream is not None:
            _chk(lib().mps_set_stream(self.h, stream))

    def close(self):
        if getattr(self, "h", None):
            lib().mps_free(self.h)
            self.h = None

    __del__ = close

    def apply(self, U, sites):
        s = (ctypes.c_int * len(sites))(*sites)
        _chk(lib().mps_apply_gate(self.h, _p(U), s, len(sites)), "mps_apply_gate")

    def apply_layer(self, gates):
        """gates: list of (U records, sites)."""
        n = len(gates)
        ptrs = (ctypes.c_void_p * max(n, 1))(*[U.ctypes.data for U, _ in gates])
        flat = [q for _, s in gates for q in s]
        sf = (ctypes.c_int * max(len(flat), 1))(*flat)
        ks = (ctypes.c_int * max(n, 1))(*[len(s) for _, s in gates])
        _chk(lib().mps_apply_layer(self.h, n, ptrs, sf, ks), "mps_apply_layer")

    def amplitude(self, bits):
        b = np.asarray(bits, np.uint8)
        out = _empty(self.p, 2)
        _chk(lib().mps_amplitude(self.h, _p(b), _p(out)), "mps_amplitude")
        return out

    def to_dense(self):
        out = _empty(self.p, 2 << self.n)
        _chk(lib().mps_to_dense(self.h, _p(out)), "mps_to_dense")
        return out

    def rdo(self, sites):
        """Reduced density operator, 2^k x 2^k complex records, row-major."""
        k = len(sites)
        s = (ctypes.c_int * k)(*sites)
        out = _empty(self.p, 2 << (2 * k))
        lib().mps_rdo.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        _chk(lib().mps_rdo(self.h, s, k, _p(out)), "mps_rdo")
        return out

    def norm2(self):
        out = _empty(self.p, 1)
        _chk(lib().mps_norm2(self.h, _p(out)), "mps_norm2")
        return out

    def expect(self, O, sites):
        s = (ctypes.c_int * len(sites))(*sites)
        out = _empty(self.p, 2)
        _chk(lib().mps_expect(self.h, _p(O), s, len(sites), _p(out)), "mps_expect")
        return out

    def bond_dims(self):
        out = np.zeros(max(self.n - 1, 1), np.int32)
        _chk(lib().mps_bond_dims(self.h, _p(out)), "mps_bond_dims")
        return out[: self.n - 1].tolist()

    def schmidt(self, bond: int):
        m = ctypes.c_int(0)
        _chk(lib().mps_schmidt(self.h, bond, None, ctypes.byref(m)))
        out = _empty(self.p, m.value)
        _chk(lib().mps_schmidt(self.h, bond, _p(out), ctypes.byref(m)))
        return out

    def get_site(self, s: int):
        ml, mr = ctypes.c_int(0), ctypes.c_int(0)
        _chk(lib().mps_get_site(self.h, s, None, ctypes.byref(ml), ctypes.byref(mr)))
        out = _empty(self.p, 4 * ml.value * mr.value)
        _chk(lib().mps_get_site(self.h, s, _p(out), ctypes.byref(ml), ctypes.byref(mr)))
        return out, ml.value, mr.value

    def set_schmidt(self, bond: int, lam):
        _chk(lib().mps_set_schmidt(self.h, bond, _p(lam), len(lam)))

    def set_site(self, s: int, G, ml: int, mr: int):
        _chk(lib().mps_set_site(self.h, s, _p(G), ml, mr))

    def sync(self):
        _chk(lib().mps_sync(self.h), "mps_sync")

    def stats(self) -> dict:
        import json
        buf = ctypes.create_string_buffer(1 << 16)
        _chk(lib().mps_stats(self.h, buf, len(buf)))
        return json.loads(buf.value.decode())
