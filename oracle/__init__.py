"""ORACLE — test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  It wraps liboracle.so (oracle/*.cpp: own RNE
bignum + plain step-by-step TEBD) with ctypes and shares no
code with paper_1111_3124_b200/.  Records in and out use synth.records.

Parity status of each oracle function:
  arithmetic (+ - x / sqrt, complex x)   pinned: bitwise vs mpmath, vs IEEE binary64 at p=53
  jacobi_svd                              pinned: mpmath.svd_c, 2x2 closed form, known sigma,
                                                  sum sigma^2 = ||A||_F^2, reconstruction
  two-/three-/one-site update, MPS        pinned: dense state vector (n <= 12), GHZ, QFT,
                                                  echo closed forms, paper §3.2 golden
  dense simulator                         pinned: GHZ / QFT closed forms, unitarity
  expectation                             pinned: dense <psi|O|psi> and closed forms
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from synth import records as R

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = ["mp.cpp", "tebd.cpp", "capi.cpp"]

ERRORS = {0: "OK", -1: "EINVAL", -2: "ENOTUNITARY", -3: "ENOCONV", -4: "EZEROBOND",
          -5: "EOVERLAP", -6: "EUNSUPPORTED", -7: "ENOMEM", -10: "ETOOBIG", -99: "EXCEPTION"}


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, s) for s in _SRC] + [os.path.join(_HERE, h) for h in ("mp.hpp", "tebd.hpp")]
    if not force and os.path.exists(_SO) and all(os.path.getmtime(_SO) >= os.path.getmtime(s) for s in srcs):
        return _SO
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-o", _SO] + \
          [os.path.join(_HERE, s) for s in _SRC]
    subprocess.check_call(cmd)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        c_p = ctypes.c_void_p
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_mps_sweeps.restype = ctypes.c_long
        L.orc_mps_free.argtypes = [c_p]
        L.orc_dense_free.argtypes = [c_p]
        L.orc_update2_batch.argtypes = [ctypes.c_int] * 6 + [ctypes.c_double] + [c_p] * 6 + \
            [c_p, c_p, c_p, c_p, c_p, c_p, c_p, ctypes.c_int]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, rc):
        msg = ERRORS.get(rc, str(rc))
        if rc == -99:
            msg += ": " + lib().orc_last_error().decode()
        super().__init__(msg)
        self.rc = rc


def _chk(rc):
    if rc != 0:
        raise OracleError(rc)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def arith(p: int, op: str, a: np.ndarray, b: np.ndarray | None = None, out: np.ndarray | None = None):
    ops = {"add": 0, "sub": 1, "mul": 2, "div": 3, "sqrt": 4, "round": 5, "cmul": 6, "fma": 7}
    o = ops[op]
    n = len(a) // 2 if o == 6 else len(a)
    if out is None:
        out = R.empty(p, len(a))
    _chk(lib().orc_arith(p, o, n, _ptr(a), _ptr(b), _ptr(out)))
    return out


def svd(p: int, A: np.ndarray, M: int, N: int):
    """A: column-major M x N complex records. Returns (sigma[N], X[M*N], V[N*N], sweeps)."""
    sig = R.empty(p, N)
    X = R.empty(p, 2 * M * N)
    V = R.empty(p, 2 * N * N)
    sw = ctypes.c_int(0)
    _chk(lib().orc_svd(p, M, N, _ptr(A), _ptr(sig), _ptr(X), _ptr(V), ctypes.byref(sw)))
    return sig, X, V, sw.value


def theta2(p: int, chi_l: int, chi_m: int, chi_r: int, GL, GR, U):
    """Theta' = U (G_L G_R) of one item (lambda = 1), records in update2_batch's theta layout."""
    out = R.empty(p, 2 * 4 * chi_l * chi_r)
    _chk(lib().orc_theta2(p, chi_l, chi_m, chi_r, _ptr(GL), _ptr(GR), _ptr(U), _ptr(out)))
    return out


def update2_batch(p, batch, chi_l, chi_m, chi_r, chi_max, thr, GL, GR, U, lam_l=None, lam_m=None, lam_r=None,
                  want_theta=False, nthreads=None):
    nsig = min(2 * chi_l, 2 * chi_r)
    sig = R.empty(p, batch * nsig)
    k = np.zeros(batch, np.int32)
    GLo = R.empty(p, batch * 2 * 2 * chi_l * chi_max)
    GRo = R.empty(p, batch * 2 * 2 * chi_max * chi_r)
    lam = R.empty(p, batch * chi_max)
    th = R.empty(p, batch * 2 * 4 * chi_l * chi_r) if want_theta else None
    sw = np.zeros(batch, np.int32)
    nt = nthreads or os.cpu_count()
    rc = lib().orc_update2_batch(p, batch, chi_l, chi_m, chi_r, chi_max, thr, _ptr(GL), _ptr(GR), _ptr(lam_l),
                                 _ptr(lam_m), _ptr(lam_r), _ptr(U), _ptr(sig), _ptr(k), _ptr(GLo), _ptr(GRo),
                                 _ptr(lam), _ptr(th), _ptr(sw), nt)
    _chk(rc)
    return dict(sigma=sig, k=k, GL=GLo, GR=GRo, lam=lam, theta=th, sweeps=sw)


class OracleMPS:
    """Oracle MPS (Vidal Gamma-lambda form, Eq. 1)."""

    def __init__(self, n: int, p: int, chi_max: int, thr: float):
        self.n, self.p = n, p
        h = ctypes.c_void_p()
        _chk(lib().orc_mps_new(n, p, chi_max, ctypes.c_double(thr), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_mps_free(self.h)
            self.h = None

    def apply(self, U: np.ndarray, sites):
        s = (ctypes.c_int * len(sites))(*sites)
        _chk(lib().orc_mps_apply(self.h, _ptr(U), s, len(sites)))

    def apply_layer(self, gates, nthreads=None):
        """gates: list of (U records, sites); disjoint gates computed in parallel threads."""
        n = len(gates)
        ptrs = (ctypes.c_void_p * max(n, 1))(*[U.ctypes.data for U, _ in gates])
        flat = [q for _, s in gates for q in s]
        sf = (ctypes.c_int * max(len(flat), 1))(*flat)
        ks = (ctypes.c_int * max(n, 1))(*[len(s) for _, s in gates])
        _chk(lib().orc_mps_apply_layer(self.h, n, ptrs, sf, ks, nthreads or os.cpu_count()))

    def amplitude(self, bits) -> np.ndarray:
        b = np.asarray(bits, np.uint8)
        out = R.empty(self.p, 2)
        _chk(lib().orc_mps_amplitude(self.h, _ptr(b), _ptr(out)))
        return out

    def to_dense(self) -> np.ndarray:
        out = R.empty(self.p, 2 << self.n)
        _chk(lib().orc_mps_to_dense(self.h, _ptr(out)))
        return out

    def bond_dims(self):
        out = np.zeros(max(self.n - 1, 1), np.int32)
        _chk(lib().orc_mps_bond_dims(self.h, _ptr(out)))
        return out[: self.n - 1].tolist()

    def schmidt(self, bond: int) -> np.ndarray:
        m = ctypes.c_int(0)
        _chk(lib().orc_mps_schmidt(self.h, bond, None, ctypes.byref(m)))
        out = R.empty(self.p, m.value)
        _chk(lib().orc_mps_schmidt(self.h, bond, _ptr(out), ctypes.byref(m)))
        return out

    def get_site(self, s: int):
        ml, mr = ctypes.c_int(0), ctypes.c_int(0)
        _chk(lib().orc_mps_get_site(self.h, s, None, ctypes.byref(ml), ctypes.byref(mr)))
        out = R.empty(self.p, 2 * 2 * ml.value * mr.value)
        _chk(lib().orc_mps_get_site(self.h, s, _ptr(out), ctypes.byref(ml), ctypes.byref(mr)))
        return out, ml.value, mr.value

    def set_schmidt(self, bond: int, lam: np.ndarray):
        _chk(lib().orc_mps_set_schmidt(self.h, bond, _ptr(lam), len(lam)))

    def set_site(self, s: int, G: np.ndarray, ml: int, mr: int):
        _chk(lib().orc_mps_set_site(self.h, s, _ptr(G), ml, mr))

    def norm2(self) -> np.ndarray:
        out = R.empty(self.p, 1)
        _chk(lib().orc_mps_norm2(self.h, _ptr(out)))
        return out

    def expect(self, O: np.ndarray, sites):
        s = (ctypes.c_int * len(sites))(*sites)
        out = R.empty(self.p, 2)
        raw = R.empty(self.p, 2)
        _chk(lib().orc_mps_expect(self.h, _ptr(O), s, len(sites), _ptr(out), _ptr(raw)))
        return out, raw

    def sweeps(self) -> int:
        return lib().orc_mps_sweeps(self.h)


class OracleDense:
    def __init__(self, n: int, p: int):
        self.n, self.p = n, p
        h = ctypes.c_void_p()
        _chk(lib().orc_dense_new(n, p, ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_dense_free(self.h)
            self.h = None

    def apply(self, U, sites):
        s = (ctypes.c_int * len(sites))(*sites)
        _chk(lib().orc_dense_apply(self.h, _ptr(U), s, len(sites)))

    def state(self) -> np.ndarray:
        out = R.empty(self.p, 2 << self.n)
        _chk(lib().orc_dense_get(self.h, _ptr(out)))
        return out


def bench_update2(p: int, chi: int, nthreads: int, max_pairs: int, GL, GR, U):
    """Per-thread (contraction seconds, seconds for max_pairs Jacobi pair evaluations)."""
    tc = np.zeros(nthreads)
    tp = np.zeros(nthreads)
    pd = np.zeros(nthreads, np.int64)
    L = lib()
    L.orc_bench_update2.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long] + [ctypes.c_void_p] * 6
    _chk(L.orc_bench_update2(p, nthreads, chi, max_pairs, _ptr(GL), _ptr(GR), _ptr(U), _ptr(tc), _ptr(tp), _ptr(pd)))
    return tc, tp
