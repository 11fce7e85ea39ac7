"""Site-sharded block states on one GPU (the C-ABI part of SURVEY §8(e)): two blocks
[0, n/2) and [n/2, n) exchange the block-edge halo with device copies in exactly the
order paper_1111_3124_b200/dist.py uses with NCCL; the result must be BITWISE equal to
the single-state run in every site tensor and Schmidt vector (the per-gate decomposition
depends only on the tensors); amplitudes chained across the blocks (the partial vector
crosses the edge rounded to p-bit records) agree within tau."""
import ctypes

import mpmath
import numpy as np
import pytest

from synth import gen
from synth import records as R
from tests.helpers import cplx, tau

pytestmark = pytest.mark.gpu


def run_blocks(n, p, chi, thr, layers):
    from paper_1111_3124_b200.dist import CudaBlockEngine
    h = n // 2
    A = CudaBlockEngine(n, 0, h, p, chi, thr)
    B = CudaBlockEngine(n, h, n, p, chi, thr)
    for layer in layers:
        la, lb, edge = [], [], None
        for U, s in layer:
            if s[-1] < h:
                la.append((U, list(s)))
            elif s[0] >= h:
                lb.append((U, [q - h for q in s]))
            else:
                edge = U
        if edge is not None:
            G, lam, ml, mr = B.export_first()
        A.apply_layer(la)
        B.apply_layer(lb)
        if edge is not None:
            Gout, lam_mid, k = A.boundary_apply(edge, G, mr, lam if len(lam) else None)
            B.import_first(Gout, lam_mid, k)
    return A, B


@pytest.mark.parametrize("p,n,chi,depth", [(280, 8, 16, 6), (512, 10, 8, 5)])
def test_two_blocks_equal_single_state(p, n, chi, depth):
    import paper_1111_3124_b200 as m
    thr = 2.0 ** -(p // 2)
    layers = [[(gen.haar_unitary(p, 4, 4343, t, s), (s, s + 1)) for s in range(t % 2, n - 1, 2)] for t in range(depth)]
    A, B = run_blocks(n, p, chi, thr, layers)
    ref = m.MPS(n, p, chi, thr)
    for layer in layers:
        ref.apply_layer(layer)
    assert A.dims()[1] == B.dims()[0] == ref.bond_dims()[n // 2 - 1]
    L = m.lib()
    for blk, off in ((A, 0), (B, n // 2)):
        for q in range(blk.n):
            ml, mr = ctypes.c_int(0), ctypes.c_int(0)
            L.mps_get_site(blk.h, q, None, ctypes.byref(ml), ctypes.byref(mr))
            g = R.empty(p, 4 * ml.value * mr.value)
            L.mps_get_site(blk.h, q, g.ctypes.data_as(ctypes.c_void_p), ctypes.byref(ml), ctypes.byref(mr))
            want, wl, wr = ref.get_site(off + q)
            assert (ml.value, mr.value) == (wl, wr)
            assert g.tobytes() == want.tobytes(), (off + q)
    rng = np.random.default_rng(1)
    for bits in [[0] * n, [1] * n] + rng.integers(0, 2, (6, n)).tolist():
        v = A.amplitude_block(bits[: n // 2], None)
        a = cplx(B.amplitude_block(bits[n // 2:], v))[0]
        w = cplx(ref.amplitude(bits))[0]
        with mpmath.workprec(2 * p):
            assert abs(a - w) <= tau(p) * max(abs(w), mpmath.mpf(2) ** (-n / 2.0))
