"""Site-sharded block states on one GPU (the C-ABI part of SURVEY §8(e)): two blocks
[0, n/2) and [n/2, n) exchange the block-edge halo with device copies in exactly the
order paper_1111_3124_b200/dist.py uses with NCCL; the result must be BITWISE equal to
the single-state run (the per-gate decomposition depends only on the tensors)."""
import numpy as np
import pytest

from synth import gen

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
    rng = np.random.default_rng(1)
    for bits in [[0] * n, [1] * n] + rng.integers(0, 2, (6, n)).tolist():
        v = A.amplitude_block(bits[: n // 2], None)
        a = B.amplitude_block(bits[n // 2:], v)
        assert a.tobytes() == ref.amplitude(bits).tobytes()
