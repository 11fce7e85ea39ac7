"""The oracle's layer-parallel apply is the sequential apply (same arithmetic, disjoint gates)."""
import oracle
from synth import gen
from synth import records as R


def test_layer_parallel_equals_sequential():
    p = 256
    n = 8
    gates = gen.brickwall(n, 3, p, 77, one_site_layer=True) + gen.triples(n, 2, p, 78)
    a = oracle.OracleMPS(n, p, 8, 2.0 ** -128)
    b = oracle.OracleMPS(n, p, 8, 2.0 ** -128)
    for U, s in gates:
        a.apply(U, s)
    # group into layers of disjoint gates in order
    layer, used = [], set()
    for U, s in gates:
        span = set(range(s[0], s[-1] + 1))
        if span & used:
            b.apply_layer(layer, nthreads=4)
            layer, used = [], set()
        layer.append((U, s))
        used |= span
    b.apply_layer(layer, nthreads=4)
    assert a.bond_dims() == b.bond_dims()
    assert (a.to_dense() == b.to_dense()).all()
