"""Multi-rank path of the site-sharded MPS on CPU: world_size 2 over gloo.
The sharded driver (paper_1111_3124_b200/dist.py) exchanges block-edge halos by
torch.distributed point-to-point; the local arithmetic is the test-only oracle engine.
Result: equal to the single-process oracle MPS (bond updates are the same oracle update
on the same tensors, so Schmidt vectors agree bitwise; amplitudes within tau)."""
import os
import socket

import mpmath
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from synth import gen
from tests.helpers import cplx, tau

N, P, CHI, THR, DEPTH = 8, 256, 8, 2.0 ** -128, 5


def layers():
    out = []
    for t in range(DEPTH):
        out.append([(gen.haar_unitary(P, 4, 4242, t, s), (s, s + 1)) for s in range(t % 2, N - 1, 2)])
    return out


def bitlist():
    return [[0] * N, [1] * N, [0, 1] * (N // 2), [1, 1, 0, 1, 0, 0, 1, 0]]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1111_3124_b200.dist import ShardedMPS
    from tests.dist_oracle_engine import OracleBlockEngine
    S = ShardedMPS(N, P, CHI, THR, engine_factory=OracleBlockEngine)
    for layer in layers():
        S.apply_layer(layer)
    amps = [S.amplitude(b).tobytes().hex() for b in bitlist()]
    lam_edge = S.engine.lam_er.tobytes().hex() if rank == 0 else S.engine.lam_el.tobytes().hex()
    q.put((rank, amps, lam_edge))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2])
def test_sharded_two_ranks_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, amps, lam = q.get(timeout=600)
        res[r] = (amps, lam)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # reference: single-process oracle MPS
    ref = oracle.OracleMPS(N, P, CHI, THR)
    for layer in layers():
        for U, s in layer:
            ref.apply(U, s)
    import numpy as np
    from synth import records as R
    # the mirrored edge Schmidt vector is identical on both ranks and equals the oracle's
    assert res[0][1] == res[1][1] == ref.schmidt(N // 2 - 1).tobytes().hex()
    for i, bits in enumerate(bitlist()):
        want = cplx(ref.amplitude(bits))[0]
        for r in range(world):
            got = cplx(np.frombuffer(bytes.fromhex(res[r][0][i]), dtype=R.record_dtype(P)))[0]
            with mpmath.workprec(2 * P):
                assert abs(got - want) <= tau(P), (r, bits, got, want)
