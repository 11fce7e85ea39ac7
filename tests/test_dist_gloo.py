"""Multi-rank path of the site-sharded MPS on CPU ranks over gloo.

The sharded driver (paper_1111_3124_b200/dist.py: LPT placement, batched point-to-point
migration of site tensors, one all-reduce of the new Schmidt vectors per layer) runs with
the test-only oracle engine (tests/dist_oracle_engine.py) as its arithmetic.  Every gate
is the same oracle update on the same tensors wherever it runs, so the result must be
BITWISE equal to a single-process oracle MPS: every Schmidt vector, every site tensor
(gathered on rank 0) and the amplitudes.  The circuits put two-site gates, three-site U(8)
gates and span-3 two-qubit gates across the block edges, with
world sizes 2 and 3 (uneven blocks, so LPT moves gates off their owners).

plan_layer itself is pinned on configs[4]'s saturated bond profile against SURVEY §8(e):
owner-computes gives E(8) ~ 0.74, LPT ~ 0.98."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from synth import gen

N, P, CHI, THR = 9, 256, 8, 2.0 ** -128


def layers():
    out = []
    for t in range(4):  # brick-wall U(4)
        out.append([(gen.haar_unitary(P, 4, 4242, t, s), (s, s + 1)) for s in range(t % 2, N - 1, 2)])
    for t in range(4, 7):  # U(8) triples at offsets 0, 1, 2 (every block edge is crossed)
        o = t % 3
        out.append([(gen.haar_unitary(P, 8, 4242, t, s), (s, s + 1, s + 2)) for s in range(o, N - 2, 3)])
    # span-3 two-qubit gates (embedded into U(8)) and one-qubit gates
    out.append([(gen.haar_unitary(P, 4, 4242, 7, s), (s, s + 2)) for s in (0, 3, 6)])
    out.append([(gen.haar_unitary(P, 2, 4242, 8, s), (s,)) for s in range(N)])
    out.append([(gen.haar_unitary(P, 4, 4242, 9, s), (s, s + 1)) for s in range(0, N - 1, 2)])
    return out


def bitlist():
    return [[0] * N, [1] * N, [0, 1] * (N // 2) + [0], [1, 1, 0, 1, 0, 0, 1, 0, 1]]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1111_3124_b200.dist import ShardedMPS
    from tests.dist_oracle_engine import OracleEngine
    S = ShardedMPS(N, P, CHI, THR, engine_factory=OracleEngine)
    for layer in layers():
        S.apply_layer(layer)
    lam = [S.schmidt(b).tobytes().hex() for b in range(N - 1)]
    amps = [S.amplitude(b).tobytes().hex() for b in bitlist()]  # gathers every site on rank 0
    sites = [S.engine.m.get_site(s)[0].tobytes().hex() for s in range(N)] if rank == 0 else None
    q.put((rank, lam, amps, sites, S.dims, S.stats["moved_gates"]))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gloo_bitwise_equals_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, lam, amps, sites, dims, moved = q.get(timeout=900)
        res[r] = (lam, amps, sites, dims, moved)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = oracle.OracleMPS(N, P, CHI, THR)
    for layer in layers():
        ref.apply_layer(layer, nthreads=1)
    want_lam = [ref.schmidt(b).tobytes().hex() for b in range(N - 1)]
    want_amp = [ref.amplitude(b).tobytes().hex() for b in bitlist()]
    want_sites = [ref.get_site(s)[0].tobytes().hex() for s in range(N)]
    for r in range(world):
        assert res[r][0] == want_lam, r          # Schmidt vectors replicated, bitwise
        assert res[r][1] == want_amp, r          # amplitudes on every rank, bitwise
        assert res[r][3] == ref.bond_dims(), r
    assert res[0][2] == want_sites               # every site tensor, bitwise
    if world == 3:
        assert res[0][4] > 0                     # LPT ran some gates away from their owners


def test_plan_layer_configs4_efficiency():
    """configs[4] (n = 64, chi_max = 256) at saturation, 8 ranks of 8 sites (SURVEY §8(e)
    efficiency analysis): per two layers, owner-computes E(8) ~ 0.74; LPT >= 0.95."""
    from paper_1111_3124_b200.dist import block_range, plan_layer
    n, chi, world = 64, 256, 8
    dims = [min(chi, 2 ** min(b + 1, n - b - 1)) for b in range(n - 1)]
    bounds = [block_range(n, world, r) for r in range(world)]
    E = {}
    for lpt in (False, True):
        tot = [0.0] * world
        for off in (0, 1):
            gates = [(None, (s, s + 1)) for s in range(off, n - 1, 2)]
            _, loads = plan_layer(gates, dims, n, chi, bounds, lpt=lpt)
            E[(lpt, off)] = sum(loads) / (world * max(loads))
            tot = [a + b for a, b in zip(tot, loads)]
    assert 0.70 <= E[(False, 0)] <= 0.78 and 0.70 <= E[(False, 1)] <= 0.78, E
    assert E[(True, 0)] >= 0.95 and E[(True, 1)] >= 0.95, E
