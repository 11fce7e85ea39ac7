"""The site-sharded driver with the CUDA engine (paper_1111_3124_b200/dist.py).

* Several ranks sharing cuda:0 (gloo transport with host staging; the kernels of different
  ranks never wait on one another, only the host exchanges do): 2 and 3 ranks run a circuit
  whose two-site, three-site U(8) and span-3 gates cross every block edge, with LPT moving
  gates off their owners.  Result BITWISE equal to the single-process run of the same layers
  (every Schmidt vector, every site tensor, amplitudes): the per-gate arithmetic does not
  depend on placement or batch composition (SURVEY §8(c) pin "1-GPU versus k-GPU bitwise").
* NCCL over NVLink, one rank per GPU (torchrun): the same check, skipped when fewer than two
  GPUs are visible (the pool's boxes have one)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from synth import gen

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def circuit(n, p, seed):
    out = []
    for t in range(6):
        out.append([(gen.haar_unitary(p, 4, seed, t, s), (s, s + 1)) for s in range(t % 2, n - 1, 2)])
    for t in range(6, 9):
        o = t % 3
        out.append([(gen.haar_unitary(p, 8, seed, t, s), (s, s + 1, s + 2)) for s in range(o, n - 2, 3)])
    out.append([(gen.haar_unitary(p, 4, seed, 9, s), (s, s + 2)) for s in range(0, n - 2, 4)])
    out.append([(gen.haar_unitary(p, 4, seed, 10, s), (s, s + 1)) for s in range(1, n - 1, 2)])
    return out


def bitlist(n):
    g = gen.rng(0xB175, n)
    return [[0] * n] + g.integers(0, 2, size=(6, n)).tolist()


def run(n, p, chi, thr, seed, out_path):
    """Body of one rank (or the single-process reference when not distributed)."""
    import json

    import torch
    import torch.distributed as dist

    from paper_1111_3124_b200.dist import ShardedMPS
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) if os.environ.get("MPS_SHARD_NCCL") else 0)
    S = ShardedMPS(n, p, chi, thr)
    for layer in circuit(n, p, seed):
        S.apply_layer(layer)
    lam = [S.schmidt(b).tobytes().hex() for b in range(n - 1)]
    amps = [S.amplitude(b).tobytes().hex() for b in bitlist(n)]
    sites = [S.engine.mps.get_site(q)[0].tobytes().hex() for q in range(n)] if rank == 0 else None
    res = {"rank": rank, "world": world, "lam": lam, "amps": amps, "sites": sites, "dims": S.dims,
           "moved": S.stats["moved_gates"], "migrated_bytes": S.stats["migrated_bytes"]}
    with open(f"{out_path}.{rank}", "w") as f:
        json.dump(res, f)


WORKER = """
import os, sys
sys.path.insert(0, {root!r})
import torch, torch.distributed as dist
from tests.test_gpu_sharded import run
backend = "nccl" if os.environ.get("MPS_SHARD_NCCL") else "gloo"
if backend == "nccl":
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
else:
    dist.init_process_group("gloo")
run({n}, {p}, {chi}, {thr!r}, {seed}, {out!r})
dist.barrier()
dist.destroy_process_group()
"""


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch(world, n, p, chi, thr, seed, out, nccl=False):
    script = out + ".py"
    with open(script, "w") as f:
        f.write(WORKER.format(root=ROOT, n=n, p=p, chi=chi, thr=thr, seed=seed, out=out))
    env = dict(os.environ)
    if nccl:
        env["MPS_SHARD_NCCL"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", script]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    import json
    return [json.load(open(f"{out}.{k}")) for k in range(world)]


CASES = [(14, 512, 32, 2.0 ** -256, 31), (12, 280, 64, 1e-60, 32)]


@pytest.fixture(scope="module", params=CASES, ids=[f"n{c[0]}_p{c[1]}_chi{c[2]}" for c in CASES])
def reference(request, tmp_path_factory):
    n, p, chi, thr, seed = request.param
    out = str(tmp_path_factory.mktemp("ref") / "ref")
    run(n, p, chi, thr, seed, out)
    import json
    return request.param, json.load(open(out + ".0"))


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_sharing_one_gpu_bitwise(world, reference, tmp_path):
    (n, p, chi, thr, seed), ref = reference
    res = launch(world, n, p, chi, thr, seed, str(tmp_path / "shard"))
    for r in res:
        assert r["lam"] == ref["lam"], r["rank"]
        assert r["amps"] == ref["amps"], r["rank"]
        assert r["dims"] == ref["dims"], r["rank"]
    assert res[0]["sites"] == ref["sites"]
    print(f"n={n} p={p} chi={chi} world={world}: dims {max(ref['dims'])}, gates moved by LPT {res[0]['moved']}, "
          f"migrated {res[0]['migrated_bytes'] / 1e6:.1f} MB")


def test_nccl_two_gpus_bitwise(reference, tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("NCCL sharding needs >= 2 GPUs (this box has one)")
    (n, p, chi, thr, seed), ref = reference
    res = launch(2, n, p, chi, thr, seed, str(tmp_path / "nccl"), nccl=True)
    for r in res:
        assert r["lam"] == ref["lam"] and r["amps"] == ref["amps"]
    assert res[0]["sites"] == ref["sites"]
