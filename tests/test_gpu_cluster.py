"""Cluster-cooperative Jacobi (C CTAs per matrix): results are bitwise independent of C
(determinism pin of SURVEY §8(c)/(e): the per-pair arithmetic does not depend on which
CTA/warp performs it).  C is capped through MPS_JACOBI_MAX_CLUSTER in child processes."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_1111_3124_b200 as m
from synth import gen
out = []
for (p, M, N) in [(280, 64, 64), (280, 128, 96), (512, 64, 64)]:
    A = gen.gaussian_cplx(p, M * N, 57, M, N)
    sig, sw, rps, rc = m.svd_batch(p, M, N, 1, A)
    assert rc == 0
    out.append(sig.tobytes().hex())
A, B, U = gen.update_batch_inputs(280, 32, 2, first=7)
r = m.update_batch(280, 32, 2, A, B, U)
out.append(r["sigma"].tobytes().hex() + r["GL"].tobytes().hex() + r["GR"].tobytes().hex())
print("|".join(out))
""" % ROOT


def run(cap):
    env = dict(os.environ, MPS_JACOBI_MAX_CLUSTER=str(cap))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().split("|")


def test_cluster_size_does_not_change_results():
    one = run(1)
    many = run(8)
    assert len(one) == len(many) == 4
    for a, b in zip(one, many):
        assert a == b
