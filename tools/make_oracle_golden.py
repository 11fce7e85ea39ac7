"""Cache the ORACLE's results for a BASELINE config (calls only oracle/ and synth/).

    python tools/make_oracle_golden.py --config 2 [--depth D] [--threads T]

Writes tests/golden/cfg{idx}_oracle.json: bond dimensions, every Schmidt vector and the
amplitudes of |0...0> plus 64 seeded bitstrings as exact hex records, the stored-state
norm, sweep count and the wall time / core count of the run (the cached oracle run of
SURVEY §8(c) "cfg3, cfg4 end-to-end").  Gates of one layer are disjoint and run through
OracleMPS.apply_layer (parallel threads, unchanged arithmetic).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import gen  # noqa: E402


def layers_of(gates):
    out, cur, used = [], [], set()
    for U, s in gates:
        span = set(range(s[0], s[-1] + 1))
        if span & used:
            out.append(cur)
            cur, used = [], set()
        cur.append((U, s))
        used |= span
    if cur:
        out.append(cur)
    return out


def sample_bits(n, seed, count=64):
    rng = gen.rng(seed, 0xB175)
    return [[0] * n] + rng.integers(0, 2, size=(count, n)).tolist()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--depth", type=int, default=None)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--chi", type=int, default=None, help="override chi_max (scaled-down run)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    n, p, chi, thr, gates = gen.config_circuit(a.config, depth=a.depth, chi_max=a.chi)
    t0 = time.time()
    m = oracle.OracleMPS(n, p, chi, thr)
    ls = layers_of(gates)
    for i, layer in enumerate(ls):
        m.apply_layer(layer, nthreads=a.threads)
        print(f"layer {i + 1}/{len(ls)} dims max {max(m.bond_dims())} t={time.time() - t0:.0f}s", flush=True)
    secs = time.time() - t0
    hexrec = lambda arr: [bytes(arr[i:i + 1].tobytes()).hex() for i in range(len(arr))]
    bits = sample_bits(n, gen.SEED0 + a.config)
    res = {
        "config": a.config, "n": n, "prec": p, "chi_max": chi, "thr": thr,
        "depth": a.depth, "chi_override": a.chi, "gates": len(gates), "layers": len(ls),
        "bond_dims": m.bond_dims(),
        "schmidt": [hexrec(m.schmidt(b)) for b in range(n - 1)],
        "bits": bits,
        "amplitudes": [hexrec(m.amplitude(b)) for b in bits],
        "norm2": hexrec(m.norm2()),
        "sweeps_total": m.sweeps(),
        "seconds": secs, "threads": a.threads, "cpu": platform.processor() or platform.machine(),
        "generator": "tools/make_oracle_golden.py (oracle/ only)",
    }
    out = a.out or os.path.join(ROOT, "tests", "golden", f"cfg{a.config}_oracle{'' if a.depth is None else f'_d{a.depth}'}{'' if a.chi is None else f'_chi{a.chi}'}.json")
    json.dump(res, open(out, "w"))
    print("wrote", out, f"{secs:.0f}s")


if __name__ == "__main__":
    main()
