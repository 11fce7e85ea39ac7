#!/usr/bin/env python
"""Benchmark: two-site gate updates/s at chi=128, 280-bit (BASELINE.json metric, configs[1]).

A step = one pass of the whole hot path (contraction + gate, one-sided Jacobi SVD,
truncation/renormalisation, split) over one batch of `--batch`
synthetic Theta problems (configs[1]: Gamma_A, Gamma_B in C^{2 x chi x chi} complex
Gaussian, Haar U(4), lambda = 1), inputs resident in HBM.  Multi-GPU (torchrun): every
rank processes its own batch — the batch items are independent, so the path shards with
no data-path collective ("scaling": "weak"); time = max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the oracle (oracle/, the plain CPU implementation) on a bounded
sample of the same workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import gen  # noqa: E402
from synth import records as R  # noqa: E402

def metric_name(chi: int, p: int) -> str:
    return f"two-site gate updates/sec at chi={chi}, {p}-bit"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chi", type=int, default=128)
    ap.add_argument("--prec", type=int, default=280)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--distinct", type=int, default=128, help="distinct seeded items, tiled to --batch")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--oracle-pairs", type=int, default=1500)
    ap.add_argument("--workload", default="cfg1", choices=["cfg1", "cfg4"],
                    help="cfg1: the configs[1] batch (default, BASELINE metric); cfg4: the configs[4] circuit "
                         "(n=64, chi_max=256, 512 bits) sharded over the ranks (strong scaling)")
    ap.add_argument("--depth", type=int, default=12, help="cfg4: circuit depth (configs[4] is 40)")
    ap.add_argument("--no-lpt", action="store_true", help="cfg4: owner-computes placement")
    return ap.parse_args()


def executed_imad_wide(counts, chi: int, p: int) -> float:
    """IMAD.WIDE the p-bit Jacobi kernel executes: every evaluated pair
    computes gamma (4 truncated real products per row, (L-1) + L(L+1)/2 IMAD.WIDE each: 64
    at 280 bits), every sweep refreshes the exact column norms (2 products per entry), and
    the rotation phase executes the digit products counted on the device (counter [4]: the
    zero-digit variants skip known-zero coefficient digits).  The recovery of V and the
    preconditioner are separate kernels (not counted here)."""
    M = 2 * chi
    L = 10 if p <= 280 else 19
    per = (L - 1) + L * (L + 1) // 2
    rot, ev, normw, recw, uprods = counts[:5]
    return float(ev * 4 * M + normw * 2) * per + float(uprods)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thr = threading.Thread(target=self._read, daemon=True)
            self.thr.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def oracle_sample(args, nthreads: int):
    """Bounded sample of the same workload on the oracle: thread t contracts item t and
    runs the first --oracle-pairs Jacobi pair evaluations; extrapolated with the pair
    count of a full update (N(N-1)/2 pairs per sweep x S sweeps)."""
    import oracle
    chi, p = args.chi, args.prec
    A, B, U = gen.update_batch_inputs(p, chi, nthreads)
    tc, tp = oracle.bench_update2(p, chi, nthreads, args.oracle_pairs, A, B, U)
    return tc, tp


def oracle_sweeps(chi: int, p: int):
    """Sweeps of the oracle's own textbook cyclic Jacobi on this workload (final check-only sweep
    included): the mean over the cached full oracle updates of configs[1] items
    (tests/golden/cfg1_p{p}_chi{chi}_item*.json, written by tools/make_cfg1_golden.py, which
    calls only oracle/).  Without such a file: 15.91, the round-robin textbook iteration's mean
    measured on the GPU with the preconditioner off (MPS_NO_PRECOND=1), labelled as such."""
    import glob
    fs = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", f"cfg1_p{p}_chi{chi}_item*.json")))
    sw = [json.load(open(f))["sweeps"] for f in fs]
    if sw:
        return float(np.mean(sw)), f"mean of {len(sw)} complete oracle updates of this workload (tests/golden)"
    return 15.91, "GPU-measured textbook-Jacobi sweeps (MPS_NO_PRECOND=1): no cached oracle update for this chi/p"


def oracle_rate(args, tc, tp, sweeps_mean, nthreads):
    N = 2 * args.chi
    pairs_total = N * (N - 1) / 2 * sweeps_mean
    per_gate = float(np.mean(tc)) + float(np.mean(tp)) / args.oracle_pairs * pairs_total
    return nthreads / per_gate, per_gate


def run_reference(args, rank, world):
    if rank != 0:
        return
    nthreads = os.cpu_count() or 1
    S, S_src = oracle_sweeps(args.chi, args.prec)
    times, vals = [], []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        tc, tp = oracle_sample(args, nthreads)
        dt = time.perf_counter() - t0
        v, per_gate = oracle_rate(args, tc, tp, S, nthreads)
        if it >= args.warmup:
            times.append(dt)
            vals.append(v)
    value = float(np.mean(vals))
    sample = (f"per step: {nthreads} threads, each one chi={args.chi} {args.prec}-bit item: full contraction + first "
              f"{args.oracle_pairs} Jacobi pair evaluations, extrapolated to {S:.2f} sweeps ({S_src}) x N(N-1)/2 pairs")
    line = {"impl": "reference", "metric": metric_name(args.chi, args.prec), "value": value, "unit": "gate_updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": f"u64-limb bignum (oracle), p={args.prec}",
            "data": "synthetic", "config": workload_config(args.batch, args.chi, args.prec, args.distinct, world),
            "cpu_baseline": {"value": value, "unit": "gate_updates/s", "cores": nthreads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "gate_updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(batch, chi, p, nd, world):
    """The config both arms report (the reference arm times a bounded sample of it)."""
    return {"workload": f"configs[1]: batch of {batch} Theta (2chi x 2chi), chi={chi}, {p}-bit, "
                        f"contraction+Jacobi SVD+truncate+split; {nd} distinct seeded items tiled",
            "chi": chi, "prec_bits": p, "batch_per_gpu": batch,
            "l2": "inputs+workspace >> 126 MB L2 (no flush needed)", "parallelism": f"replicas x{world}"}


def run_cfg4(args, rank, world, local):
    """configs[4] (BASELINE: 64 qubits, brick-wall Haar U(4), chi_max = 256, 512 bits) sharded
    over the ranks by paper_1111_3124_b200.dist.ShardedMPS: sites in contiguous
    blocks, LPT placement per layer, NCCL send/recv of migrated site tensors, one all-reduce of
    the new Schmidt vectors per layer.  One timed run of the depth --depth prefix of the
    circuit through the public API (gates uploaded from host records every layer; the
    amplitude of |0...0> read back at the end), CUDA events on each rank's stream, max over
    ranks.  Warm-up: the first two layers on a throw-away state."""
    import torch

    from paper_1111_3124_b200.dist import ShardedMPS
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    n, p, chi, thr, gates = gen.config_circuit(4, depth=args.depth)
    layers, i = [], 0
    for t in range(args.depth):  # brickwall() lists layer t's gates (s = t % 2, t % 2 + 2, ...) in order
        k = len(range(t % 2, n - 1, 2))
        layers.append(gates[i:i + k])
        i += k
    assert i == len(gates)
    for _ in range(max(1, min(args.warmup, 1))):
        W = ShardedMPS(n, p, chi, thr, lpt=not args.no_lpt)
        for layer in layers[:2]:
            W.apply_layer(layer)
        del W
    S = ShardedMPS(n, p, chi, thr, lpt=not args.no_lpt)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        t0 = time.perf_counter()
        per_layer = []
        for layer in layers:
            tl = time.perf_counter()
            S.apply_layer(layer)
            per_layer.append(time.perf_counter() - tl)
        amp = S.amplitude([0] * n)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t0
        if dist is not None:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms, wall * 1e3], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, wall = float(t[0].item()), float(t[1].item()) / 1e3
    ng = len(gates)
    if rank == 0:
        loads = S.stats["loads"]
        line = {
            "metric": f"configs[4] gate updates/sec (n=64, chi_max={chi}, {p}-bit, depth {args.depth})",
            "value": ng / (ms / 1e3), "unit": "gate_updates/s", "n_gpus": world, "steps": 1, "warmup": 1,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": f"int32 radix-2^28 limbs (fixed-point columns) + u32-limb float, p={p}", "data": "synthetic",
            "config": {"workload": f"configs[4] prefix: {args.depth} brick-wall layers of seeded Haar U(4) on 64 qubits, "
                                   f"chi_max={chi}, thr=2^-256, {p}-bit; sites in contiguous blocks of "
                                   f"{n // world} per GPU, {'owner-computes' if args.no_lpt else 'LPT'} placement",
                       "gates": ng, "final_bond_dims_max": max(S.dims), "parallelism": f"site-sharded x{world}"},
            "e2e": {"value": ng / wall, "unit": "gate_updates/s",
                    "h2d_bytes_per_step": int(sum(U.nbytes for U, _ in gates)), "d2h_bytes_per_step": int(amp.nbytes)},
            "sharding": {"predicted_efficiency": sum(loads) / (world * max(loads)) if max(loads) > 0 else 1.0,
                         "gates_moved": S.stats["moved_gates"], "migrated_bytes": S.stats["migrated_bytes"]},
            "per_layer_s": [round(x, 3) for x in per_layer],
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.workload == "cfg4":
        run_cfg4(args, rank, world, local)
        return
    import torch
    import paper_1111_3124_b200 as mps

    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    chi, p, batch = args.chi, args.prec, args.batch
    nd = min(args.distinct, batch)
    # rank r generates items r*nd .. (r+1)*nd-1 (distinct across ranks), tiled to the batch
    A, B, U = gen.update_batch_inputs(p, chi, nd, first=rank * nd)
    reps = (batch + nd - 1) // nd
    A = np.tile(A, reps)[: batch * 4 * chi * chi]
    B = np.tile(B, reps)[: batch * 4 * chi * chi]
    U = np.tile(U, reps)[: batch * 32]
    rb = R.record_bytes(p)
    tA = torch.from_numpy(A.view(np.uint8)).to(dev)
    tB = torch.from_numpy(B.view(np.uint8)).to(dev)
    tU = torch.from_numpy(U.view(np.uint8)).to(dev)
    sig = torch.empty(batch * 2 * chi * rb, dtype=torch.uint8, device=dev)
    kk = torch.empty(batch, dtype=torch.int32, device=dev)
    Ao = torch.empty(batch * 2 * chi * chi * 2 * rb, dtype=torch.uint8, device=dev)
    Bo = torch.empty_like(Ao)
    lam = torch.empty(batch * chi * rb, dtype=torch.uint8, device=dev)
    sw = torch.empty(batch, dtype=torch.int32, device=dev)
    ws = torch.empty(mps.update_batch_workspace(p, chi, batch), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        mps.update_batch_device(p, chi, chi, batch, 0.0, tA, tB, tU, sig, kk, Ao, Bo, lam, sw, ws,
                                stream=stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    launches_per_step = mps.last_launch_count()
    sweeps = sw.cpu().numpy().astype(np.float64)
    ks = kk.cpu().numpy()
    assert (ks == chi).all(), "unexpected truncation in the benchmark workload"

    def barrier():
        if dist is not None:
            dist.barrier()

    mps.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    ms = e0.elapsed_time(e1)
    counts = mps.profile_counts(9)
    q = {name: mps.profile_query(k) for name, k in
         (("jacobi", mps.PROF_JACOBI), ("contraction", mps.PROF_CONTRACT), ("truncate_split", mps.PROF_FINALIZE),
          ("precondition", mps.PROF_PRECOND), ("recover_v", mps.PROF_RECOVER), ("binary64_jacobi", mps.PROF_JDB),
          ("refinement_sweeps", mps.PROF_XS), ("tensor_mma", mps.PROF_TCMMA), ("binary32_jacobi", mps.PROF_JSP))}
    mps.profile_enable(False)
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_items = batch * args.steps * world
    value = total_items / (ms / 1e3)

    # Rooflines of the three kernel classes that make up the step; the one with the
    # largest share of the step is reported as `roofline`, the others under `roofline.kernels`.
    #  * k_tc_mma (every tensor-core GEMM): int8 MACs issued (counted on the device) over the time of
    #    all its launches (CUDA events on the launching stream), against the int8 dense peak = the
    #    measured bf16 peak x 2 (nominal 4.5 / 2.25 PFLOP/s) / 2 (MAC = 2 ops);
    #  * k_jacobi_blk<double> (binary64 block Jacobi, fp64 pipe): algorithmic DFMA per block-pair
    #    visit over its launch time, against the measured DFMA peak;
    #  * k_jacobi_blk<float> (its binary32 first phase, R27; the time includes the hand-over GEMMs):
    #    algorithmic FFMA against 128 lanes x 148 SMs x the SM clock under load.
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_INT_PEAKS.json")))
    dfma_peak = peaks["dfma_per_s"]
    traffic_tab = {}
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        traffic_tab = json.load(open(tfile))
    mp_file = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp_file):
        i8_peak = json.load(open(mp_file))["bf16_tflops"] * 1e12
        i8_src = "MEASURED_PEAKS.json bf16_tflops x 2 (int8/bf16) / 2 (MAC = 2 ops)"
    else:
        i8_peak = 2.25e15
        i8_src = "nominal 4.5 POPS int8 dense (B200_PROFILING.md) / 2"

    def kclass(name, bound, unit, count, peak, peak_src, kernel, counts_note, traffic_key):
        t_ms, n_l = q[name]
        rate = count / (t_ms / 1e3) if t_ms else None
        tr = traffic_tab.get(traffic_key)
        return {"bound": bound, "achieved": rate, "peak": peak, "unit": unit, "frac": (rate / peak) if rate else None,
                "traffic": tr.get("bytes_per_launch") if isinstance(tr, dict) else tr,
                "traffic_source": tr.get("source") if isinstance(tr, dict) else None,
                "kernel": kernel, "peak_source": peak_src, "achieved_counts": counts_note,
                "ops_per_step": count / args.steps, "kernel_ms_per_step": t_ms / args.steps,
                "launches_per_step": n_l / args.steps, "share_of_step": t_ms / ms if ms else None}

    sm_mhz = (clk.summary() or {}).get("sm_mhz") or 1965.0
    classes = {
        "tensor_gemm": kclass("tensor_mma", "tensor", "int8 MAC/s", counts[mps.CNT_TC_MAC], i8_peak, i8_src,
                              "k_tc_mma (all launches: contraction, Newton-Schulz, refinement-sweep, A_1 / P, Gram, "
                              "first-order finish and V-recovery GEMMs; tcgen05 kind::i8, TMEM)",
                              "MMAs issued x 128 x TC_N x 32 int8 MACs (device counter)", f"tc_mma_chi{chi}_p{p}"),
        "binary64_jacobi": kclass("binary64_jacobi", "alu", "DFMA/s", counts[mps.CNT_JDB_DFMA], dfma_peak,
                                  "MEASURED_INT_PEAKS.json dfma_per_s (tools/peaks/int_peak.cu)",
                                  "k_jacobi_blk<double> (binary64 block Jacobi, fp64 pipe)",
                                  "algorithmic DFMA per block-pair visit: Gram 4 nc2(nc2+1)/2 M, inner rotations, "
                                  "W applied to A and V 4 nc2^2 (M + N) (DESIGN.md §4)", f"jacobi_db_chi{chi}_p{p}_batch{batch}"),
        "binary32_jacobi": kclass("binary32_jacobi", "alu", "FFMA/s", counts[mps.CNT_JSP_FFMA], 128 * 148 * sm_mhz * 1e6,
                                  "128 FP32 lanes x 148 SMs x the sampled SM clock (B200_PROFILING.md unit counts)",
                                  "k_jacobi_blk<float> + hand-over (binary32 first phase of the block Jacobi, R27)",
                                  "algorithmic FFMA per block-pair visit (same formula as the binary64 phase)",
                                  f"jacobi_sp_chi{chi}_p{p}_batch{batch}"),
    }
    dom = max(classes, key=lambda k_: classes[k_]["share_of_step"] or 0.0)
    jac_ms, jac_n = q["jacobi"]
    # end to end through the public C API with host buffers (pinned), one step; the device
    # buffers of the timed path are released first (at 512 bits both sets do not fit in HBM)
    e2e = None
    if not args.no_e2e:
        del tA, tB, tU, sig, kk, Ao, Bo, lam, sw, ws
        torch.cuda.empty_cache()
        def pinned(a):
            return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).pin_memory().numpy().view(a.dtype)

        pA, pB, pU = pinned(A), pinned(B), pinned(U)
        rdt = A.dtype
        ob = {"sigma": pinned(np.empty(batch * 2 * chi, rdt)), "k": pinned(np.zeros(batch, np.int32)),
              "GL": pinned(np.empty(batch * 4 * chi * chi, rdt)), "GR": pinned(np.empty(batch * 4 * chi * chi, rdt)),
              "lam": pinned(np.empty(batch * chi, rdt)), "sweeps": pinned(np.zeros(batch, np.int32))}
        mps.update_batch(p, chi, batch, pA, pB, pU, out_buffers=ob)  # warm-up (device arena, host pages)
        barrier()
        t0 = time.perf_counter()
        out = mps.update_batch(p, chi, batch, pA, pB, pU, out_buffers=ob)
        t1 = time.perf_counter()
        barrier()
        dt = t1 - t0
        if dist is not None:
            t = torch.tensor([dt], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        h2d = A.nbytes + B.nbytes + U.nbytes
        d2h = sum(out[k_].nbytes for k_ in ("sigma", "k", "GL", "GR", "lam", "sweeps"))
        e2e = {"value": batch * world / dt, "unit": "gate_updates/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        nthreads = os.cpu_count() or 1
        tc, tp = oracle_sample(args, nthreads)
        S, S_src = oracle_sweeps(chi, p)
        v, per_gate = oracle_rate(args, tc, tp, S, nthreads)
        cpu = {"value": v, "unit": "gate_updates/s", "cores": nthreads, "kind": "oracle",
               "sample": f"{nthreads} threads x one chi={chi} {p}-bit item each: full contraction "
                         f"({np.mean(tc):.1f}s) + first {args.oracle_pairs} Jacobi pairs ({np.mean(tp):.1f}s), "
                         f"extrapolated to {S:.2f} sweeps ({S_src}) x N(N-1)/2 pairs = "
                         f"{per_gate:.0f} s/gate/core"}

    if rank == 0:
        line = {
            "metric": metric_name(chi, p), "value": value, "unit": "gate_updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": f"int32 radix-2^28 limbs (fixed-point columns) + u32-limb float, p={p}",
            "data": "synthetic",
            "config": dict(workload_config(batch, chi, p, nd, world), sweeps_mean=float(np.mean(sweeps))),
            "roofline": dict(classes[dom], dominant=dom,
                             step_ms={k: v[0] / args.steps for k, v in q.items()},
                             kernels={k: v for k, v in classes.items() if k != dom},
                             p_bit_jacobi={"kernel": "k_jacobi (items not closed by the first-order finish, R23)",
                                           "share_of_step": jac_ms / ms if ms else None,
                                           "counters": {"rotations": counts[0], "pair_evals": counts[1],
                                                        "u_digit_products": counts[4], "certified_stops": counts[5]}}),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
