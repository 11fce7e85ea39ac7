"""Small invocations of every kernel class for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck) — measurement tool, VERDICT r01 "Next round" 8.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py [cfg0|cfg1|cfg3]

cfg0: BASELINE configs[0] (n = 8, depth 8, chi_max 16, 280 bits) through mps_apply_layer, plus
      one U(2), one U(8) and one span-3 gate; cfg1: a configs[1] update batch (4 items,
      chi = 32, 280 bits: contraction, binary64 Jacobi, Newton-Schulz, tensor-core GEMMs,
      refinement sweeps, first-order finish, truncation, split) and the 512-bit tier (2 items,
      chi = 16); cfg3: a depth-4 prefix of configs[3] (U(8) three-site updates).
Prints one line per case with the return codes; the sanitizer's own summary follows."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_3124_b200 as m  # noqa: E402
from synth import gen  # noqa: E402
from tests.test_gpu_configs import layers_of  # noqa: E402


def run_circuit(cfg, depth=None):
    n, p, chi, thr, gates = gen.config_circuit(cfg, depth=depth)
    st = m.MPS(n, p, chi, thr)
    for layer in layers_of(gates):
        st.apply_layer(layer)
    if cfg == 0:
        st.apply(gen.haar_unitary(p, 2, 1, 2, 3), [3])
        st.apply(gen.haar_unitary(p, 8, 1, 2, 4), [2, 3, 4])
        st.apply(gen.haar_unitary(p, 4, 1, 2, 5), [1, 3])
    st.sync()
    a = st.amplitude([0] * n)
    print(f"circuit cfg{cfg}: bond dims {st.bond_dims()} stats {st.stats()['status']}", flush=True)
    st.close()
    return a


def run_batch(p, chi, batch):
    A, B, U = gen.update_batch_inputs(p, chi, batch)
    out = m.update_batch(p, chi, batch, A, B, U)
    print(f"update batch p={p} chi={chi} x{batch}: k {out['k'].tolist()} sweeps {out['sweeps'].tolist()}", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg0", "cfg1"]
    for w in which:
        if w == "cfg0":
            run_circuit(0)
        elif w == "cfg1":
            run_batch(280, 32, 4)
            run_batch(280, 64, 2)
            run_batch(512, 16, 2)
        elif w == "cfg3":
            run_circuit(3, depth=4)
    print("sanitize_case done", flush=True)
