"""Debug: per-sweep certified-stop bounds of the p-bit Jacobi (MPS_JACOBI_TRACE) for a few
configs[1] items, to see how far the preconditioner brings the columns.  GPU only.
  MPS_JACOBI_TRACE=4 python tools/trace_sweeps.py [chi] [p] [batch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_3124_b200 as m  # noqa: E402
from synth import gen  # noqa: E402

chi = int(sys.argv[1]) if len(sys.argv) > 1 else 128
p = int(sys.argv[2]) if len(sys.argv) > 2 else 280
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 4
A, B, U = gen.update_batch_inputs(p, chi, batch)
out = m.update_batch(p, chi, batch, A, B, U, thr=2.0 ** -140)
import collections
print("sweeps", dict(collections.Counter(int(x) for x in out["sweeps"])), "k", dict(collections.Counter(int(x) for x in out["k"])), flush=True)
