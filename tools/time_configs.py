"""Wall time of BASELINE circuit configs end to end on the GPU MPS (layers through
mps_apply_layer), next to the cached oracle run's time in tests/golden — measurement tool.
usage: python tools/time_configs.py [golden.json ...]
       python tools/time_configs.py --config 3 --depth 16   (GPU only, no cached oracle run)"""
import glob
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root before site-packages
import paper_1111_3124_b200 as m  # noqa: E402
from synth import gen  # noqa: E402
from tests.test_gpu_configs import layers_of  # noqa: E402

if len(sys.argv) > 2 and sys.argv[1] == "--config":
    cfg = int(sys.argv[2])
    depth = int(sys.argv[4]) if len(sys.argv) > 4 else None
    n, p, chi, thr, gates = gen.config_circuit(cfg, depth=depth)
    layers = layers_of(gates)
    st = m.MPS(n, p, chi, thr)
    st.sync()
    t0 = time.perf_counter()
    per = []
    for layer in layers:
        t1 = time.perf_counter()
        st.apply_layer(layer)
        st.sync()
        per.append(round(time.perf_counter() - t1, 3))
    print(json.dumps({"config": cfg, "depth": depth, "n": n, "prec": p, "chi_max": chi, "gates": len(gates),
                      "layers": len(layers), "gpu_seconds": round(time.perf_counter() - t0, 3), "max_bond": max(st.bond_dims()),
                      "seconds_per_layer": per, "stats": st.stats()}), flush=True)
    sys.exit(0)
files = sys.argv[1:] or sorted(glob.glob(os.path.join("tests", "golden", "cfg*_oracle*.json")))
for f in files:
    g = json.load(open(f))
    n, p, chi, thr, gates = gen.config_circuit(g["config"], depth=g["depth"], chi_max=g.get("chi_override"))
    layers = layers_of(gates)
    st = m.MPS(n, p, chi, thr)
    st.sync()
    t0 = time.perf_counter()
    for layer in layers:
        st.apply_layer(layer)
    st.sync()
    dt = time.perf_counter() - t0
    ok = st.bond_dims() == g["bond_dims"]
    print(json.dumps({"golden": os.path.basename(f), "config": g["config"], "n": n, "prec": p, "chi_max": chi,
                      "gates": len(gates), "layers": len(layers), "gpu_seconds": round(dt, 3),
                      "oracle_seconds": round(g["seconds"], 1), "oracle_threads": g["threads"],
                      "bond_dims_equal": ok, "max_bond": max(st.bond_dims())}), flush=True)
