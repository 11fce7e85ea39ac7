"""Debug: Schmidt vectors after every layer of a config circuit, dumped as hex records (compare two runs)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_3124_b200 as m
from synth import gen
from tests.test_gpu_configs import layers_of
cfg, depth, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
n, p, chi, thr, gates = gen.config_circuit(cfg, depth=depth)
st = m.MPS(n, p, chi, thr)
res = []
for li, layer in enumerate(layers_of(gates)):
    st.apply_layer(layer)
    res.append({"layer": li, "sites": [list(map(int, g[1])) for g in layer],
                "dims": st.bond_dims(), "schmidt": [bytes(st.schmidt(b).tobytes()).hex() for b in range(n - 1)]})
json.dump({"p": p, "n": n, "layers": res}, open(out, "w"))
