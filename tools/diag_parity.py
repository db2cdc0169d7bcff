"""Print per-tensor norm-wise errors of the device path vs the oracle for every
parity case (used to set / investigate tolerances). Usage:
    python tools/diag_parity.py [bf16|fp32] [n]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle.cnn_ref import OracleNet  # noqa: E402
from paper_1909_12291_b200.network import instantiate  # noqa: E402
from parity_util import CASES, case_genome, make_batch, rel  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
for name, text, shape in CASES:
    g = case_genome(text)
    net = instantiate(g, shape, seed=3)
    o = OracleNet.from_network(net)
    x, y = make_batch(N, shape, seed=11)
    dev = net.to_device(0, prec, max_batch=N)
    dev.keep_grads()
    lg = dev.forward(x)
    ro = o.forward(x)
    acts = []
    for li, layer in enumerate(net.layers):
        shp = layer.out_shape if hasattr(layer, "out_shape") else (layer.out_units,)
        acts.append(rel(dev.activation(li, N, shp), o.outs[li]))
    loss = dev.train_batch(x, y, 1e-3, 0.9)
    rl = o.train_batch(x, y, 1e-3, 0.9)
    gr = []
    for p, (w, b) in enumerate(net.weights):
        gw, gb = dev.get_grads(p, w.shape, b.shape)
        nw, nb, vw, vb = dev.get_params(p, w.shape, b.shape)
        gr.append((rel(gw, o.grads[p][0]), rel(gb, o.grads[p][1]), rel(nw, o.params[p][0])))
    print(f"{name:22s} loss {loss:.6f}/{rl:.6f} logits {rel(lg, ro):.2e}")
    print("   acts", " ".join(f"{a:.1e}" for a in acts))
    print("   dW/db/W", " | ".join(f"{a:.1e} {b:.1e} {c:.1e}" for a, b, c in gr), flush=True)
    net.release()
