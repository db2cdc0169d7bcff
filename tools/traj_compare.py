"""Multi-step loss trajectories on fixed batches: device bf16 / fp32 vs oracle.
    python tools/traj_compare.py <parity case name> <batch> <steps>
"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle.cnn_ref import OracleNet  # noqa: E402
from paper_1909_12291_b200.network import instantiate  # noqa: E402
from parity_util import CASES, case_genome, rel  # noqa: E402
from paper_1909_12291_b200.patches import default_splits  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_g15"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 12
text, shape = [(t, s) for n, t, s in CASES if n == name][0]
g = case_genome(text)
splits = default_splits()
x_all = splits.train.as_float()
y_all = splits.train.labels.astype(np.int64)
rng = np.random.default_rng(0)
batches = [rng.permutation(len(x_all))[:B] for _ in range(steps)]
net = instantiate(g, shape, seed=0)
oracle = OracleNet.from_network(net)
devs = {p: net.to_device(0, p, max_batch=B) for p in ("fp32",)}
bnet = instantiate(g, shape, seed=0)
devs["bf16"] = bnet.to_device(0, "bf16", max_batch=B)
for step, idx in enumerate(batches):
    x, y = x_all[idx], y_all[idx]
    lo = oracle.train_batch(x, y, g.learn.lr, g.learn.momentum)
    ls = {p: d.train_batch(x, y, g.learn.lr, g.learn.momentum) for p, d in devs.items()}
    errs = []
    for p, d in devs.items():
        for pi, (w, b) in enumerate(net.weights):
            nw, nb, vw, vb = d.get_params(pi, w.shape, b.shape)
            errs.append(f"{p}:W{pi}={rel(nw, oracle.params[pi][0]):.1e}/V{pi}={rel(vw, oracle.vel[pi][0]):.1e}")
    print(f"step {step:3d} oracle {lo:10.4g} fp32 {ls['fp32']:10.4g} bf16 {ls['bf16']:10.4g}  " + " ".join(errs),
          flush=True)
