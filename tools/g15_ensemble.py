"""C2 genome #15 (2d5ebb4eae1bf684: conv 256 k5 s3 -> dense 523 at lr 0.017) over its full
budget under summation-order variants that do not change the math (every batch's
samples shuffled by default_rng(s); s = 0: reference order), in fp32 and bf16: how
often does the trajectory leave the finite range? The fp32 reference itself stays
finite in reference order (tests/golden/candidate.json c2_g15_full).

    python tools/g15_ensemble.py [--variants 16] [--out gpurun_out/g15_ensemble.json]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_1909_12291_b200.candidate import DATASETS, epoch_permutations  # noqa: E402
from paper_1909_12291_b200.network import instantiate  # noqa: E402
from paper_1909_12291_b200.patches import default_splits  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", type=int, default=16)
    ap.add_argument("--genome", type=int, default=15)
    ap.add_argument("--out", default="gpurun_out/g15_ensemble.json")
    a = ap.parse_args()
    splits = default_splits()
    g = bench.population(16)[a.genome]
    n, bs = len(splits.train), min(g.learn.batch_size, len(splits.train))
    ds = DATASETS.get(splits.train, 0)
    out = {"genome": g.id}
    for prec in ("fp32", "bf16"):
        rows = []
        for s in range(a.variants):
            perms = epoch_permutations(0, n, 2)
            if s:
                rng = np.random.default_rng(s)
                for e in range(2):
                    for start in range(0, n - bs + 1, bs):
                        perms[e, start:start + bs] = perms[e, start:start + bs][rng.permutation(bs)]
            net = instantiate(g, splits.train.input_shape, seed=0)
            dev = net.to_device(0, prec, max_batch=128)
            losses, _ = dev.train(ds, perms, n // bs, bs, g.learn.lr, g.learn.momentum)
            net.release()
            bad = np.flatnonzero(~np.isfinite(losses))
            rows.append({"s": s, "first_nonfinite": int(bad[0]) if len(bad) else None,
                         "max_loss": float(np.nanmax(np.where(np.isfinite(losses), losses, np.nan)))})
        out[prec] = rows
        print(prec, "diverged", sum(r["first_nonfinite"] is not None for r in rows), "of", len(rows),
              [r["first_nonfinite"] for r in rows], flush=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
