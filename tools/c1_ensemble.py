"""The C1 candidate (FIXED, B=64, 2 epochs) through ce_train + ce_predict under
summation-order variants that do not change the math: every batch's samples
in an order shuffled by default_rng(s) (s = 0: the reference order), exactly
the perm<s> variants tools/c1_sensitivity.py runs on the numpy oracle. The
distribution of val decisions / AUC over s is compared with the reference's
own distribution under the same perturbations (profiles/r02_c1_sensitivity.json).

    python tools/c1_ensemble.py [--variants 32] [--out gpurun_out/c1_ensemble.json]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1909_12291_b200 import parse_genome  # noqa: E402
from paper_1909_12291_b200.candidate import DATASETS, epoch_permutations  # noqa: E402
from paper_1909_12291_b200.genes import FIXED  # noqa: E402
from paper_1909_12291_b200.network import instantiate  # noqa: E402
from paper_1909_12291_b200.patches import default_splits  # noqa: E402
from paper_1909_12291_b200.scoring import auc_roc, confusion_counts  # noqa: E402


def shuffled_perms(n, bs, s):
    perms = epoch_permutations(0, n, 2)
    if s == 0:
        return perms
    rng = np.random.default_rng(s)
    out = perms.copy()
    for e in range(2):
        for start in range(0, n - bs + 1, bs):
            idx = out[e, start:start + bs]
            out[e, start:start + bs] = idx[rng.permutation(bs)]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", type=int, default=32)
    ap.add_argument("--out", default="gpurun_out/c1_ensemble.json")
    a = ap.parse_args()
    splits = default_splits()
    genome = parse_genome(FIXED)
    n, bs = len(splits.train), genome.learn.batch_size
    ds_tr = DATASETS.get(splits.train, 0)
    ds_val = DATASETS.get(splits.val, 0)
    out = {}
    for prec in ("fp32", "bf16"):
        rows = []
        for s in range(a.variants):
            net = instantiate(genome, splits.train.input_shape, seed=0)
            dev = net.to_device(0, prec, max_batch=128)
            losses, _ = dev.train(ds_tr, shuffled_perms(n, bs, s), n // bs, bs, genome.learn.lr, genome.learn.momentum)
            scores, preds = dev.predict(ds_val, 128)
            conf = confusion_counts(preds, splits.val.labels)
            rows.append({"s": s, "confusion": {k: int(v) for k, v in conf.items()},
                         "auc": float(auc_roc(scores, splits.val.labels)), "finite": bool(np.isfinite(losses).all()),
                         "last_loss": float(losses[-1])})
            net.release()
        out[prec] = rows
        tps = [r["confusion"]["tp"] for r in rows]
        aucs = [r["auc"] for r in rows]
        print(prec, "tp", tps, "auc %.4f..%.4f" % (min(aucs), max(aucs)), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
