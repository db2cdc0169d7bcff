"""How sensitive is the REFERENCE's own C1 outcome to float summation order?

Runs the numpy oracle (oracle/cnn_ref.py, bit-identical to convevo on C1:
every per-step loss equal, tools/c1_trajectory.py --oracle) for the FIXED
genome's full budget in variants that change only the order of floating-point
additions, never the math:
  ref        the reference order (= tests/golden/candidate.json c1_fixed_full)
  rev_batch  every batch's samples in reverse order (the batch mean and the
             gradient sums over the batch add in the opposite order)
  rev_taps   conv taps accumulated in reverse order (nn.py:88-91, 108-113)
  fp64       the same arithmetic in float64
  perm<s>    every batch's samples in an order shuffled by default_rng(s)
and reports each one's val confusion counts and AUC next to the golden. The
spread is the reference's own uncertainty at full budget (SURVEY §0 item 10:
the trajectory is chaotic), i.e. the smallest tolerance a T4 comparison of
any other implementation can be held to.

    OPENBLAS_NUM_THREADS=1 python tools/c1_sensitivity.py [--out profiles/r02_c1_sensitivity.json]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(variant):
    from oracle import cnn_ref as O
    from paper_1909_12291_b200 import parse_genome
    from paper_1909_12291_b200.genes import FIXED
    from paper_1909_12291_b200.network import instantiate
    from paper_1909_12291_b200.patches import default_splits
    from paper_1909_12291_b200.scoring import auc_roc, confusion_counts
    if variant == "rev_taps":
        def conv_forward(x, w, b, stride):
            n, c, h, wd = x.shape
            co, ci, k, _ = w.shape
            oh, ow = (h - k) // stride + 1, (wd - k) // stride + 1
            acc = np.zeros((n, oh, ow, co), dtype=x.dtype)
            for i in reversed(range(k)):
                for j in reversed(range(k)):
                    tap = x[:, :, i:i + stride * oh:stride, j:j + stride * ow:stride]
                    acc += np.tensordot(tap, w[:, :, i, j], axes=([1], [1]))
            return np.ascontiguousarray(acc.transpose(0, 3, 1, 2) + b[None, :, None, None])
        O.conv_forward = conv_forward
    dt = np.float64 if variant == "fp64" else np.float32
    splits = default_splits()
    genome = parse_genome(FIXED)
    net = O.OracleNet.from_network(instantiate(genome, splits.train.input_shape, seed=0), dtype=dt)
    x = splits.train.pixels.astype(dt) / dt(255.0)
    y = splits.train.labels.astype(np.int64)
    n, bs = len(splits.train), genome.learn.batch_size
    rng = np.random.default_rng([0, 0xDA7A])
    shuffle = np.random.default_rng(int(variant[4:])) if variant.startswith("perm") else None
    losses = []
    for epoch in range(2):
        perm = rng.permutation(n)
        for start in range(0, n - bs + 1, bs):
            idx = perm[start:start + bs]
            if variant == "rev_batch":
                idx = idx[::-1]
            elif shuffle is not None:
                idx = idx[shuffle.permutation(len(idx))]
            losses.append(net.train_batch(x[idx], y[idx], genome.learn.lr, genome.learn.momentum))
    scores, preds = O.predict_scores(net, splits.val, dtype=dt)
    conf = confusion_counts(preds, splits.val.labels)
    return variant, {"confusion": {k: int(v) for k, v in conf.items()}, "auc": float(auc_roc(scores, splits.val.labels)),
                     "losses": [float(v) for v in losses], "scores": scores.tolist(), "preds": preds.tolist()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r02_c1_sensitivity.json")
    ap.add_argument("--variants", default="ref,rev_batch,rev_taps,fp64")
    a = ap.parse_args()
    variants = a.variants.split(",")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    with mp.get_context("spawn").Pool(len(variants)) as pool:
        res = dict(pool.map(run, variants))
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "candidate.json")))["c1_fixed_full"]
    out = {"golden": {"confusion": gold["confusion"], "auc": gold["val_auc"]}, "variants": {}}
    for v, r in res.items():
        d = np.abs(np.asarray(r["losses"]) - gold["losses"]) / np.abs(gold["losses"])
        out["variants"][v] = {**r, "loss_rel_first_above_1e-4": int(np.argmax(d > 1e-4)) if (d > 1e-4).any() else None,
                              "loss_rel_last": float(d[-1])}
        print(v, r["confusion"], round(r["auc"], 4), out["variants"][v]["loss_rel_first_above_1e-4"], flush=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
