"""C1 (FIXED, B=64, 2 epochs) loss trajectory through ce_train vs the reference's
own run (tests/golden/candidate.json c1_fixed_full): per-step relative loss
difference, where it first exceeds 1e-4 / 1e-2 / 1e-1, and the val decisions.
Also (--oracle) the same for the numpy oracle in float64 on this host: the
reference's own sensitivity to summation precision.

    python tools/c1_trajectory.py [--oracle] [--out gpurun_out/c1_traj.json]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1909_12291_b200 import TrainBudget, parse_genome  # noqa: E402
from paper_1909_12291_b200.genes import FIXED  # noqa: E402
from paper_1909_12291_b200.patches import default_splits  # noqa: E402


def summary(losses, gold_losses):
    a, b = np.asarray(losses, np.float64), np.asarray(gold_losses, np.float64)
    n = min(len(a), len(b))
    d = np.abs(a[:n] - b[:n]) / np.maximum(np.abs(b[:n]), 1e-30)
    first = {str(t): int(np.argmax(d > t)) if (d > t).any() else None for t in (1e-6, 1e-4, 1e-2, 1e-1)}
    return {"rel_diff": d.tolist(), "first_step_above": first}


def decisions(scores, preds, gold, labels):
    preds, gp = np.asarray(preds), np.asarray(gold["preds"])
    lab = np.asarray(labels)
    conf = {"tp": int(((preds == 1) & (lab == 1)).sum()), "fp": int(((preds == 1) & (lab == 0)).sum()),
            "fn": int(((preds == 0) & (lab == 1)).sum())}
    return {"confusion": conf, "ref_confusion": gold["confusion"], "flips": int((preds != gp).sum()),
            "scores_rel": float(np.linalg.norm(np.asarray(scores) - gold["scores"]) / np.linalg.norm(gold["scores"]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--out", default="gpurun_out/c1_traj.json")
    a = ap.parse_args()
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "candidate.json")))
    gold = gold["c1_fixed_full"]
    splits = default_splits()
    genome = parse_genome(FIXED)
    out = {}
    if a.oracle:
        from oracle import cnn_ref as O
        from paper_1909_12291_b200.network import instantiate
        for dt in (np.float32, np.float64):
            net = O.OracleNet.from_network(instantiate(genome, splits.train.input_shape, seed=0), dtype=dt)
            losses, _, bad = O.train_short(net, genome, splits.train, 2, 0, dtype=dt)
            scores, preds = O.predict_scores(net, splits.val, dtype=dt)
            out[f"oracle_{np.dtype(dt).name}"] = {**summary(losses, gold["losses"]),
                                                  **decisions(scores, preds, gold, splits.val.labels)}
            print(np.dtype(dt).name, out[f"oracle_{np.dtype(dt).name}"]["first_step_above"],
                  out[f"oracle_{np.dtype(dt).name}"]["confusion"], flush=True)
    else:
        from paper_1909_12291_b200.candidate import predict_scores, train_short
        for prec in ("fp32", "bf16"):
            net, _ = train_short(genome, splits.train, TrainBudget(epochs=2), seed=0, precision=prec)
            scores, preds = predict_scores(net, splits.val)
            out[prec] = {**summary(net.last_losses, gold["losses"]),
                         **decisions(scores, preds, gold, splits.val.labels),
                         "losses": np.asarray(net.last_losses).tolist()}
            net.release()
            print(prec, out[prec]["first_step_above"], out[prec]["confusion"], out[prec]["flips"], flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
