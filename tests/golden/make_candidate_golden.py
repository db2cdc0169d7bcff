"""Candidate-level golden fixtures from the REFERENCE (convevo), run in the
build container. They pin the product path (ce_train -> ce_predict ->
metrics -> EvalRecord) at BASELINE scale, SURVEY §8(c) tiers T3/T4.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_candidate_golden.py [c1] [c2] [g15]

  c1   FIXED genome on the C1 data, full budget (2 epochs x 62 steps, B=64),
       evaluator.py:145-186 composed exactly as evaluate() does (:223-255):
       every per-step loss (train_batch wrapped, nothing else changed), the
       400 val scores / preds, confusion counts, F1, AUC, FLOPs, params and
       the flop_proxy fitness. ~7 min of CPU.
  c2   the 16 C2 genomes (Master seed 0 bootstrap) through convevo's own
       evaluate() at TrainBudget(epochs=1, max_batches_per_epoch=2), plus the
       val scores / preds of the same training (train_short is deterministic).
  g15  C2 genome #15 (2d5ebb4eae1bf684, 137 M-param head, lr 0.017) over its
       full budget: does the fp32 reference itself diverge? Every loss until
       the first non-finite one (evaluator.py:166-170).

Output: tests/golden/candidate.json (the conv weights are stored as SHA-256
digests only; the parity tests compare against the live oracle, which is
itself pinned by these losses).
"""

import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

REF = os.environ.get("CONVEVO_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from convevo import data as rdata  # noqa: E402
from convevo import evaluator as rev  # noqa: E402
from convevo import evolution as revo  # noqa: E402
from convevo import fitness as rfit  # noqa: E402
from convevo import genome as rgen  # noqa: E402
from convevo import metrics as rmet  # noqa: E402
from convevo import nn as rnn  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "candidate.json")

FIXED = ("id=fixed0000000000 parents= lr=0.0003 momentum=0.9 batch_size=64 "
         "f0=conv:oc=32,k=4,s=2,relu=1 f1=conv:oc=64,k=4,s=1,relu=1 f2=pool:size=2,s=2 "
         "f3=conv:oc=128,k=4,s=1,relu=1 h0=dense:units=64")
FLOP_OBJ = ("flop_proxy", -0.2, 1e8, 1e9)


def splits():
    d = rdata.generate_synthetic(*rdata.default_counts(4800), h=100, w=100, seed=0)
    return rdata.stratified_split(d, (5 / 6, 1 / 12, 1 / 12), seed=0)


class LossLog:
    """Wraps evaluator.train_batch (evaluator.py:166) to record each loss."""

    def __init__(self):
        self.losses = []
        self._orig = rev.train_batch

    def __enter__(self):
        def wrapped(*a, **k):
            loss = self._orig(*a, **k)
            self.losses.append(float(loss))
            return loss
        rev.train_batch = wrapped
        return self

    def __exit__(self, *exc):
        rev.train_batch = self._orig


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def scored(genome, sp, budget, seed=0):
    """train_short + predict_scores + the evaluate() arithmetic (evaluator.py:223-251)."""
    t0 = time.time()
    with LossLog() as log:
        try:
            net, _ = rev.train_short(genome, sp.train, budget, seed)
        except rev.EvalFailure as e:
            return {"ok": False, "failure_reason": str(e), "losses": log.losses, "cpu_s": time.time() - t0}
    scores, preds = rev.predict_scores(net, sp.val)
    conf = rmet.confusion_counts(preds, sp.val.labels)
    f1 = rmet.f1_score(conf["tp"], conf["fp"], conf["fn"])
    auc = rmet.auc_roc(scores, sp.val.labels)
    shape = sp.train.input_shape
    flops = rev.count_flops_inference(net, shape)
    params = rev.count_params(net)
    obj = rfit.ObjectiveConfig(*FLOP_OBJ)
    fv = rfit.score(f1, rev.raw_objective(obj.kind, flops, params, None), obj)
    weights = {f"{li}_{nm}": [list(a.shape), sha(a), float(np.linalg.norm(a.astype(np.float64)))]
               for li, nm, a in net.parameters()}
    return {"ok": True, "failure_reason": "", "losses": log.losses, "scores": scores.tolist(),
            "preds": preds.tolist(), "confusion": {k: int(v) for k, v in conf.items()}, "val_f1": f1,
            "val_auc": auc, "flops_inference": flops, "params": params, "objective_m": fv.m, "fitness": fv.f,
            "weights": weights, "cpu_s": time.time() - t0}


def c2_genomes():
    m = revo.Master(rgen.SearchSpace(), rfit.ObjectiveConfig(*FLOP_OBJ),
                    revo.EvolutionSettings(capacity=16, max_evaluations=16), seed=0)
    return [m.issue("golden") for _ in range(16)]


def main(which):
    out = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            out = json.load(fh)
    out["meta"] = {"numpy": np.__version__, "python": platform.python_version(),
                   "blas": "scipy-openblas 0.3.30 (numpy wheel)", "reference": REF,
                   "cpu": platform.processor() or platform.machine(), "threads": os.cpu_count()}
    sp = splits()
    if "c1" in which:
        out["c1_fixed_full"] = scored(rgen.parse_genome(FIXED), sp, rev.TrainBudget(epochs=2), seed=0)
        out["c1_fixed_full"]["budget"] = [2, None]
        print("c1", out["c1_fixed_full"]["val_f1"], out["c1_fixed_full"]["val_auc"], flush=True)
    if "c2" in which:
        budget = rev.TrainBudget(epochs=1, max_batches_per_epoch=2)
        rows = []
        for g in c2_genomes():
            rec = rev.evaluate(g, sp, budget, rfit.ObjectiveConfig(*FLOP_OBJ), seed=0)
            row = scored(g, sp, budget, seed=0)
            row["genome"] = rgen.format_genome(g)
            row["record"] = rec.to_json_dict()
            row.pop("weights", None)
            rows.append(row)
            print("c2", g.id, rec.ok, rec.val_f1, rec.val_auc, f"{row['cpu_s']:.1f}s", flush=True)
        out["c2_2steps"] = {"budget": [1, 2], "rows": rows}
    if "g15" in which:
        g = [x for x in c2_genomes() if x.id == "2d5ebb4eae1bf684"][0]
        row = scored(g, sp, rev.TrainBudget(epochs=2), seed=0)
        row.pop("scores", None)
        row.pop("preds", None)
        row["genome"] = rgen.format_genome(g)
        out["c2_g15_full"] = row
        print("g15", row["ok"], row["failure_reason"], len(row["losses"]), flush=True)
    with open(OUT + ".tmp", "w") as fh:
        json.dump(out, fh)
    os.replace(OUT + ".tmp", OUT)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or {"c1", "c2", "g15"})
