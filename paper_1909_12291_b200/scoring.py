"""Scalar scoring of a candidate: classification metrics and the scalarised
multi-objective fitness f = v + alpha * m.

Restates convevo/metrics.py:15-81 (confusion counts, positive-class F1,
mid-rank AUC, slide time) and convevo/fitness.py:12-82 (ObjectiveConfig,
normalisation, score, the total order used for selection and eviction).
All results are bit-identical to the reference for identical inputs: the
arithmetic is the same sequence of Python float operations.
"""

import json
from dataclasses import dataclass, field

import numpy as np

OBJECTIVE_KINDS = ("none", "flop_proxy", "param_count", "measured_latency")
FAILED_FITNESS = float("-inf")


# --------------------------------------------------------------------------
# metrics (metrics.py:15-81)

def confusion_counts(predictions, labels):
    p = np.asarray(predictions)
    y = np.asarray(labels)
    if p.shape != y.shape:
        raise ValueError(f"predictions shape {p.shape} != labels shape {y.shape}")
    pos_p, pos_y = p == 1, y == 1
    neg_p, neg_y = p == 0, y == 0
    return {"tp": int(np.count_nonzero(pos_p & pos_y)),
            "fp": int(np.count_nonzero(pos_p & neg_y)),
            "fn": int(np.count_nonzero(neg_p & pos_y)),
            "tn": int(np.count_nonzero(neg_p & neg_y))}


def f1_score(tp, fp, fn):
    """Positive-class F1; 0.0 when there is no true positive."""
    if tp == 0:
        return 0.0
    precision = tp / (tp + fp)
    recall = tp / (tp + fn)
    return 2 * precision * recall / (precision + recall)


def f1_degenerate(tp, fp, fn):
    return tp == 0 and fp == 0 and fn == 0


def _average_ranks(values):
    """1-based ranks with ties replaced by their mean (stable mergesort)."""
    order = np.argsort(values, kind="mergesort")
    sv = values[order]
    ranks = np.empty(len(values), dtype=np.float64)
    n = len(values)
    start = 0
    while start < n:
        stop = start
        while stop + 1 < n and sv[stop + 1] == sv[start]:
            stop += 1
        ranks[order[start:stop + 1]] = (start + stop) / 2.0 + 1.0
        start = stop + 1
    return ranks


def auc_roc(scores, labels):
    """P(random positive outscores random negative), ties count half."""
    s = np.asarray(scores, dtype=np.float64)
    y = np.asarray(labels)
    n_pos = int(np.sum(y == 1))
    n_neg = int(np.sum(y == 0))
    if n_pos == 0 or n_neg == 0:
        raise ValueError(
            f"AUC needs both classes, got {n_pos} positives / {n_neg} negatives")
    u = _average_ranks(s)[y == 1].sum() - n_pos * (n_pos + 1) / 2.0
    return float(u / (n_pos * n_neg))


def slide_seconds(prediction_rate, patches=200_000):
    if prediction_rate <= 0:
        raise ValueError("prediction rate must be positive")
    return patches / prediction_rate


@dataclass
class MetricsReport:
    f1: float
    auc: float
    confusion: dict
    prediction_rate_patches_per_s: float
    model_id: str = ""
    dataset_id: str = ""
    f1_degenerate: bool = False
    extras: dict = field(default_factory=dict)

    def to_json(self):
        payload = dict(f1=self.f1, auc=self.auc, confusion=self.confusion,
                       prediction_rate_patches_per_s=self.prediction_rate_patches_per_s,
                       model_id=self.model_id, dataset_id=self.dataset_id,
                       f1_degenerate=self.f1_degenerate)
        payload.update(self.extras)
        return json.dumps(payload, sort_keys=True)

    def to_text(self):
        c = self.confusion
        return "\n".join([
            f"model:            {self.model_id}",
            f"dataset:          {self.dataset_id}",
            f"f1 (positive):    {self.f1:.4f}" + ("  [degenerate]" if self.f1_degenerate else ""),
            f"auc:              {self.auc:.4f}",
            f"confusion:        tp={c['tp']} fp={c['fp']} fn={c['fn']} tn={c['tn']}",
            f"prediction rate:  {self.prediction_rate_patches_per_s:.1f} patches/s",
            f"est. slide time:  {slide_seconds(self.prediction_rate_patches_per_s):.1f} s (200000 patches)",
        ])


# --------------------------------------------------------------------------
# fitness (fitness.py:12-82)

@dataclass
class ObjectiveConfig:
    kind: str = "none"
    alpha: float = 0.0
    lo: float | None = None
    hi: float | None = None
    clamp: bool = True

    def __post_init__(self):
        if self.kind not in OBJECTIVE_KINDS:
            raise ValueError(f"objective kind {self.kind!r} not in {OBJECTIVE_KINDS}")
        bounded = self.lo is not None and self.hi is not None
        if self.kind != "none" and bounded and not self.lo < self.hi:
            raise ValueError(f"objective bounds need lo < hi, got lo={self.lo} hi={self.hi}")

    @property
    def calibrated(self):
        return self.kind == "none" or (self.lo is not None and self.hi is not None)


@dataclass
class FitnessValue:
    v: float
    m: float
    f: float


def normalize_objective(raw, lo, hi, clamp=True):
    if not lo < hi:
        raise ValueError(f"normalization bounds need lo < hi, got {lo}, {hi}")
    m = (raw - lo) / (hi - lo)
    return min(max(m, 0.0), 1.0) if clamp else m


def fitness(v, m, alpha):
    return v + alpha * m


def score(v, raw, objective):
    if objective.kind == "none":
        return FitnessValue(v=v, m=0.0, f=v)
    if not objective.calibrated:
        raise ValueError("objective bounds not calibrated")
    m = normalize_objective(raw, objective.lo, objective.hi, objective.clamp)
    return FitnessValue(v=v, m=m, f=fitness(v, m, objective.alpha))


def sort_key(record):
    """Best first: higher fitness, then fewer inference FLOPs, then id."""
    return (-record.fitness, record.flops_inference, record.genome_id)


def compare(a, b):
    ka, kb = sort_key(a), sort_key(b)
    return -1 if ka < kb else (1 if ka > kb else 0)
