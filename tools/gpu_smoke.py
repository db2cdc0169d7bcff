"""Ad-hoc GPU check: evaluate FIXED (bf16 + fp32) and a few random genomes."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1909_12291_b200 import (EvolutionSettings, Master, ObjectiveConfig, SearchSpace, TrainBudget,  # noqa
                                   evaluate, parse_genome)
from paper_1909_12291_b200.genes import FIXED
from paper_1909_12291_b200.patches import default_splits

t = time.time()
splits = default_splits()
print("data", time.time() - t, flush=True)
obj = ObjectiveConfig("measured_latency", -0.2, 1e-4, 1e-1)
g = parse_genome(FIXED)
for prec in ("bf16", "fp32", "bf16"):
    t = time.time()
    r = evaluate(g, splits, TrainBudget(epochs=2), obj, seed=0, precision=prec)
    print(prec, "wall", round(time.time() - t, 3), r.to_json_dict(), flush=True)
m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1e6, 1e11), EvolutionSettings(capacity=16, max_evaluations=16), seed=0)
for i in range(16):
    gg = m.issue("w0")
    t = time.time()
    r = evaluate(gg, splits, TrainBudget(epochs=2), obj, seed=0, precision="bf16")
    print(i, gg.id, "wall", round(time.time() - t, 3), "train", round(r.train_time_s, 4), r.ok, r.failure_reason, round(r.val_f1, 3), round(r.val_auc, 3), flush=True)
