"""Evaluate one C2 genome (index) at a given precision; print the record."""
import sys
sys.path.insert(0, ".")
from paper_1909_12291_b200 import (EvolutionSettings, Master, ObjectiveConfig, SearchSpace, TrainBudget, evaluate)  # noqa
from paper_1909_12291_b200.patches import default_splits
splits = default_splits()
m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0), EvolutionSettings(capacity=16, max_evaluations=16), seed=0)
pop = [m.issue("w") for _ in range(16)]
obj = ObjectiveConfig("measured_latency", -0.2, 1e-5, 1e-2)
for prec in sys.argv[2:] or ["bf16"]:
    for i in [int(a) for a in sys.argv[1].split(",")]:
        r = evaluate(pop[i], splits, TrainBudget(), obj, seed=0, precision=prec)
        print(prec, i, pop[i].id, r.ok, r.failure_reason, round(r.train_time_s, 4), round(r.val_f1, 3), round(r.val_auc, 3), flush=True)
