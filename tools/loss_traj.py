"""Print the per-step loss trajectory of one C2 genome on the GPU (both precisions)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1909_12291_b200 import (EvolutionSettings, Master, ObjectiveConfig, SearchSpace, TrainBudget)  # noqa
from paper_1909_12291_b200.candidate import train_short
from paper_1909_12291_b200.faults import EvalFailure
from paper_1909_12291_b200.patches import default_splits
splits = default_splits()
m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0), EvolutionSettings(capacity=16, max_evaluations=16), seed=0)
pop = [m.issue("w") for _ in range(16)]
idx = int(sys.argv[1])
for prec in sys.argv[2:] or ["bf16", "fp32"]:
    try:
        net, t = train_short(pop[idx], splits.train, TrainBudget(), 0, precision=prec)
        ls = net.last_losses
    except EvalFailure as e:
        ls = e.losses
        print(prec, "failed:", e)
    print(prec, " ".join(f"{i}:{ls[i]:.4g}" for i in range(0, len(ls), 20)), flush=True)
