"""A few fp32 training steps of one C2 genome (ncu target)."""
import sys
sys.path.insert(0, ".")
from paper_1909_12291_b200 import EvolutionSettings, Master, ObjectiveConfig, SearchSpace, TrainBudget  # noqa
from paper_1909_12291_b200.candidate import train_short
from paper_1909_12291_b200.patches import default_splits
splits = default_splits()
m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0), EvolutionSettings(capacity=16, max_evaluations=16), seed=0)
pop = [m.issue("w") for _ in range(16)]
net, t = train_short(pop[int(sys.argv[1])], splits.train, TrainBudget(epochs=1, max_batches_per_epoch=4), 0,
                     precision=sys.argv[2] if len(sys.argv) > 2 else "fp32")
print("train", t)
