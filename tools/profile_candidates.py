"""Evaluate a few C2 genomes with a short budget (for ncu launch lists)."""
import sys

sys.path.insert(0, ".")
from paper_1909_12291_b200 import (EvolutionSettings, Master, ObjectiveConfig, SearchSpace, TrainBudget,  # noqa
                                   evaluate, parse_genome)
from paper_1909_12291_b200.genes import FIXED
from paper_1909_12291_b200.patches import default_splits

idx = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8, 9]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
splits = default_splits()
m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0), EvolutionSettings(capacity=16, max_evaluations=16), seed=0)
pop = [m.issue("w") for _ in range(16)]
obj = ObjectiveConfig("measured_latency", -0.2, 1e-5, 1e-2)
for i in idx:
    g = parse_genome(FIXED) if i < 0 else pop[i]
    r = evaluate(g, splits, TrainBudget(epochs=1, max_batches_per_epoch=steps), obj, seed=0)
    print(i, g.id, r.ok, r.failure_reason, round(r.train_time_s, 5), flush=True)
