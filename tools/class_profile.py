"""Per-genome kernel-class profile of the C2 population (library per-class CUDA
events, steps run un-graphed): ms and launches per class per genome.
    python tools/class_profile.py [precision] [max_batches_per_epoch]
(a small max_batches_per_epoch keeps ncu launch-list passes short)
"""
import sys

sys.path.insert(0, ".")
from paper_1909_12291_b200 import (EvolutionSettings, Master, ObjectiveConfig, SearchSpace, TrainBudget,  # noqa
                                   evaluate)
from paper_1909_12291_b200.patches import default_splits

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
mbe = int(sys.argv[2]) if len(sys.argv) > 2 else None
splits = default_splits()
m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0), EvolutionSettings(capacity=16, max_evaluations=16), seed=0)
pop = [m.issue("w") for _ in range(16)]
obj = ObjectiveConfig("measured_latency", -0.2, 1e-5, 1e-2)
tot = {}
for i, g in enumerate(pop):
    r = evaluate(g, splits, TrainBudget(max_batches_per_epoch=mbe), obj, seed=0, precision=prec, profile=True)
    prof = r.extras.get("kernel_profile", {})
    steps = r.extras.get("train_steps", 0)
    parts = []
    for name, (launches, ms, *_) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        if launches:
            parts.append(f"{name}={ms:.1f}ms/{launches}")
            t = tot.setdefault(name, [0.0, 0])
            t[0] += ms
            t[1] += launches
    print(f"{i:2d} steps={steps} train={r.train_time_s:.3f}s " + " ".join(parts), flush=True)
print("TOTAL " + " ".join(f"{k}={v[0]:.1f}ms/{v[1]} ({1000 * v[0] / max(v[1], 1):.1f}us)" for k, v in
                          sorted(tot.items(), key=lambda kv: -kv[1][0])))
