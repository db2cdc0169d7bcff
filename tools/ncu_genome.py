"""One C2 genome (index into the Master-seed-0 bootstrap population) through
evaluate() with a short budget, for ncu captures of its kernels:

    python tools/ncu_genome.py <index> [max_batches] [precision]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_1909_12291_b200 import ObjectiveConfig, TrainBudget, evaluate  # noqa: E402
from paper_1909_12291_b200.patches import default_splits  # noqa: E402

mb = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
if sys.argv[1].isdigit():
    i = int(sys.argv[1])
    g = bench.population(16)[i]
else:  # a canonical genome by name: FIXED, VGG16STYLE, SWEET
    from paper_1909_12291_b200 import genes, parse_genome
    i, g = sys.argv[1], parse_genome(getattr(genes, sys.argv[1]))
r = evaluate(g, default_splits(), TrainBudget(epochs=1, max_batches_per_epoch=mb),
             ObjectiveConfig("flop_proxy", -0.2, 1e8, 1e9), seed=0, precision=prec, confirm_divergence=False)
print(i, g.id, r.ok, r.failure_reason, r.extras.get("precision"), "train_s", r.train_time_s,
      "steps", r.extras.get("train_steps"))
