"""Per-candidate device train time / wall time for the C2 population (+ FIXED)."""
import sys
import time
sys.path.insert(0, ".")
from paper_1909_12291_b200 import (EvolutionSettings, Master, ObjectiveConfig, SearchSpace, TrainBudget, evaluate,  # noqa
                                   parse_genome)
from paper_1909_12291_b200.genes import FIXED, format_genome
from paper_1909_12291_b200.patches import default_splits
splits = default_splits()
m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0), EvolutionSettings(capacity=16, max_evaluations=16), seed=0)
pop = [m.issue("w") for _ in range(16)] + [parse_genome(FIXED)]
obj = ObjectiveConfig("measured_latency", -0.2, 1e-5, 1e-2)
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
evaluate(pop[-1], splits, TrainBudget(), obj, seed=0, precision=prec)  # warm-up (module load, pools)
tot = 0.0
for i, g in enumerate(pop):
    t0 = time.perf_counter()
    r = evaluate(g, splits, TrainBudget(), obj, seed=0, precision=prec)
    wall = time.perf_counter() - t0
    tot += wall
    print(f"{i:2d} {g.id} ok={r.ok} prec={r.extras.get('precision')} train={r.train_time_s:.4f}s wall={wall:.3f}s "
          f"f1={r.val_f1:.3f} auc={r.val_auc:.3f} lat={r.latency.median_s_per_batch*1e3 if r.latency else 0:.3f}ms "
          f"{r.extras.get('bf16_failure', '')}", flush=True)
print(f"total wall {tot:.2f}s")
