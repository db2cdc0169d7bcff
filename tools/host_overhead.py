"""Fixed per-candidate cost of a C2 population pass: the same evaluate_population
as bench.py but with training cut to `steps` batches per epoch, so what is left
is instantiate + net creation + device init + graph capture + predict + latency
(+ host work) per candidate.
    python tools/host_overhead.py [steps] [slots]
"""
import sys
import time

sys.path.insert(0, ".")
from paper_1909_12291_b200 import EvolutionSettings, Master, ObjectiveConfig, SearchSpace, TrainBudget  # noqa
from paper_1909_12291_b200.patches import default_splits  # noqa
from paper_1909_12291_b200.population import evaluate_population  # noqa

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
slots = int(sys.argv[2]) if len(sys.argv) > 2 else 4
splits = default_splits()
m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0), EvolutionSettings(capacity=16, max_evaluations=16), seed=0)
pop = [m.issue("w") for _ in range(16)]
obj = ObjectiveConfig("measured_latency", -0.2, 1e-5, 1e-2)
budget = TrainBudget(max_batches_per_epoch=steps)
for rep in range(4):
    t0 = time.perf_counter()
    recs, rep_ = evaluate_population(pop, splits, budget, obj, seed=0, slots_per_gpu=slots)
    dt = time.perf_counter() - t0
    print(f"pass {rep}: {dt * 1000:.1f} ms for 16 candidates ({dt / 16 * 1000:.1f} ms each, {steps} steps/epoch)",
          flush=True)
