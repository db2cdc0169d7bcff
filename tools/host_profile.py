"""cProfile of a short-budget C2 population pass (1 slot): where host time goes
per candidate outside the kernels.  python tools/host_profile.py [steps]"""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
from paper_1909_12291_b200 import EvolutionSettings, Master, ObjectiveConfig, SearchSpace, TrainBudget  # noqa
from paper_1909_12291_b200.patches import default_splits  # noqa
from paper_1909_12291_b200.population import evaluate_population  # noqa

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
splits = default_splits()
m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0), EvolutionSettings(capacity=16, max_evaluations=16), seed=0)
pop = [m.issue("w") for _ in range(16)]
obj = ObjectiveConfig("measured_latency", -0.2, 1e-5, 1e-2)
budget = TrainBudget(max_batches_per_epoch=steps)
evaluate_population(pop, splits, budget, obj, seed=0, slots_per_gpu=1)  # warm
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    evaluate_population(pop, splits, budget, obj, seed=0, slots_per_gpu=1)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
