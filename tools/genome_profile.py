"""Per-class kernel profile of one genome given as text (library CUDA events,
steps un-graphed): python tools/genome_profile.py "<genome text>" [precision]"""
import sys
sys.path.insert(0, ".")
from paper_1909_12291_b200 import ObjectiveConfig, TrainBudget, evaluate, parse_genome  # noqa: E402
from paper_1909_12291_b200.patches import default_splits  # noqa: E402

g = parse_genome(sys.argv[1])
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
splits = default_splits()
obj = ObjectiveConfig("measured_latency", -0.2, 1e-5, 1e-2)
r = evaluate(g, splits, TrainBudget(), obj, seed=0, precision=prec)
print("plain", r.ok, r.failure_reason, round(r.train_time_s, 4), r.extras.get("precision"), flush=True)
r = evaluate(g, splits, TrainBudget(), obj, seed=0, precision=prec, profile=True)
print("profiled", r.ok, round(r.train_time_s, 4), flush=True)
print(r.extras.get("kernel_profile"), flush=True)
