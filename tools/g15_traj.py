"""Loss trajectory of C2 genome #15 in fp32 and bf16 (first 40 steps), next to the
reference's own fp32 losses (tests/golden/candidate.json c2_g15_full)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1909_12291_b200 import TrainBudget  # noqa: E402
from paper_1909_12291_b200.candidate import train_short  # noqa: E402
from paper_1909_12291_b200.faults import EvalFailure  # noqa: E402
from paper_1909_12291_b200.patches import default_splits  # noqa: E402

splits = default_splits()
g = bench.population(16)[15]
gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "candidate.json")))
ref = gold["c2_g15_full"]["losses"]
np.set_printoptions(linewidth=200, precision=4)
for prec in ("fp32", "bf16"):
    try:
        net, _ = train_short(g, splits.train, TrainBudget(epochs=1, max_batches_per_epoch=40), seed=0, precision=prec)
        losses = net.last_losses
        net.release()
    except EvalFailure as e:
        losses = e.losses
    print(prec, np.asarray(losses[:40]))
print("ref ", np.asarray(ref[:40]))
