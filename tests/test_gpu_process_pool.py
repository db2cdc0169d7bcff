"""Process-per-GPU pool (socket transport, scheduler.ProcessGpuPool): a
worker process per GPU evaluates candidates and the records equal the
in-process evaluate() of the same genomes (transport equivalence)."""

import numpy as np
import pytest

from paper_1909_12291_b200.candidate import TrainBudget, evaluate
from paper_1909_12291_b200.genes import SearchSpace, random_genome
from paper_1909_12291_b200.patches import default_splits
from paper_1909_12291_b200.population import ListMaster
from paper_1909_12291_b200.scheduler import ProcessGpuPool
from paper_1909_12291_b200.scoring import ObjectiveConfig

pytestmark = pytest.mark.gpu

CONFIG = {"budget": {"epochs": 1, "max_batches_per_epoch": 3},
          "objective": {"kind": "flop_proxy", "alpha": -0.2, "lo": 1.0, "hi": 2.0}, "seed": 0, "precision": "bf16"}


def test_process_pool_matches_in_process():
    rng = np.random.default_rng(7)
    gs = [random_genome(rng, SearchSpace()) for _ in range(4)]
    master = ListMaster(gs)
    report = ProcessGpuPool(master, CONFIG, devices=(0,), slots_per_gpu=2).run()
    assert sorted(master.records) == sorted(g.id for g in gs)
    assert sum(st.evaluations_done for st in report.stats.values()) == 4
    splits = default_splits()
    for g in gs:
        want = evaluate(g, splits, TrainBudget(**CONFIG["budget"]), ObjectiveConfig(**CONFIG["objective"]), 0)
        got = master.records[g.id]
        assert got.ok == want.ok
        assert got.flops_inference == want.flops_inference and got.params == want.params
        if want.ok:
            assert got.val_f1 == want.val_f1 and got.val_auc == want.val_auc
        assert got.worker_id.startswith("g0s")
