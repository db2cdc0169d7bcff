"""C1 (BASELINE.json configs[0]): the FIXED genome, B=64, 2 epochs x 62 steps
on the 4,000 synthetic train patches; train img/s from the device-timed
ce_train loop (CUDA events around the graph replays), with nvidia-smi clocks,
against the SURVEY §8(d) roofline of 55.6 us per step. Also K replicas of the
same candidate packed on K slots (streams) of one GPU: aggregate img/s.

    python tools/c1_bench.py [--reps 5] [--replicas 1,4,8] [--precision bf16]
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import ClockSampler  # noqa: E402
from paper_1909_12291_b200 import ObjectiveConfig, TrainBudget, parse_genome  # noqa: E402
from paper_1909_12291_b200.candidate import evaluate, train_short  # noqa: E402
from paper_1909_12291_b200.genes import FIXED  # noqa: E402
from paper_1909_12291_b200.patches import default_splits  # noqa: E402

ROOFLINE_US = 55.6  # 48.96 GFLOP + 298.7 MB per step


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--replicas", default="1,4,8")
    ap.add_argument("--precision", default="bf16")
    a = ap.parse_args()
    splits = default_splits()
    g = parse_genome(FIXED)
    budget = TrainBudget(epochs=2)
    steps = 2 * (len(splits.train) // g.learn.batch_size)
    for _ in range(2):  # warm-up: library, pools, graphs
        net, _ = train_short(g, splits.train, budget, seed=0, precision=a.precision)
        net.release()
    clocks = ClockSampler(0)
    clocks.start()
    secs = []
    for _ in range(a.reps):
        net, s = train_short(g, splits.train, budget, seed=0, precision=a.precision)
        net.release()
        secs.append(s)
    s = statistics.median(secs)
    out = {"config": "C1 FIXED B=64 2 epochs (124 steps) on 4000 synthetic 100x100x3 patches", "precision": a.precision,
           "train_s": s, "train_img_per_s": steps * g.learn.batch_size / s, "us_per_step": 1e6 * s / steps,
           "roofline_us_per_step": ROOFLINE_US, "roofline_frac": ROOFLINE_US / (1e6 * s / steps),
           "reps": secs}
    # whole evaluate() of the candidate (train + 400 val + device-timed latency), wall clock
    t0 = time.perf_counter()
    rec = evaluate(g, splits, budget, ObjectiveConfig("measured_latency", -0.2, 1e-5, 1e-2), seed=0,
                   precision=a.precision)
    out["evaluate_wall_s"] = time.perf_counter() - t0
    out["candidates_per_hour_one_slot"] = 3600.0 / out["evaluate_wall_s"]
    out["record"] = {"ok": rec.ok, "val_f1": rec.val_f1, "val_auc": rec.val_auc}
    for k in [int(v) for v in a.replicas.split(",")]:
        res = [None] * k

        def run(i):
            res[i] = train_short(g, splits.train, budget, seed=0, precision=a.precision)

        threads = [threading.Thread(target=run, args=(i,)) for i in range(k)]
        t0 = time.perf_counter()
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        wall = time.perf_counter() - t0
        for net, _ in res:
            net.release()
        out[f"replicas_{k}"] = {"wall_s": wall, "train_img_per_s": k * steps * g.learn.batch_size / wall}
    out["clocks"] = clocks.stop()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
