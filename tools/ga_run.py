"""C3: the steady-state multi-objective GA, population 64 x 5
generations (= 320 evaluations), with the population evaluated across the GPUs
of one box by the process-per-GPU pull scheduler (scheduler.ProcessGpuPool:
one gpu_worker process per GPU, `--slots` socket workers each).

    python tools/ga_run.py [--gpus N] [--slots K] [--evals 320] [--out log.jsonl]

Prints one JSON line: candidates/h from the first work request to the last
record (and including worker-process start-up), best genome and fitness,
failures, per-worker busy fractions. The master is the
reference's (ga.Master: evolution.py:99-186); selection is bit-exact given the
arrival order of the records, which pull scheduling makes run-dependent, so
the best genome can differ between runs (as in the reference's WorkerPool).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1909_12291_b200 import EvolutionSettings, Master, ObjectiveConfig, SearchSpace  # noqa: E402
from paper_1909_12291_b200.ga import JsonlLog  # noqa: E402
from paper_1909_12291_b200.genes import format_genome  # noqa: E402
from paper_1909_12291_b200.scheduler import ProcessGpuPool  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--slots", type=int, default=4)
    ap.add_argument("--capacity", type=int, default=64)
    ap.add_argument("--evals", type=int, default=320)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=None, help="JSONL audit log of the master")
    a = ap.parse_args()
    obj = {"kind": "measured_latency", "alpha": -0.2, "lo": 1e-5, "hi": 1e-2}
    config = {"budget": {"epochs": 2}, "objective": obj, "seed": 0, "precision": "bf16"}
    log = JsonlLog(a.out) if a.out else None
    master = Master(SearchSpace(), ObjectiveConfig(**obj),
                    EvolutionSettings(capacity=a.capacity, elite_count=2, tournament_size=3, crossover_prob=0.5,
                                      max_evaluations=a.evals), seed=a.seed, log=log)
    failures = []
    collect = master.collect

    def counted(record):
        if not record.ok:
            failures.append(record.failure_reason)
        collect(record)
    master.collect = counted
    first = {}  # device -> time of that worker process's first work request
    issue = master.issue

    def timed_issue(worker_id):
        dev = worker_id.split("s")[0]
        first.setdefault(dev, time.perf_counter())
        return issue(worker_id)
    master.issue = timed_issue
    pool = ProcessGpuPool(master, config, devices=tuple(range(a.gpus)), slots_per_gpu=a.slots, order="fifo")
    t0 = time.perf_counter()
    report = pool.run()
    wall = time.perf_counter() - t0
    if log:
        log.close()
    best = master.best
    busy = {w: round(s.busy_time_s / max(wall, 1e-9), 3) for w, s in sorted(report.stats.items())}
    # the clock starts once EVERY worker process is up (its first work request), so
    # slower CUDA-context start-up of some processes does not count as GA time
    ready = max(first.values()) - t0 if len(first) == a.gpus else None
    print(json.dumps({
        "config": "C3 steady-state GA", "gpus": a.gpus, "slots_per_gpu": a.slots, "capacity": a.capacity,
        "evaluations": master.completed, "wall_s": round(wall, 3),
        "startup_s": round(ready, 3) if ready is not None else None,
        "first_request_s": {d: round(t - t0, 3) for d, t in sorted(first.items())},
        "candidates_per_h": master.completed / (wall - (ready or 0.0)) * 3600.0,
        "candidates_per_h_incl_startup": master.completed / wall * 3600.0,
        "note": "candidates_per_h is timed from the moment every worker process has made its first work request",
        "failures": len(failures), "failure_reasons": sorted(set(map(str, failures)))[:8],
        "best_genome": format_genome(best.genome) if best else None,
        "best_fitness": best.record.fitness if best and best.record.ok else None,
        "protocol_errors": master.protocol_errors, "worker_busy_frac": busy}))


if __name__ == "__main__":
    main()
