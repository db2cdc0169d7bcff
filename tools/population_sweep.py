"""C5: one generation of 512 bootstrap-random genomes
(Master(capacity=512, max_evaluations=512, seed=0)) at N GPUs x K slots, total
work fixed (strong scaling). One process per GPU under torchrun; the genomes
are sharded longest-estimated-first over the ranks (population.shard_lpt, no
data-path collective), each rank runs population.evaluate_population on its
shard, and the generation time is the max over ranks (device synchronised,
barrier on both sides).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port 29511 tools/population_sweep.py --slots K [--population 512]

Rank 0 prints one JSON line (candidates/h for the generation, per-rank times).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--population", type=int, default=512)
    ap.add_argument("--slots", type=int, default=4)
    ap.add_argument("--order", default="two_ended")
    ap.add_argument("--pull", type=int, default=0,
                    help="N>0: no torchrun; one master pulls work for N GPU worker processes "
                         "(scheduler.ProcessGpuPool, longest-estimated first) instead of static LPT shards")
    a = ap.parse_args()
    if a.pull:
        return pull_mode(a)
    import torch
    import torch.distributed as dist
    from paper_1909_12291_b200 import (EvolutionSettings, Master, ObjectiveConfig, SearchSpace, TrainBudget,
                                       estimate_cost, evaluate_population)
    from paper_1909_12291_b200.patches import default_splits
    from paper_1909_12291_b200.population import shard_lpt
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0),
               EvolutionSettings(capacity=a.population, max_evaluations=a.population), seed=0)
    genomes = [m.issue("sweep") for _ in range(a.population)]
    splits = default_splits()
    budget = TrainBudget(epochs=2)
    obj = ObjectiveConfig("measured_latency", -0.2, 1e-5, 1e-2)
    mine = shard_lpt(genomes, world, lambda g: estimate_cost(g, len(splits.train), budget))[rank]
    # warm-up: library load, device pools, one tiny candidate per slot
    evaluate_population(mine[-a.slots:], splits, TrainBudget(epochs=1, max_batches_per_epoch=2), obj, 0,
                        devices=(local,), slots_per_gpu=a.slots, order=a.order)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    recs, report = evaluate_population(mine, splits, budget, obj, 0, devices=(local,), slots_per_gpu=a.slots,
                                       order=a.order)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt, float(sum(1 for r in recs if r is not None and r.ok)), float(len(recs))],
                     device="cuda", dtype=torch.float64)
    if world > 1:
        ts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(ts, t)
        dist.barrier()
    else:
        ts = [t]
    import collections
    reasons = collections.Counter(" ".join(str(r.failure_reason).split()[:3]) for r in recs
                                  if r is not None and not r.ok)
    from paper_1909_12291_b200.genes import format_genome
    byid = {g.id: g for g in mine}
    top = sorted(report.trace, key=lambda t: t[2] - t[3])[:4]
    print(json.dumps({"rank": rank, "failure_reasons": reasons.most_common(6),
                      "longest": [[round(b - a, 3), format_genome(byid[gid])] for gid, _, a, b in top]}),
          file=sys.stderr, flush=True)
    if rank == 0:
        per = [x.tolist() for x in ts]
        tmax = max(p[0] for p in per)
        print(json.dumps({"config": "C5 single-generation sweep", "population": a.population, "gpus": world,
                          "slots_per_gpu": a.slots, "order": a.order, "generation_s": round(tmax, 3),
                          "candidates_per_h": a.population / tmax * 3600.0,
                          "per_rank_s": [round(p[0], 3) for p in per], "ok": int(sum(p[1] for p in per)),
                          "evaluated": int(sum(p[2] for p in per)), "scaling": "strong"}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def pull_mode(a):
    """Dynamic balance across GPUs: every slot of every GPU pulls the next
    longest-estimated candidate from one master (candidates whose cost the
    static estimate misjudges no longer pin one rank)."""
    import collections
    from paper_1909_12291_b200 import EvolutionSettings, Master, ObjectiveConfig, SearchSpace, estimate_cost
    from paper_1909_12291_b200.population import ListMaster
    from paper_1909_12291_b200.scheduler import ProcessGpuPool
    m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0),
               EvolutionSettings(capacity=a.population, max_evaluations=a.population), seed=0)
    genomes = [m.issue("sweep") for _ in range(a.population)]
    obj = {"kind": "measured_latency", "alpha": -0.2, "lo": 1e-5, "hi": 1e-2}
    config = {"budget": {"epochs": 2}, "objective": obj, "seed": 0, "precision": "bf16"}
    master = ListMaster(genomes)
    pool = ProcessGpuPool(master, config, devices=tuple(range(a.pull)), slots_per_gpu=a.slots, order="lpt",
                          cost_fn=lambda g: estimate_cost(g, 4000, None))
    first = []
    issue = master.issue

    def timed_issue(worker_id):  # the clock starts when the first worker asks for work
        if not first:
            first.append(time.perf_counter())
        return issue(worker_id)
    master.issue = timed_issue
    t0 = time.perf_counter()
    pool.run()
    t1 = time.perf_counter()
    dt = t1 - first[0]
    recs = list(master.records.values())
    reasons = collections.Counter(" ".join(str(r.failure_reason).split()[:3]) for r in recs if not r.ok)
    print(json.dumps({"config": "C5 single-generation sweep", "population": a.population, "gpus": a.pull,
                      "slots_per_gpu": a.slots, "order": "pull (one master, LPT issue)",
                      "generation_s": round(dt, 3), "candidates_per_h": a.population / dt * 3600.0,
                      "ok": sum(1 for r in recs if r.ok), "evaluated": len(recs), "scaling": "strong",
                      "failure_reasons": reasons.most_common(4),
                      "startup_s": round(first[0] - t0, 3),
                      "note": "clock starts at the first work request (worker start-up excluded)"}), flush=True)


if __name__ == "__main__":
    main()
