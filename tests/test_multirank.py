"""N>1 host logic on CPU: two gloo ranks deal the same generation to their
slot workers from ONE shared queue (TCPStore counters, as bench.py does):
every candidate is claimed exactly once, big slots take from the long end and
the others from the short end, and a fast rank steals the slow rank's share.
Timings combine as the bench does (max over ranks, sum of counts)."""

import os
import threading
import time

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, out, slow_rank):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1909_12291_b200 import TrainBudget
    from paper_1909_12291_b200.population import SharedQueueMaster, StoreCounter, estimate_cost
    from paper_1909_12291_b200.scheduler import is_big_slot
    genomes = bench.workload_genomes("c2", world)
    store = dist.distributed_c10d._get_default_store()
    master = SharedQueueMaster(genomes, StoreCounter(store, "gen1"), lambda g: estimate_cost(g, 4000, TrainBudget()),
                               big_worker=lambda wid: is_big_slot(wid, 1))
    claimed = {}

    def slot(k):
        wid = f"g{rank}s{k}"
        while True:
            g = master.issue(wid)
            if g is None:
                return
            claimed.setdefault(wid, []).append(g.id)
            time.sleep(0.05 if rank == slow_rank else 0.005)

    threads = [threading.Thread(target=slot, args=(k,)) for k in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    allc = [None] * world
    dist.all_gather_object(allc, claimed)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n = torch.tensor([float(sum(len(v) for v in claimed.values()))], dtype=torch.float64)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    if rank == 0:
        out.put((allc, [g.id for g in master.genomes], t.item(), n.item()))
    dist.destroy_process_group()


def test_two_rank_shared_queue():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, 1)) for r in range(2)]
    for p in procs:
        p.start()
    allc, order, tmax, count = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = [i for per_rank in allc for v in per_rank.values() for i in v]
    assert sorted(ids) == sorted(order) and len(order) == 32 and len(set(ids)) == 32
    assert tmax == 2.0 and count == 32.0
    # big slots (s0) claim a prefix of the longest-first order, the others a suffix (two-ended)
    big = [i for per_rank in allc for wid, v in per_rank.items() if wid.endswith("s0") for i in v]
    small = [i for per_rank in allc for wid, v in per_rank.items() if not wid.endswith("s0") for i in v]
    assert set(big) == set(order[:len(big)]) and set(small) == set(order[len(order) - len(small):])
    # work stealing: the fast rank (0) took more than its static half
    assert sum(len(v) for v in allc[0].values()) > 16


def test_replicas_keep_the_per_gpu_work_fixed():
    import bench
    base = bench.workload_genomes("c2", 1)
    four = bench.workload_genomes("c2", 4)
    assert len(base) == 16 and len(four) == 64 and len({g.id for g in four}) == 64
    for r in range(4):
        chunk = four[16 * r:16 * (r + 1)]
        assert [(g.feature_layers, g.head_layers, g.learn) for g in chunk] == \
               [(g.feature_layers, g.head_layers, g.learn) for g in base]


def test_local_counter_matches_store_semantics():
    from paper_1909_12291_b200.population import LocalCounter, SharedQueueMaster
    import bench
    gs = bench.workload_genomes("c2", 1)
    m = SharedQueueMaster(gs, LocalCounter(), lambda g: len(g.feature_layers), big_worker=lambda wid: wid == "big")
    got = []
    while True:
        g = m.issue("big" if len(got) % 3 == 0 else "small")
        if g is None:
            break
        got.append(g.id)
    assert sorted(got) == sorted(g.id for g in gs)
    assert m.issue("big") is None


if __name__ == "__main__":
    pytest.main([__file__, "-q"])
