"""N>1 host logic on CPU: two gloo ranks build the same 16*N bootstrap
population, take disjoint LPT shards that cover it, and combine per-rank
timings as the bench does (max over ranks, sum of counts)."""

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1909_12291_b200 import TrainBudget
    from paper_1909_12291_b200.population import estimate_cost, shard_lpt
    genomes = bench.population(world)
    mine = shard_lpt(genomes, world, lambda g: estimate_cost(g, 4000, TrainBudget()))[rank]
    ids = [None] * world
    dist.all_gather_object(ids, [g.id for g in mine])
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n = torch.tensor([float(len(mine))], dtype=torch.float64)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    if rank == 0:
        out.put((ids, [g.id for g in genomes], t.item(), n.item()))
    dist.destroy_process_group()


def test_two_rank_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ids, all_ids, tmax, count = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert set(ids[0]).isdisjoint(ids[1])
    assert sorted(ids[0] + ids[1]) == sorted(all_ids) and len(all_ids) == 32
    assert tmax == 2.0 and count == 32.0


def test_lpt_balances_better_than_fifo():
    import bench
    from paper_1909_12291_b200 import TrainBudget
    from paper_1909_12291_b200.population import estimate_cost, shard_lpt
    genomes = bench.population(8)
    cost = lambda g: estimate_cost(g, 4000, TrainBudget())  # noqa: E731
    lpt = max(sum(cost(g) for g in s) for s in shard_lpt(genomes, 8, cost))
    fifo = max(sum(cost(g) for g in genomes[i::8]) for i in range(8))
    assert lpt <= fifo
    assert lpt <= 1.2 * sum(cost(g) for g in genomes) / 8 + max(cost(g) for g in genomes)


if __name__ == "__main__":
    pytest.main([__file__, "-q"])
