"""Device-level failures never turn into candidate results (SURVEY §5,
failure detection): a sticky CUDA fault propagates out of evaluate(), retires
that GPU's workers and reissues the candidate to a healthy device (in-process
GpuPool and the socket transport); an out-of-memory status is retried once
with the device to itself before the candidate is failed."""

import threading
import time

import numpy as np
import pytest

from paper_1909_12291_b200 import candidate
from paper_1909_12291_b200.candidate import LEASES, EvalRecord, TrainBudget, evaluate
from paper_1909_12291_b200.faults import CE_ECUDA, CE_ENOMEM, NativeError
from paper_1909_12291_b200.genes import FIXED, SearchSpace, parse_genome, random_genome
from paper_1909_12291_b200.patches import PatchSet, Splits
from paper_1909_12291_b200.population import ListMaster
from paper_1909_12291_b200.scheduler import GpuPool, SocketPool, run_socket_worker
from paper_1909_12291_b200.scoring import ObjectiveConfig

STICKY = "an illegal memory access was encountered"


def tiny_splits():
    rng = np.random.default_rng(0)
    ps = [PatchSet(rng.integers(0, 256, (n, 3, 100, 100)).astype(np.uint8), (np.arange(n) % 2).astype(np.uint8))
          for n in (8, 8, 8)]
    return Splits(*ps)


def genomes(n, seed=0):
    rng = np.random.default_rng(seed)
    return [random_genome(rng, SearchSpace()) for _ in range(n)]


def _run_evaluate(monkeypatch, raise_fn):
    monkeypatch.setattr(candidate, "train_short", raise_fn)
    return evaluate(parse_genome(FIXED), tiny_splits(), TrainBudget(epochs=1), ObjectiveConfig("flop_proxy", 0.0, 1, 2),
                    seed=0, device=0)


def test_sticky_fault_propagates_out_of_evaluate(monkeypatch):
    def boom(*a, **k):
        raise NativeError(CE_ECUDA, f"train loop: {STICKY}")
    with pytest.raises(NativeError) as ei:
        _run_evaluate(monkeypatch, boom)
    assert ei.value.sticky


def test_non_sticky_native_error_is_a_failed_record(monkeypatch):
    def bad(*a, **k):
        raise NativeError(CE_ECUDA, "invalid argument")
    rec = _run_evaluate(monkeypatch, bad)
    assert not rec.ok and "invalid argument" in rec.failure_reason and rec.fitness == float("-inf")


def test_enomem_is_retried_alone_then_failed(monkeypatch):
    calls = []

    def oom(*a, **k):
        calls.append(0 in LEASES._writer)  # exclusive lease held?
        raise NativeError(CE_ENOMEM, "device allocation of 1 bytes failed")
    rec = _run_evaluate(monkeypatch, oom)
    assert calls == [False, True]
    assert not rec.ok and rec.failure_reason.startswith("out of device memory")
    assert "enomem_retry" in rec.extras


def test_exclusive_lease_waits_for_shared_holders():
    order = []
    entered = threading.Event()

    def holder():
        with LEASES.shared(5):
            entered.set()
            time.sleep(0.2)
            order.append("shared done")

    t = threading.Thread(target=holder)
    t.start()
    entered.wait()
    with LEASES.exclusive(5):
        order.append("exclusive")
    t.join()
    assert order == ["shared done", "exclusive"]
    with LEASES.shared(6):  # other devices are independent
        pass


def test_gpu_pool_retires_faulted_device_and_reissues():
    gs = genomes(12)
    faults = []

    def fn(genome, worker_id, device):
        if device == 0:
            faults.append(genome.id)
            raise NativeError(CE_ECUDA, STICKY)
        time.sleep(0.005)
        return EvalRecord(genome_id=genome.id, ok=True, fitness=1.0, worker_id=worker_id)

    master = ListMaster(gs)
    pool = GpuPool(fn, master, devices=(0, 1), slots_per_gpu=2, order="fifo")
    report = pool.run()
    assert report.unhealthy_devices == (0,)
    assert len(master.records) == len(gs)
    assert all(r.ok and r.worker_id.startswith("g1") for r in master.records.values())
    assert 1 <= len(faults) <= 2 and report.timeouts_reissued == len(faults)


def test_socket_worker_drops_connection_on_sticky_fault():
    gs = genomes(10, seed=3)
    master = ListMaster(gs)
    pool = SocketPool(2, None, master, spawn_local_workers=False)
    stuck = []

    def faulty(genome, worker_id):
        raise NativeError(CE_ECUDA, STICKY)

    def good(genome, worker_id):
        time.sleep(0.01)
        return EvalRecord(genome_id=genome.id, ok=True, fitness=2.0, worker_id=worker_id)

    def start():
        threading.Thread(target=run_socket_worker, args=("127.0.0.1", pool.port, "g0s0", faulty, stuck.append),
                         daemon=True).start()
        time.sleep(0.05)
        threading.Thread(target=run_socket_worker, args=("127.0.0.1", pool.port, "g1s0", good),
                         daemon=True).start()
        return []

    pool._start_workers = start
    report = pool.run()
    assert len(stuck) == 1 and stuck[0].sticky
    assert len(master.records) == len(gs) and all(r.ok for r in master.records.values())
    assert report.timeouts_reissued == 1
