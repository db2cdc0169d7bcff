"""Socket transport (wire.py, scheduler.SocketPool): frame format of
convevo/wire.py, exactly-once collection over TCP with local worker threads,
and immediate reissue of work held by a worker that disconnects (the
process-per-GPU fault-isolation path)."""

import json
import socket
import struct
import threading

import numpy as np
import pytest

from paper_1909_12291_b200 import wire
from paper_1909_12291_b200.candidate import EvalRecord
from paper_1909_12291_b200.faults import ProtocolError
from paper_1909_12291_b200.genes import SearchSpace, format_genome, random_genome
from paper_1909_12291_b200.population import ListMaster
from paper_1909_12291_b200.scheduler import SocketPool, idle_fraction, start_pool


def genomes(n, seed=0):
    rng = np.random.default_rng(seed)
    return [random_genome(rng, SearchSpace()) for _ in range(n)]


def stub(genome, worker_id):
    return EvalRecord(genome_id=genome.id, ok=True, fitness=float(len(genome.feature_layers)), worker_id=worker_id)


def test_frame_bytes():
    a, b = socket.socketpair()
    with a, b:
        wire.send_message(a, "HELLO", "w3")
        raw = b.recv(64)
        assert raw == struct.pack(">I", 8) + b"HELLO w3"
        wire.send_message(a, "SHUTDOWN")
        assert wire.recv_message(b) == ("SHUTDOWN", "")
        a.sendall(struct.pack(">I", 0))
        with pytest.raises(ProtocolError):
            wire.recv_message(b)  # empty payload is not a known kind
        a.close()
        assert wire.recv_frame(b) is None  # clean EOF


def test_frame_errors():
    with pytest.raises(ProtocolError):
        wire.encode_message("BOGUS")
    with pytest.raises(ProtocolError):
        wire.decode_message(b"\xff\xfe")
    a, b = socket.socketpair()
    with a, b:
        a.sendall(struct.pack(">I", wire.MAX_FRAME + 1))
        with pytest.raises(ProtocolError):
            wire.recv_frame(b)
    a, b = socket.socketpair()
    with b:
        a.sendall(struct.pack(">I", 10) + b"RESU")
        a.close()
        with pytest.raises(ProtocolError):
            wire.recv_frame(b)


def test_socket_pool_exactly_once():
    gs = genomes(20)
    master = ListMaster(gs)
    pool = start_pool(4, stub, master, transport="socket")
    report = pool.run()
    assert sorted(master.records) == sorted(g.id for g in gs)
    assert sum(st.evaluations_done for st in report.stats.values()) == 20
    assert report.dropped_duplicates == 0
    assert 0.0 <= idle_fraction(report)["aggregate"] <= 1.0


def test_work_of_a_lost_worker_is_reissued():
    gs = genomes(6, seed=1)
    master = ListMaster(gs)
    pool = SocketPool(1, stub, master, spawn_local_workers=False)
    got = {}

    def deserter():
        with socket.create_connection(("127.0.0.1", pool.port)) as s:
            wire.send_message(s, "HELLO", "bad")
            wire.send_message(s, "REQ", "bad")
            kind, body = wire.recv_message(s)
            got["taken"] = body  # then drop the connection mid-evaluation

    def honest():
        from paper_1909_12291_b200.scheduler import run_socket_worker
        run_socket_worker("127.0.0.1", pool.port, "good", stub)

    runner = threading.Thread(target=lambda: got.setdefault("report", pool.run()), daemon=True)
    runner.start()  # accept loop up before anyone connects
    t = threading.Thread(target=deserter, daemon=True)
    t.start()
    t.join(timeout=10)
    w = threading.Thread(target=honest, daemon=True)
    w.start()
    runner.join(timeout=30)
    report = got["report"]
    assert sorted(master.records) == sorted(g.id for g in gs)
    assert all(r.ok for r in master.records.values())
    assert report.timeouts_reissued == 1
    assert got["taken"] == format_genome(gs[0])


def test_records_travel_as_reference_json():
    rec = EvalRecord(genome_id="abc", ok=False, failure_reason="non-finite loss", worker_id="g0s1")
    body = json.dumps(rec.to_json_dict(), sort_keys=True)
    back = EvalRecord.from_json_dict(json.loads(wire.decode_message(wire.encode_message("RESULT", body))[1]))
    assert back.genome_id == "abc" and not back.ok and back.fitness == rec.fitness
