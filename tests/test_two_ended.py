"""PoolCore "two_ended" dispatch: big workers take the longest remaining
payload, the others the shortest; every payload is issued exactly once."""

from dataclasses import dataclass

from paper_1909_12291_b200.candidate import EvalRecord
from paper_1909_12291_b200.scheduler import PoolCore


@dataclass(frozen=True)
class P:
    id: str
    cost: float


class M:
    def __init__(self, items):
        self.items, self.done = list(items), []

    def issue(self, wid):
        return self.items.pop(0) if self.items else None

    def collect(self, rec):
        self.done.append(rec.genome_id)


def test_two_ended_order():
    payloads = [P(f"p{i}", c) for i, c in enumerate([5, 1, 9, 3, 7, 2])]
    m = M(payloads)
    core = PoolCore(m, order="two_ended", cost_fn=lambda p: p.cost)
    core.big_worker = lambda wid: wid == "big"
    got = [core.get_work("big").cost, core.get_work("small").cost, core.get_work("small").cost,
           core.get_work("big").cost, core.get_work("small").cost, core.get_work("big").cost]
    assert got == [9, 1, 2, 7, 3, 5]
    assert core.get_work("big") is None
    for p in payloads:
        core.submit(EvalRecord(genome_id=p.id, ok=True))
    assert core.finished() and sorted(m.done) == sorted(p.id for p in payloads)
