"""Deferred measured-latency objectives (candidate.LatencyWindow): records are
completed in place at flush with the same raw objective / fitness arithmetic
as the immediate path (evaluator.py:213-243), and the device net is released."""

import numpy as np

from paper_1909_12291_b200.candidate import EvalRecord, LatencyWindow, raw_objective
from paper_1909_12291_b200.scoring import ObjectiveConfig, score


class _Dev:
    def latency(self, x, warmup, reps):
        return np.array([0.004, 0.002, 0.003, 0.005, 0.0025][:reps])


class _Net:
    input_shape = (3, 8, 8)
    device_net = _Dev()
    released = False

    def release(self):
        self.released = True


def test_flush_completes_records_in_place():
    obj = ObjectiveConfig("measured_latency", -0.2, 1e-3, 1e-2)
    rec = EvalRecord(genome_id="g", ok=True, val_f1=0.5, flops_inference=10, params=3, extras={"latency_pending": True})
    net = _Net()
    w = LatencyWindow()
    w.add(rec, net, 64, 5, 1, 0, obj)
    assert rec.latency is None
    w.flush()
    assert net.released and "latency_pending" not in rec.extras
    assert rec.latency.median_s_per_batch == 0.003
    raw = raw_objective(obj.kind, 10, 3, rec.latency)
    fv = score(0.5, raw, obj)
    assert (rec.objective_raw, rec.objective_m, rec.fitness) == (raw, fv.m, fv.f)
    assert not w.pending


class _SizedDev(_Dev):
    def __init__(self, nbytes):
        self.nbytes = nbytes

    def device_bytes(self):
        return self.nbytes


class _SizedNet(_Net):
    def __init__(self, nbytes):
        self.device_net = _SizedDev(nbytes)


def test_window_caps_held_device_bytes():
    """Past the cap a candidate is measured at once (C5: 512 deferred nets on one GPU)."""
    w = LatencyWindow(cap_bytes=100)
    assert w.try_reserve(_SizedNet(60))
    assert not w.try_reserve(_SizedNet(50))   # 110 > 100: measure inline
    assert w.try_reserve(_SizedNet(40))       # exactly at the cap
    assert w.held_bytes == 100 and w.measured_inline == 1
    w.flush()
    assert w.held_bytes == 0 and w.try_reserve(_SizedNet(90))


def test_window_measures_inline_without_size():
    assert not LatencyWindow().try_reserve(_Net())  # no device_bytes(): never defer blindly
