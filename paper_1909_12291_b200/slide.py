"""Streamed whole-slide inference and the classification report.

The reference scores a patch set with predict_scores (evaluator.py:174-186)
and reports F1 / AUC / confusion plus a prediction rate and the whole-slide
time at 200,000 patches (metrics.py:77-119; SPEC.md cli-report predict_cmd).
Here the patches stay u8 in host memory and stream to the B200 through
ce_predict_stream: pinned H2D copies on a copy stream, double-buffered against
the u8 -> bf16 gather, the forward and the softmax head on the compute stream.
The rate is device-timed from the first copy to the last result.
"""

import numpy as np

from . import native
from .scoring import MetricsReport, auc_roc, confusion_counts, f1_degenerate, f1_score, slide_seconds

__all__ = ["pinned_pixels", "predict_stream", "predict_report", "predict_cmd"]


def pinned_pixels(pixels):
    """Copy u8 NCHW patches into page-locked host memory (torch), so that
    repeated streams skip the per-call page locking."""
    import torch
    t = torch.empty(pixels.shape, dtype=torch.uint8, pin_memory=True)
    t.numpy()[...] = pixels
    return t


def predict_stream(network, pixels, batch_size=128):
    """(scores f64, preds i64, device seconds) for u8 NCHW host patches."""
    if len(pixels) == 0:
        raise ValueError("empty patch stream")
    if tuple(pixels.shape[1:]) != tuple(network.input_shape):
        raise ValueError(f"patches {tuple(pixels.shape[1:])} do not match the model input {network.input_shape}")
    return network.device_net.predict_stream(pixels, batch_size)


def predict_report(network, pset, batch_size=128, warmup=1, model_id="", dataset_id="", pixels=None):
    """MetricsReport of `network` on `pset` with the streamed prediction rate.

    `pixels` may pass a pinned copy of pset.pixels (see pinned_pixels)."""
    px = pset.pixels if pixels is None else pixels
    for _ in range(warmup):
        predict_stream(network, px[:min(len(px), batch_size)], batch_size)
    scores, preds, secs = predict_stream(network, px, batch_size)
    labels = np.asarray(pset.labels)
    conf = confusion_counts(preds, labels)
    rate = len(px) / secs
    return MetricsReport(f1=f1_score(conf["tp"], conf["fp"], conf["fn"]), auc=auc_roc(scores, labels),
                         confusion=conf, prediction_rate_patches_per_s=rate, model_id=model_id,
                         dataset_id=dataset_id, f1_degenerate=f1_degenerate(conf["tp"], conf["fp"], conf["fn"]),
                         extras={"slide_seconds": slide_seconds(rate), "batch_size": batch_size,
                                 "device_seconds": secs, "patches": len(px)})


def predict_cmd(model_path, patchset_path, batch_size=128, precision="bf16", device=0):
    """SPEC.md predict_cmd: load an MNDL model and a PSET file, stream the
    patches through the model on `device`, return the MetricsReport."""
    from .model_io import load_candidate
    from .patches import load_patchset
    pset = load_patchset(patchset_path)
    net = load_candidate(model_path, pset.pixels.shape[1:], model_id=str(model_path))
    net.to_device(device, precision, max_batch=batch_size)
    try:
        return predict_report(net, pset, batch_size, model_id=str(model_path), dataset_id=str(patchset_path))
    finally:
        net.release()
