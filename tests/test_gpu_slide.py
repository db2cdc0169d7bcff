"""MNDL models on the B200 and streamed whole-slide prediction.

- the reference-written fixture (tests/golden/small.mndl) loads into the
  operator API (nn.Network) and into the candidate runtime; both reproduce the
  reference's logits (fp32 <= 1e-5, bf16 <= 1e-2) and save back byte-exactly;
- ce_predict_stream (host u8 patches, double-buffered H2D) gives exactly the
  scores / predictions of ce_predict on the device-resident set, for pageable
  and pinned input and a ragged last chunk;
- predict_report / predict_cmd produce a consistent MetricsReport."""

import json
import os

import numpy as np
import pytest
import torch

from paper_1909_12291_b200 import model_io, slide
from paper_1909_12291_b200.candidate import predict_scores
from paper_1909_12291_b200.network import instantiate
from paper_1909_12291_b200.genes import FIXED, parse_genome
from paper_1909_12291_b200.patches import PatchSet, generate_synthetic, save_patchset

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
META = json.load(open(os.path.join(GOLD, "small_mndl.json")))
PATH = os.path.join(GOLD, "small.mndl")


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def batch():
    return np.random.default_rng(META["batch_seed"]).random((META["batch"], *META["input_shape"]), dtype=np.float32)


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-5), ("bf16", 1e-2)])
def test_operator_api_loads_reference_model(prec, tol, tmp_path):
    net = model_io.load_network(PATH, dtype=np.float32 if prec == "fp32" else "bf16")
    logits = net.forward(torch.from_numpy(batch()).cuda()).cpu().numpy()
    assert rel(logits, META["logits"]) <= tol
    out = tmp_path / "again.mndl"
    model_io.save_network(net, str(out))
    assert out.read_bytes() == open(PATH, "rb").read()


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-5), ("bf16", 1e-2)])
def test_candidate_runtime_loads_reference_model(prec, tol, tmp_path):
    net = model_io.load_candidate(PATH, tuple(META["input_shape"]))
    dev = net.to_device(0, prec, max_batch=16)
    assert rel(dev.forward(batch()), META["logits"]) <= tol
    out = tmp_path / "cand.mndl"
    model_io.save_network(net, str(out))  # pulls the device weights back
    assert out.read_bytes() == open(PATH, "rb").read()
    net.release()


@pytest.mark.parametrize("pinned", [False, True])
def test_stream_matches_resident_predict(pinned):
    pset = generate_synthetic(180, 820, h=100, w=100, seed=3)
    net = instantiate(parse_genome(FIXED), (3, 100, 100), seed=0)
    net.to_device(0, "bf16", max_batch=128)
    s_res, p_res = predict_scores(net, pset, batch_size=128)
    px = slide.pinned_pixels(pset.pixels) if pinned else pset.pixels
    s_str, p_str, secs = slide.predict_stream(net, px, batch_size=128)  # 1000 = 7 x 128 + 104
    np.testing.assert_array_equal(s_str, s_res)
    np.testing.assert_array_equal(p_str, p_res)
    assert secs > 0
    net.release()


def test_predict_cmd(tmp_path):
    pset = generate_synthetic(60, 140, h=100, w=100, seed=4)
    ppath = tmp_path / "val.pset"
    save_patchset(pset, str(ppath))
    mpath = tmp_path / "fixed.mndl"
    model_io.save_network(instantiate(parse_genome(FIXED), (3, 100, 100), seed=0), str(mpath))
    rep = slide.predict_cmd(str(mpath), str(ppath), batch_size=64, precision="bf16")
    c = rep.confusion
    assert c["tp"] + c["fp"] + c["fn"] + c["tn"] == 200
    assert rep.prediction_rate_patches_per_s > 0 and 0.0 <= rep.auc <= 1.0
    assert rep.extras["slide_seconds"] == pytest.approx(200000 / rep.prediction_rate_patches_per_s)
    assert "est. slide time" in rep.to_text()
