"""MNDL container (paper_1909_12291_b200/model_io.py) against a fixture the
REFERENCE serializer wrote (tests/golden/make_mndl.py): byte-exact decode /
encode, candidate export bit-exact to the reference's instantiate(seed=0)
file, and the reference's FormatError offsets (model_io.py:70-152)."""

import json
import os
import struct

import numpy as np
import pytest

from paper_1909_12291_b200 import model_io
from paper_1909_12291_b200.faults import FormatError
from paper_1909_12291_b200.genes import format_genome, parse_genome
from paper_1909_12291_b200.network import instantiate
from paper_1909_12291_b200.scoring import MetricsReport

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
META = json.load(open(os.path.join(GOLD, "small_mndl.json")))
DATA = open(os.path.join(GOLD, "small.mndl"), "rb").read()


def test_decode_encode_round_trip_is_byte_exact():
    specs = model_io.decode_mndl(DATA)
    assert [s[0] for s in specs] == ["conv", "relu", "pool", "conv", "relu", "flatten", "dense", "dense"]
    assert model_io.encode_mndl(specs) == DATA


def test_candidate_export_matches_reference_file():
    net = instantiate(parse_genome(META["genome"]), tuple(META["input_shape"]), seed=0)
    assert model_io.encode_mndl(model_io.specs_of(net)) == DATA


def test_genome_of_specs():
    g = model_io.genome_of_specs(model_io.decode_mndl(DATA))
    ref = parse_genome(META["genome"])
    assert g.feature_layers == ref.feature_layers and g.head_layers == ref.head_layers
    assert "f0=conv:oc=8,k=3,s=1,relu=1" in format_genome(g)


def test_load_candidate_host(tmp_path):
    path = tmp_path / "m.mndl"
    path.write_bytes(DATA)
    net = model_io.load_candidate(str(path), tuple(META["input_shape"]))
    ref = instantiate(parse_genome(META["genome"]), tuple(META["input_shape"]), seed=0)
    for (w, b), (rw, rb) in zip(net.weights, ref.weights):
        np.testing.assert_array_equal(w, rw)
        np.testing.assert_array_equal(b, rb)
    with pytest.raises(FormatError):
        model_io.load_candidate(str(path), (3, 26, 26))  # flatten width 400 != 256


@pytest.mark.parametrize("mutate,offset", [
    (lambda d: b"XXXX" + d[4:], 0),
    (lambda d: d[:4] + struct.pack("<I", 2) + d[8:], 4),
    (lambda d: d[:-3], None),
    (lambda d: d + b"\0", len(DATA)),
])
def test_format_errors(mutate, offset):
    with pytest.raises(FormatError) as e:
        model_io.decode_mndl(mutate(DATA))
    if offset is not None:
        assert e.value.offset == offset


def test_unknown_tag():
    bad = DATA[:12] + bytes([9]) + DATA[13:]
    with pytest.raises(FormatError) as e:
        model_io.decode_mndl(bad)
    assert e.value.offset == 12


def test_report_text():
    r = MetricsReport(f1=0.5, auc=0.75, confusion={"tp": 1, "fp": 1, "fn": 1, "tn": 1},
                      prediction_rate_patches_per_s=1000.0, model_id="m", dataset_id="d")
    txt = r.to_text()
    assert "est. slide time:  200.0 s" in txt and "tp=1 fp=1 fn=1 tn=1" in txt
    assert json.loads(r.to_json())["prediction_rate_patches_per_s"] == 1000.0
