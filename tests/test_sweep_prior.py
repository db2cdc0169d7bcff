"""Sweep -> throughput prior host pipeline against the reference
(tests/golden/sweep.json from tests/golden/make_sweep_golden.py): build_prior,
CSV round trip, top-k, timing_distribution and prior-biased random_genome
draws (bench.py:80-238, genome.py:122-173) are bit-exact."""

import json
import os

import numpy as np
import pytest

from paper_1909_12291_b200 import sweep
from paper_1909_12291_b200.genes import SearchSpace, format_genome, random_genome

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sweep.json")))


def rows():
    return [sweep.SweepRow(in_channels=r[0], out_channels=r[1], kernel=r[2], stride=r[3], batch_size=r[4],
                           height=24, width=24, median_forward_backward_s=r[5], flops_per_layer=r[6],
                           flops_per_s=r[7]) for r in GOLD["rows"]]


def test_grid_and_flops():
    g = sweep.SweepGrid()
    assert g.size() == 4 * 5 * 6 * 3 * 2 == len(list(g.configs()))
    for r in GOLD["rows"][:50]:
        assert sweep.conv_layer_flops(r[0], r[1], r[2], r[3], 24, 24) == r[6]


def test_build_prior_matches_reference():
    prior = sweep.build_prior(rows(), k=40, beta=0.5)
    for hp in ("out_channels", "kernel", "stride"):
        got = {str(k): v for k, v in getattr(prior, hp).items()}
        assert got == GOLD["prior"][hp]
    with pytest.raises(ValueError):
        sweep.top_k_by_throughput(rows(), len(GOLD["rows"]) + 1)


def test_prior_biased_genomes_match_reference():
    prior = sweep.build_prior(rows(), k=40, beta=0.5)
    rng = np.random.default_rng(0)
    got = [format_genome(random_genome(rng, SearchSpace(), prior=prior)) for _ in range(50)]
    assert got == GOLD["genomes_with_prior"]


def test_csv_round_trip(tmp_path):
    path = tmp_path / "sweep.csv"
    sweep.write_sweep_csv(rows(), str(path))
    assert path.read_text().splitlines()[0] == ",".join(sweep.SWEEP_CSV_FIELDS)
    again = sweep.read_sweep_csv(str(path))
    assert again == rows()


@pytest.mark.parametrize("name", ["unimodal", "bimodal"])
def test_timing_distribution(name):
    g = GOLD["timing"][name]
    s = sweep.timing_distribution(g["values"], bins=20)
    assert s.modes == g["modes"]
    assert list(s.mode_centers) == g["centers"]
    assert s.separation_stat == g["stat"]
    assert [int(c) for c in s.counts] == g["counts"]
    with pytest.raises(ValueError):
        sweep.timing_distribution(g["values"][:29])
