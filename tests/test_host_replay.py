"""T5: the host-side restatements are bit-exact to the reference given the
same seeds, records and arrival order (golden fixtures from convevo)."""

import hashlib
import json
import os
from dataclasses import replace

import numpy as np
import pytest

from paper_1909_12291_b200 import genes as G
from paper_1909_12291_b200 import ga, patches, scoring
from paper_1909_12291_b200.candidate import EvalRecord
from paper_1909_12291_b200.network import instantiate

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def host():
    with open(os.path.join(GOLD, "host.json")) as fh:
        return json.load(fh)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.slow
def test_synthetic_data_and_split_bytes(host):
    d = patches.generate_synthetic(*patches.default_counts(4800), h=100, w=100, seed=0)
    gold = host["data"]
    assert list(patches.default_counts(4800)) == gold["counts"]
    assert sha(d.pixels) == gold["pixels"] and sha(d.labels) == gold["labels"]
    sp = patches.stratified_split(d, (5 / 6, 1 / 12, 1 / 12), seed=0)
    for name in ("train", "val"):
        part = getattr(sp, name)
        n, hp, hl, pos = gold[name]
        assert (len(part), sha(part.pixels), sha(part.labels), int(part.labels.sum())) == (n, hp, hl, pos)
    assert [len(sp.test), sha(sp.test.pixels), sha(sp.test.labels)] == gold["test"]


def test_small_synthetic_bytes(host):
    d = patches.generate_synthetic(5, 7, h=40, w=36, seed=3)
    assert sha(d.pixels) == host["data_small"]["pixels"]
    assert d.labels.tolist() == host["data_small"]["labels"]


def test_instantiate_weights_bit_exact(host):
    shapes = {"small": (3, 24, 24)}
    from tests_golden_genomes import GENOMES  # noqa
    for name, gold in host["instantiate"].items():
        net = instantiate(G.parse_genome(GENOMES[name]), shapes.get(name, (3, 100, 100)), seed=0)
        assert net.flops_inference() == gold["flops"]
        assert net.param_count() == gold["count"]
        ours = [[i, nm, list(a.shape), sha(a)] for i, nm, a in net.parameters()]
        assert [o[1:] for o in ours] == [g[1:] for g in gold["params"]], name


def test_flop_and_param_accounting(host):
    for text, flops, params in host["accounting"]:
        g = G.parse_genome(text)
        assert G.format_genome(g) == text
        if flops is None:
            continue
        from paper_1909_12291_b200.network import Network, build_layers
        net = Network(g, (3, 100, 100), build_layers(g, (3, 100, 100)), [])
        assert (net.flops_inference(), net.param_count()) == (flops, params), text


def test_genome_operators_bit_exact(host):
    gold = host["genome_ops"]
    space = G.SearchSpace()
    prior = G.ThroughputPrior(out_channels={256: 0.5, 64: 0.5}, kernel={4: 0.7, 3: 0.3}, stride={1: 1.0}, beta=0.5)
    rng = np.random.default_rng(42)
    gs = []
    for i in range(400):
        g = G.random_genome(rng, space, prior if i % 3 == 0 else None)
        gs.append(g)
        assert G.format_genome(g) == gold["random"][i]
        assert G.parse_genome(gold["random"][i]) == g
    for i in range(300):
        assert G.format_genome(G.mutate(gs[i], rng, G.MutationRates(), space, prior if i % 2 else None)) == \
            gold["mutate"][i]
    for i in range(300):
        assert G.format_genome(G.crossover(gs[i], gs[i + 1], rng, space.input_shape)) == gold["crossover"][i]
    assert str(rng.bit_generator.state) == gold["final_state"]


def _fake_record(genome):
    f = (int(genome.id[:6], 16) % 1000) / 1000.0
    flops = sum(getattr(g, "out_channels", 1) for g in genome.feature_layers)
    ok = int(genome.id[6], 16) != 0
    return EvalRecord(genome_id=genome.id, ok=ok, val_f1=f, flops_inference=flops,
                      fitness=f if ok else scoring.FAILED_FITNESS)


def test_ga_replay_bit_exact(host):
    for run in host["ga"]:
        settings = ga.EvolutionSettings(capacity=8, elite_count=2, max_evaluations=40)
        m = ga.Master(G.SearchSpace(), scoring.ObjectiveConfig("flop_proxy", -0.2, 1.0, 100.0), settings,
                      seed=run["seed"])
        issued, inflight = [], []
        for ev in run["events"]:
            if ev[0] == "issue":
                g = m.issue("w")
                issued.append(G.format_genome(g))
                inflight.append(g)
            else:
                m.collect(_fake_record(inflight.pop(ev[1])))
        assert issued == run["issued"], (run["seed"], run["mode"])
        assert m.best.record.genome_id == run["best"]
        assert [mb.genome.id for mb in m.population.members] == run["population"]
        assert str(m.rng.bit_generator.state) == run["rng_state"]


def test_scoring_kats():
    assert scoring.f1_score(8, 2, 2) == 0.8000000000000002
    assert scoring.auc_roc([0.9, 0.4, 0.5, 0.1], [1, 1, 0, 0]) == 0.75
    assert scoring.normalize_objective(0.0505, 0.001, 0.1) == 0.5
    assert scoring.fitness(0.8, 0.5, -0.2) == 0.7000000000000001
    assert scoring.confusion_counts([1, 0, 1, 0], [1, 1, 0, 0]) == {"tp": 1, "fp": 1, "fn": 1, "tn": 1}
    with pytest.raises(ValueError):
        scoring.auc_roc([0.1, 0.2], [1, 1])
    a = EvalRecord("a", fitness=0.5, flops_inference=10)
    b = EvalRecord("b", fitness=0.5, flops_inference=5)
    c = EvalRecord("c", ok=False)
    assert sorted([a, b, c], key=scoring.sort_key) == [b, a, c]


def test_genome_kats():
    space = G.SearchSpace()
    g = G.Genome((G.ConvGene(8, 4, 1),), (), G.LearnParams(0.01, 0.9, 32), "x")
    assert G.validate_shapes(g, (3, 100, 100)).feature_shapes == ((8, 97, 97),)
    bad = G.Genome((G.ConvGene(8, 101, 1),), (), G.LearnParams(0.01, 0.9, 32), "x")
    with pytest.raises(G.ShapeError) as e:
        G.validate_shapes(bad, (3, 100, 100))
    assert (e.value.layer_index, e.value.dimension) == (0, "rows")
    empty = G.Genome((), (), G.LearnParams(0.01, 0.9, 32), "x")
    assert G.validate_shapes(empty, (3, 100, 100)).flat_units == 30000
    two = G.Genome((G.ConvGene(8, 7, 3), G.ConvGene(8, 7, 3)), (), G.LearnParams(0.01, 0.9, 32), "x")
    assert len(G.repair(two, (3, 8, 8)).feature_layers) == 1
    rng = np.random.default_rng(0)
    a = G.random_genome(rng, space)
    child = G.crossover(a, a, rng)
    assert child.feature_layers == a.feature_layers
    m = G.mutate(a, rng, G.MutationRates.zero(), space)
    assert m.same_structure(a) and m.parent_ids == (a.id,)
    assert G.parse_genome(G.format_genome(m)) == m


def test_calibrate_and_audit(tmp_path):
    space = G.SearchSpace()
    m = ga.Master(space, scoring.ObjectiveConfig("flop_proxy", -0.2), ga.EvolutionSettings(capacity=4,
                                                                                           max_evaluations=12))
    vals = iter([10.0, 20.0])
    assert ga.calibrate(m, lambda g: next(vals), 2) == (9.0, 22.0)
    log = ga.JsonlLog(tmp_path / "run.jsonl")
    m.log = log
    ga.write_header(log, m.objective, m.settings, 0)
    ga.run_serial(m, lambda g, wid: replace(_fake_record(g), worker_id=wid))
    log.close()
    summary = ga.audit_log(tmp_path / "run.jsonl")
    assert summary["evaluations"] == 12
