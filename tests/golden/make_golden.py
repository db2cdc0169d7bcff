"""Generate golden fixtures by running the REFERENCE (convevo) in the build
container. The reference never travels to the GPU box; these committed
fixtures (and the oracle they pin) do.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (small; big tensors are stored as SHA-256 digests):
  nn_ops.npz        conv / pool / dense / xent / sgd vectors (fp32 + fp64)
  train_steps.npz   one train_batch + a 10-step loss trajectory on small genomes
  host.json         data / split digests, instantiate digests, FLOP/param counts,
                    GA replay schedules and issued genome sequences, SPEC KATs,
                    a reduced-budget evaluate() record
"""

import hashlib
import json
import os
import platform
import sys

import numpy as np

REF = os.environ.get("CONVEVO_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from convevo import data as rdata  # noqa: E402
from convevo import evaluator as rev  # noqa: E402
from convevo import evolution as revo  # noqa: E402
from convevo import fitness as rfit  # noqa: E402
from convevo import genome as rgen  # noqa: E402
from convevo import nn as rnn  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, OUT)
import recipes  # noqa: E402

FIXED = ("id=fixed0000000000 parents= lr=0.0003 momentum=0.9 batch_size=64 "
         "f0=conv:oc=32,k=4,s=2,relu=1 f1=conv:oc=64,k=4,s=1,relu=1 f2=pool:size=2,s=2 "
         "f3=conv:oc=128,k=4,s=1,relu=1 h0=dense:units=64")
VGG16STYLE = ("id=vgg16style00000 parents= lr=0.01 momentum=0.9 batch_size=64 "
              "f0=conv:oc=64,k=3,s=1,relu=1 f1=conv:oc=64,k=3,s=1,relu=1 f2=pool:size=2,s=2 "
              "f3=conv:oc=128,k=3,s=1,relu=1 f4=conv:oc=128,k=3,s=1,relu=1 f5=pool:size=2,s=2 "
              "f6=conv:oc=256,k=3,s=1,relu=1 f7=conv:oc=256,k=3,s=1,relu=1 f8=conv:oc=256,k=3,s=1,relu=1 "
              "f9=pool:size=2,s=2 f10=conv:oc=256,k=3,s=1,relu=1 f11=conv:oc=256,k=3,s=1,relu=1 "
              "h0=dense:units=1024 h1=dense:units=1024")
SWEET = ("id=sweet00000000000 parents= lr=0.001 momentum=0.9 batch_size=64 "
         "f0=conv:oc=256,k=4,s=1,relu=1 f1=conv:oc=256,k=4,s=1,relu=1 f2=conv:oc=256,k=4,s=1,relu=1")
SMALL = ("id=small00000000000 parents= lr=0.003 momentum=0.9 batch_size=8 "
         "f0=conv:oc=8,k=3,s=1,relu=1 f1=pool:size=2,s=2 f2=conv:oc=16,k=3,s=2,relu=1 h0=dense:units=12")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def nn_ops():
    """Reference outputs for conv / pool / dense / xent / sgd on recipe inputs."""
    out = {}
    for ci, shape in enumerate(recipes.conv_shapes()):
        cin, cout, k, s, h = shape
        for dt in recipes.conv_dtypes(ci):
            tag = f"conv{ci}_{np.dtype(dt).name}"
            x, w, b, gy = recipes.conv_inputs(ci, shape, dt)
            layer = rnn.Conv2d(cin, cout, k, s, dtype=dt)
            layer.params["w"], layer.params["b"] = w, b
            y = layer.forward(x)
            gx = layer.backward(gy)
            out[tag + "_y"], out[tag + "_gx"] = y, gx
            out[tag + "_gw"], out[tag + "_gb"] = layer.grads["w"], layer.grads["b"]
    for size in (2, 3):
        for stride in (1, 2, 3):
            for variant in ("rand", "ties", "const"):
                tag = f"pool{size}{stride}_{variant}"
                x, gy = recipes.pool_input(size, stride, variant)
                layer = rnn.MaxPool(size, stride)
                out[tag + "_y"] = layer.forward(x)
                out[tag + "_arg"] = layer.argmax_indices
                out[tag + "_gx"] = layer.backward(gy)
    for di in range(len(recipes.DENSE_SHAPES)):
        x, w, b, gy = recipes.dense_inputs(di)
        layer = rnn.Dense(w.shape[1], w.shape[0])
        layer.params["w"], layer.params["b"] = w, b
        out[f"dense{di}_y"] = layer.forward(x)
        out[f"dense{di}_gx"] = layer.backward(gy)
        out[f"dense{di}_gw"], out[f"dense{di}_gb"] = layer.grads["w"], layer.grads["b"]
    r = np.random.default_rng(77)
    logits = (r.standard_normal((64, 2)) * 3).astype(np.float32)
    labels = r.integers(0, 2, 64)
    loss, grad = rnn.softmax_cross_entropy(logits, labels)
    out.update(xent_logits=logits, xent_labels=labels, xent_loss=np.array(loss), xent_grad=grad)
    # sgd: two momentum steps
    d = rnn.Dense(7, 3, rng=np.random.default_rng(3))
    net = rnn.Network([d], class_count=3)
    g1 = np.random.default_rng(4).standard_normal((3, 7)).astype(np.float32)
    g2 = np.random.default_rng(5).standard_normal((3, 7)).astype(np.float32)
    out["sgd_w0"] = d.params["w"].copy()
    d.grads = {"w": g1, "b": np.ones(3, np.float32)}
    rnn.sgd_step(net, 0.1, 0.9)
    d.grads = {"w": g2, "b": -np.ones(3, np.float32)}
    rnn.sgd_step(net, 0.1, 0.9)
    out.update(sgd_g1=g1, sgd_g2=g2, sgd_w2=d.params["w"], sgd_v2=d._vel["w"], sgd_b2=d.params["b"])
    np.savez_compressed(os.path.join(OUT, "nn_ops.npz"), **out)


def train_steps():
    out = {}
    medium = FIXED.replace("h0=dense:units=64", "h0=dense:units=8")
    for gi, (text, shape, n) in enumerate([(SMALL, (3, 24, 24), 8), (medium, (3, 60, 60), 4)]):
        g = rgen.parse_genome(text)
        net = rgen.instantiate(g, shape, seed=5)
        r = np.random.default_rng(9)
        x = (r.integers(0, 256, size=(n, *shape)).astype(np.float32) / np.float32(255.0))
        y = r.integers(0, 2, n)
        y[:2] = [0, 1]
        out[f"g{gi}_x"], out[f"g{gi}_y"] = x, y
        out[f"g{gi}_genome"] = np.array(text)
        logits = net.forward(x)
        out[f"g{gi}_logits"] = logits
        loss = rnn.train_batch(net, x, y, g.learn.lr, g.learn.momentum)
        out[f"g{gi}_loss"] = np.array(loss)
        for li, name, arr in net.parameters():
            out[f"g{gi}_p{li}_{name}"] = arr
            out[f"g{gi}_v{li}_{name}"] = net.layers[li]._vel[name]
            out[f"g{gi}_g{li}_{name}"] = net.layers[li].grads[name]
        traj = [loss]
        for step in range(9):
            traj.append(rnn.train_batch(net, x, y, g.learn.lr, g.learn.momentum))
        out[f"g{gi}_traj"] = np.array(traj)
    np.savez_compressed(os.path.join(OUT, "train_steps.npz"), **out)


def _fake_record(genome):
    """Deterministic record for GA replay: fitness from the genome id."""
    f = (int(genome.id[:6], 16) % 1000) / 1000.0
    flops = sum(getattr(g, "out_channels", 1) for g in genome.feature_layers)
    ok = int(genome.id[6], 16) != 0
    return rev.EvalRecord(genome_id=genome.id, ok=ok, val_f1=f, flops_inference=flops,
                          fitness=f if ok else rfit.FAILED_FITNESS)


def ga_replays():
    runs = []
    for seed in range(10):
        for mode in ("serial", "async4"):
            space = rgen.SearchSpace()
            settings = revo.EvolutionSettings(capacity=8, elite_count=2, max_evaluations=40)
            m = revo.Master(space, rfit.ObjectiveConfig("flop_proxy", -0.2, 1.0, 100.0), settings, seed=seed)
            sched_rng = np.random.default_rng(1000 + seed)
            events, issued, inflight = [], [], []
            while True:
                can_issue = not m.stop_reached()
                if mode == "serial":
                    if not can_issue:
                        break
                    gnm = m.issue("w0")
                    issued.append(rgen.format_genome(gnm))
                    events.append(["issue"])
                    m.collect(_fake_record(gnm))
                    events.append(["collect", 0])
                    continue
                if can_issue and len(inflight) < 4:
                    gnm = m.issue("w")
                    issued.append(rgen.format_genome(gnm))
                    inflight.append(gnm)
                    events.append(["issue"])
                    continue
                if not inflight:
                    break
                k = int(sched_rng.integers(0, len(inflight)))
                gnm = inflight.pop(k)
                m.collect(_fake_record(gnm))
                events.append(["collect", k])
            best = m.best.record.genome_id if m.best else None
            pop = [mb.genome.id for mb in m.population.members]
            runs.append({"seed": seed, "mode": mode, "events": events, "issued": issued,
                         "best": best, "population": pop, "rng_state": str(m.rng.bit_generator.state)})
    return runs


def genome_ops():
    out = {"random": [], "mutate": [], "crossover": []}
    space = rgen.SearchSpace()
    prior = rgen.ThroughputPrior(out_channels={256: 0.5, 64: 0.5}, kernel={4: 0.7, 3: 0.3}, stride={1: 1.0}, beta=0.5)
    rng = np.random.default_rng(42)
    gs = []
    for i in range(400):
        g = rgen.random_genome(rng, space, prior if i % 3 == 0 else None)
        gs.append(g)
        out["random"].append(rgen.format_genome(g))
    for i in range(300):
        g = rgen.mutate(gs[i], rng, rgen.MutationRates(), space, prior if i % 2 else None)
        out["mutate"].append(rgen.format_genome(g))
    for i in range(300):
        g = rgen.crossover(gs[i], gs[i + 1], rng, space.input_shape)
        out["crossover"].append(rgen.format_genome(g))
    out["final_state"] = str(rng.bit_generator.state)
    return out


def accounting():
    rows = []
    rng = np.random.default_rng(7)
    space = rgen.SearchSpace()
    for i in range(2000):
        g = rgen.random_genome(rng, space)
        t = rgen.validate_shapes(g, space.input_shape)
        head = t.flat_units * (t.head_units[0] if t.head_units else 2)
        if head > 3e6:  # skip giant heads: the reference would allocate them on the host
            rows.append([rgen.format_genome(g), None, None])
            continue
        net = rgen.instantiate(g, space.input_shape, seed=0)
        rows.append([rgen.format_genome(g), rev.count_flops_inference(net, space.input_shape), rev.count_params(net)])
    return rows


def main():
    nn_ops()
    train_steps()
    host = {"meta": {"numpy": np.__version__, "python": platform.python_version(),
                     "blas": "scipy-openblas 0.3.30 (numpy wheel)", "reference": REF}}
    d = rdata.generate_synthetic(*rdata.default_counts(4800), h=100, w=100, seed=0)
    sp = rdata.stratified_split(d, (5 / 6, 1 / 12, 1 / 12), seed=0)
    host["data"] = {"counts": list(rdata.default_counts(4800)), "pixels": sha(d.pixels), "labels": sha(d.labels),
                    "train": [len(sp.train), sha(sp.train.pixels), sha(sp.train.labels), int(sp.train.labels.sum())],
                    "val": [len(sp.val), sha(sp.val.pixels), sha(sp.val.labels), int(sp.val.labels.sum())],
                    "test": [len(sp.test), sha(sp.test.pixels), sha(sp.test.labels)]}
    small = rdata.generate_synthetic(5, 7, h=40, w=36, seed=3)
    host["data_small"] = {"pixels": sha(small.pixels), "labels": small.labels.tolist()}
    inst = {}
    for name, text in (("fixed", FIXED), ("vgg16style", VGG16STYLE), ("sweet", SWEET), ("small", SMALL)):
        g = rgen.parse_genome(text)
        shape = (3, 24, 24) if name == "small" else (3, 100, 100)
        net = rgen.instantiate(g, shape, seed=0)
        inst[name] = {"params": [[li, nm, list(a.shape), sha(a)] for li, nm, a in net.parameters()],
                      "flops": rev.count_flops_inference(net, shape), "count": rev.count_params(net)}
    host["instantiate"] = inst
    host["accounting"] = accounting()
    host["genome_ops"] = genome_ops()
    host["ga"] = ga_replays()
    # reduced-budget evaluate of FIXED on the C1 data (fp32, flop_proxy)
    obj = rfit.ObjectiveConfig("flop_proxy", -0.2, 1e8, 1e9)
    rec = rev.evaluate(rgen.parse_genome(FIXED), sp, rev.TrainBudget(epochs=1, max_batches_per_epoch=3), obj, seed=0)
    net, _ = rev.train_short(rgen.parse_genome(FIXED), sp.train, rev.TrainBudget(epochs=1, max_batches_per_epoch=3),
                             0)
    scores, preds = rev.predict_scores(net, sp.val)
    host["evaluate_fixed_3steps"] = {"record": rec.to_json_dict(), "scores": scores.tolist(),
                                     "preds": preds.tolist()}
    with open(os.path.join(OUT, "host.json"), "w") as fh:
        json.dump(host, fh)


if __name__ == "__main__":
    main()
