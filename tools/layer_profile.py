"""Per-(genome, layer, kernel class) profile of the C2 population: CUDA-event
time of every launch (eager, one slot) against its SURVEY §8(d) roofline time
max(F/P, B/BW) with the sustained bf16 peak and HBM copy bandwidth, sorted by
waste (measured - ideal). Shows which layer shapes the kernel work should go to.

    python tools/layer_profile.py [--precision bf16] [--max-batches N] [--top 40] [--out gpurun_out/layer_profile.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_1909_12291_b200 import TrainBudget, native  # noqa: E402
from paper_1909_12291_b200.candidate import evaluate  # noqa: E402
from paper_1909_12291_b200.genes import format_genome  # noqa: E402
from paper_1909_12291_b200.network import ConvLayer, DenseLayer, PoolLayer, instantiate  # noqa: E402
from paper_1909_12291_b200.patches import default_splits  # noqa: E402


def describe(layer, in_shape):
    if isinstance(layer, ConvLayer):
        return f"conv {layer.in_channels}->{layer.out_channels} k{layer.kernel}s{layer.stride} {in_shape[1]}->{layer.out_shape[1]}"
    if isinstance(layer, PoolLayer):
        return f"pool k{layer.size}s{layer.stride} {in_shape[1]}->{layer.out_shape[1]}"
    return f"dense {layer.in_units}->{layer.out_units}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--max-batches", type=int, default=None)
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--out", default="gpurun_out/layer_profile.json")
    ap.add_argument("--genomes", default="c2", help="c2 (the 16 C2 genomes) or a comma list of FIXED,VGG16STYLE,SWEET")
    a = ap.parse_args()
    peaks, _ = bench.load_peaks()
    native.set_prof_peaks(peaks["bf16_tflops_sustained"] * 1e12, peaks["hbm_gbs"] * 1e9)
    splits = default_splits()
    budget = TrainBudget(epochs=2, max_batches_per_epoch=a.max_batches)
    rows = []
    if a.genomes == "c2":
        genomes = bench.population(16)
    else:
        from paper_1909_12291_b200 import genes, parse_genome
        genomes = [parse_genome(getattr(genes, name)) for name in a.genomes.split(",")]
    for gi, g in enumerate(genomes):
        rec = evaluate(g, splits, budget, bench.objective(), seed=0, precision=a.precision, profile=True)
        net = instantiate(g, splits.train.input_shape, seed=0)
        shapes, shape = [], splits.train.input_shape
        for layer in net.layers:
            shapes.append(describe(layer, shape))
            shape = getattr(layer, "out_shape", shape)
        for key, (n, ms, fl, by, ideal) in rec.extras.get("layer_profile", {}).items():
            li, cls = key.split(":")
            li = int(li)
            rows.append({"genome": gi, "id": g.id, "layer": li, "desc": shapes[li] if li >= 0 else "gather/loss",
                         "class": cls, "launches": n, "ms": ms, "ideal_ms": ideal, "us_per_launch": 1e3 * ms / n,
                         "eff": ideal / ms if ms else 0.0, "tflops": fl / (ms * 1e-3) / 1e12 if ms else 0.0,
                         "gbs": by / (ms * 1e-3) / 1e9 if ms else 0.0,
                         "precision": rec.extras.get("precision"), "batch": g.learn.batch_size})
        print(f"{gi:2d} {g.id} ok={rec.ok} {rec.extras.get('precision')} {format_genome(g)[:150]}", flush=True)
    rows.sort(key=lambda r: -(r["ms"] - r["ideal_ms"]))
    tot = sum(r["ms"] for r in rows)
    ideal = sum(r["ideal_ms"] for r in rows)
    print(f"total {tot:.1f} ms, ideal {ideal:.1f} ms ({ideal / tot:.3f})")
    print(f"{'g':>2} {'layer':>5} {'class':10s} {'desc':34s} {'n':>5} {'ms':>8} {'ideal':>7} {'us/l':>7} {'eff':>5} "
          f"{'TF/s':>7} {'GB/s':>7}")
    for r in rows[:a.top]:
        print(f"{r['genome']:2d} {r['layer']:5d} {r['class']:10s} {r['desc']:34s} {r['launches']:5d} {r['ms']:8.2f} "
              f"{r['ideal_ms']:7.2f} {r['us_per_launch']:7.1f} {r['eff']:5.2f} {r['tflops']:7.1f} {r['gbs']:7.0f}")
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump({"total_ms": tot, "ideal_ms": ideal, "rows": rows}, fh)


if __name__ == "__main__":
    main()
