"""C4: whole-slide inference rate, FIXED vs VGG16STYLE.

    python tools/slide_bench.py [--patches 200000] [--batches 128,64] [--cpu-sample 256]

One JSON line per (genome, batch): patches/s device-resident (ce_predict on
the set uploaded once) and streamed (ce_predict_stream: u8 patches from
pinned host memory, H2D double-buffered against the forward), slide seconds
for 200,000 patches (metrics.py:77-81), and the oracle's CPU rate on a
bounded sample (predict_scores, extrapolated). The stream is the C1
synthetic set (generate_synthetic(default_counts(4800)), seed 0) replayed to
--patches. Weights: instantiate(seed=0) -- values do not affect speed.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402
from paper_1909_12291_b200 import native, slide  # noqa: E402
from paper_1909_12291_b200.candidate import DATASETS, predict_scores  # noqa: E402
from paper_1909_12291_b200.genes import FIXED, VGG16STYLE, parse_genome  # noqa: E402
from paper_1909_12291_b200.network import instantiate  # noqa: E402
from paper_1909_12291_b200.patches import PatchSet, default_counts, generate_synthetic  # noqa: E402
from paper_1909_12291_b200.scoring import slide_seconds  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--patches", type=int, default=200_000)
    ap.add_argument("--batches", default="128,64")
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--cpu-sample", type=int, default=256)
    args = ap.parse_args()
    base = generate_synthetic(*default_counts(4800), h=100, w=100, seed=0)
    reps = -(-args.patches // len(base.pixels))
    pix = np.tile(base.pixels, (reps, 1, 1, 1))[:args.patches]
    lab = np.tile(base.labels, reps)[:args.patches]
    stream = PatchSet(pix, lab, name="c4")
    pinned = slide.pinned_pixels(pix)
    for name, text in (("FIXED", FIXED), ("VGG16STYLE", VGG16STYLE)):
        g = parse_genome(text)
        for batch in [int(b) for b in args.batches.split(",")]:
            net = instantiate(g, (3, 100, 100), seed=0)
            net.to_device(0, args.precision, max_batch=batch)
            predict_scores(net, PatchSet(pix[:batch * 4], lab[:batch * 4]), batch_size=batch)  # warm-up
            slide.predict_stream(net, pinned[:batch * 4], batch)
            DATASETS.get(stream, 0)  # upload the resident copy outside the timed region
            clocks = ClockSampler(0)
            clocks.start()
            t0 = time.perf_counter()
            predict_scores(net, stream, batch_size=batch)
            resident_wall = time.perf_counter() - t0
            _, _, secs = slide.predict_stream(net, pinned, batch)
            ck = clocks.stop()
            # resident: ce_predict over the uploaded set, host wall around a synchronous call
            streamed = args.patches / secs
            line = {"workload": "C4 slide inference", "genome": name, "batch": batch, "precision": args.precision,
                    "patches": args.patches, "streamed_patches_per_s": streamed,
                    "streamed_slide_seconds": slide_seconds(streamed),
                    "resident_patches_per_s_wall": args.patches / resident_wall,
                    "h2d_bytes": int(pix.nbytes), "clocks": ck, "launches": native.launch_count()}
            if args.cpu_sample:
                from oracle.cnn_ref import OracleNet, predict_scores as cpu_predict
                o = OracleNet.from_network(net)
                sample = PatchSet(pix[:args.cpu_sample], lab[:args.cpu_sample])
                t0 = time.perf_counter()
                cpu_predict(o, sample, batch_size=batch)
                cpu_rate = args.cpu_sample / (time.perf_counter() - t0)
                line["cpu_oracle_patches_per_s"] = cpu_rate
                line["cpu_sample"] = f"{args.cpu_sample} patches, numpy oracle forward, {os.cpu_count()} host threads"
            print(json.dumps(line), flush=True)
            net.release()
            DATASETS.clear()


if __name__ == "__main__":
    main()
