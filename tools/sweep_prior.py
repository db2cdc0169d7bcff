"""Run the conv sweep on the B200 and derive the GA throughput prior.

    python tools/sweep_prior.py [--out profiles/r01_sweep] [--k 40] [--precision bf16]

Writes <out>.csv (bench.py sweep CSV schema) and <out>_prior.json.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_12291_b200 import sweep  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="profiles/r01_sweep")
ap.add_argument("--k", type=int, default=40)
ap.add_argument("--precision", default="bf16")
args = ap.parse_args()
t0 = time.perf_counter()
rows, skipped = sweep.sweep_conv(sweep.SweepGrid(), reps=3, precision=args.precision)
sweep.write_sweep_csv(rows, args.out + ".csv")
prior = sweep.build_prior(rows, k=args.k)
top = sweep.top_k_by_throughput(rows, 5)
json.dump({"k": args.k, "precision": args.precision, "rows": len(rows), "skipped": len(skipped),
           "sweep_seconds": time.perf_counter() - t0,
           "prior": {hp: {str(v): p for v, p in getattr(prior, hp).items()} for hp in ("out_channels", "kernel", "stride")},
           "top5": [vars(r) for r in top]}, open(args.out + "_prior.json", "w"), indent=1)
print(open(args.out + "_prior.json").read())
