"""Golden values for the sweep -> prior pipeline, produced by the REFERENCE
(convevo/bench.py build_prior / timing_distribution, genome.random_genome with
a prior). Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_sweep_golden.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("CONVEVO_SRC", "/root/reference/pkg/src"))
from convevo import bench as rb  # noqa: E402
from convevo import genome as rg  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def rows():
    """Deterministic synthetic sweep rows over the default grid (24x24)."""
    out = []
    grid = rb.SweepGrid()
    rng = np.random.default_rng(11)
    for cfg in grid.configs():
        if cfg["kernel"] > grid.height:
            continue
        fl = rb.conv_layer_flops(cfg["in_channels"], cfg["out_channels"], cfg["kernel"], cfg["stride"], 24, 24)
        t = 1e-5 + 1e-12 * fl * cfg["batch_size"] * (1.0 + rng.random())
        out.append(rb.SweepRow(in_channels=cfg["in_channels"], out_channels=cfg["out_channels"],
                               kernel=cfg["kernel"], stride=cfg["stride"], batch_size=cfg["batch_size"],
                               height=24, width=24, median_forward_backward_s=t, flops_per_layer=fl,
                               flops_per_s=fl * cfg["batch_size"] / t))
    return out


def main():
    rs = rows()
    prior = rb.build_prior(rs, k=40, beta=0.5)
    rng = np.random.default_rng(3)
    uni = list(rng.normal(1.0, 0.05, 60))
    bi = list(rng.normal(1.0, 0.02, 40)) + list(rng.normal(2.0, 0.02, 40))
    summ = {}
    for name, vals in (("unimodal", uni), ("bimodal", bi)):
        s = rb.timing_distribution(vals, bins=20)
        summ[name] = {"values": vals, "modes": s.modes, "centers": list(s.mode_centers),
                      "stat": s.separation_stat, "counts": [int(c) for c in s.counts],
                      "edges": list(map(float, s.bin_edges))}
    grng = np.random.default_rng(0)
    space = rg.SearchSpace()
    genomes = [rg.format_genome(rg.random_genome(grng, space, prior=prior)) for _ in range(50)]
    gold = {"rows": [[r.in_channels, r.out_channels, r.kernel, r.stride, r.batch_size, r.median_forward_backward_s,
                      r.flops_per_layer, r.flops_per_s] for r in rs],
            "prior": {hp: {str(k): v for k, v in getattr(prior, hp).items()}
                      for hp in ("out_channels", "kernel", "stride")},
            "timing": summ, "genomes_with_prior": genomes}
    with open(os.path.join(OUT, "sweep.json"), "w") as fh:
        json.dump(gold, fh)


if __name__ == "__main__":
    main()
