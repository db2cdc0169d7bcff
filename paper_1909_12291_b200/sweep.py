"""Conv throughput sweep -> GA throughput prior (convevo/bench.py:29-165), plus
the epoch-timing bimodality detector (bench.py:168-238).

sweep_conv times forward + backward (wgrad, dgrad) of single conv layers over
a hyper-parameter grid -- here on the B200 through the kernel-level C ABI
(ce_conv_fwd / ce_conv_wgrad / ce_conv_dgrad), device-timed with CUDA events
on the launching stream -- and build_prior turns the top-k rows by
throughput into the ThroughputPrior that biases random_genome's conv choices
(genome.py:122-132, Fig. 2). Re-deriving the prior from the B200
kernels changes what the GA samples toward shapes this hardware runs fast.

Columns keep the reference's convention (bench.py:115-116):
flops_per_layer = forward FLOPs of one patch, flops_per_s = flops_per_layer *
batch / median(fwd+bwd seconds). The ranking that build_prior uses is what
matters; the host functions (CSV, top-k, prior, timing_distribution) are
restated bit-for-bit and pinned to reference outputs (tests/golden/sweep.json).
"""

import csv
from dataclasses import dataclass

import numpy as np

from .genes import ThroughputPrior

__all__ = ["SweepGrid", "SweepRow", "SWEEP_CSV_FIELDS", "conv_layer_flops", "sweep_conv", "write_sweep_csv",
           "read_sweep_csv", "top_k_by_throughput", "build_prior", "TimingSummary", "timing_distribution",
           "write_histogram_csv"]


@dataclass
class SweepGrid:
    in_channels: tuple = (3, 8, 16, 32)
    out_channels: tuple = (8, 16, 32, 64, 128)
    kernels: tuple = (1, 2, 3, 4, 5, 7)
    strides: tuple = (1, 2, 3)
    batch_sizes: tuple = (8, 16)
    height: int = 24
    width: int = 24

    def configs(self):
        for cin in self.in_channels:
            for cout in self.out_channels:
                for k in self.kernels:
                    for s in self.strides:
                        for b in self.batch_sizes:
                            yield {"in_channels": cin, "out_channels": cout, "kernel": k, "stride": s,
                                   "batch_size": b}

    def size(self):
        return (len(self.in_channels) * len(self.out_channels) * len(self.kernels) * len(self.strides)
                * len(self.batch_sizes))


@dataclass
class SweepRow:
    in_channels: int
    out_channels: int
    kernel: int
    stride: int
    batch_size: int
    height: int
    width: int
    median_forward_backward_s: float
    flops_per_layer: int
    flops_per_s: float


SWEEP_CSV_FIELDS = ["in_channels", "out_channels", "kernel", "stride", "batch_size", "height", "width",
                    "median_forward_backward_s", "flops_per_layer", "flops_per_s"]


def conv_layer_flops(cin, cout, kernel, stride, height, width):
    oh = (height - kernel) // stride + 1
    ow = (width - kernel) // stride + 1
    return 2 * kernel * kernel * cin * cout * oh * ow


def _pad8(v):
    return (v + 7) // 8 * 8


class _ConvPass:
    """Device buffers of one sweep config; run() enqueues fwd + wgrad + dgrad."""

    def __init__(self, cfg, h, w, precision, rng):
        import torch
        from . import native
        self.native = native
        n, cin, cout, k, s = cfg["batch_size"], cfg["in_channels"], cfg["out_channels"], cfg["kernel"], cfg["stride"]
        cs, os_ = _pad8(cin), _pad8(cout)
        oh, ow = (h - k) // s + 1, (w - k) // s + 1
        dt = torch.bfloat16 if precision == "bf16" else torch.float32
        dev = torch.device("cuda", torch.cuda.current_device())
        x = torch.zeros(n, h, w, cs, dtype=dt, device=dev)
        x[..., :cin] = torch.from_numpy(rng.random((n, h, w, cin), dtype=np.float32)).to(dev, dt)
        lim = np.sqrt(6.0 / (cin * k * k))
        wt = torch.zeros(os_, k, k, cs, dtype=dt, device=dev)
        wt[:cout, ..., :cin] = torch.from_numpy(
            rng.uniform(-lim, lim, size=(cout, k, k, cin)).astype(np.float32)).to(dev, dt)
        self.t = dict(x=x, w=wt, b=torch.zeros(os_, device=dev), y=torch.empty(n, oh, ow, os_, dtype=dt, device=dev),
                      dy=torch.ones(n, oh, ow, os_, dtype=dt, device=dev),
                      dx=torch.empty(n, h, w, cs, dtype=dt, device=dev),
                      dw=torch.empty(os_, k, k, cs, device=dev), db=torch.empty(os_, device=dev))
        self.desc = native.conv_desc(n, cs, h, w, os_, k, s, precision)
        self.ws = torch.empty(max(native.conv_workspace_bytes(self.desc), 256), dtype=torch.uint8, device=dev)
        self.stream = torch.cuda.current_stream().cuda_stream

    def run(self):
        t, nat, d, st = self.t, self.native, self.desc, self.stream
        nat.conv_fwd(d, t["x"].data_ptr(), t["w"].data_ptr(), t["b"].data_ptr(), 0, t["y"].data_ptr(), st)
        nat.conv_wgrad(d, t["x"].data_ptr(), t["dy"].data_ptr(), t["dw"].data_ptr(), t["db"].data_ptr(),
                       self.ws.data_ptr(), self.ws.numel(), st)
        nat.conv_dgrad(d, t["dy"].data_ptr(), t["w"].data_ptr(), None, t["dx"].data_ptr(), self.ws.data_ptr(),
                       self.ws.numel(), st)


def sweep_conv(grid, reps=3, seed=0, log=None, precision="bf16", inner=10):
    """Time every grid config on the current CUDA device; returns (rows, skipped).

    Configs whose kernel exceeds the input are skipped with a reason
    (bench.py:80-120). Each rep is the mean of `inner` back-to-back
    fwd+bwd passes between CUDA events (one pass of a 24x24 layer is a few
    microseconds), after one untimed warm-up pass; the row holds the median."""
    import torch
    if reps < 3:
        raise ValueError(f"need reps >= 3, got {reps}")
    rng = np.random.default_rng(seed)
    rows, skipped = [], []
    for cfg in grid.configs():
        k = cfg["kernel"]
        if k > grid.height or k > grid.width:
            reason = f"kernel {k} exceeds input {grid.height}x{grid.width}"
            skipped.append((cfg, reason))
            if log:
                log(f"skip {cfg}: {reason}")
            continue
        p = _ConvPass(cfg, grid.height, grid.width, precision, rng)
        p.run()
        times = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for _ in range(inner):
                p.run()
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b) * 1e-3 / inner)
        median = float(np.median(times))
        flops = conv_layer_flops(cfg["in_channels"], cfg["out_channels"], k, cfg["stride"], grid.height, grid.width)
        rows.append(SweepRow(in_channels=cfg["in_channels"], out_channels=cfg["out_channels"], kernel=k,
                             stride=cfg["stride"], batch_size=cfg["batch_size"], height=grid.height,
                             width=grid.width, median_forward_backward_s=median, flops_per_layer=flops,
                             flops_per_s=flops * cfg["batch_size"] / median))
    return rows, skipped


def write_sweep_csv(rows, path):
    with open(path, "w", newline="") as fh:
        writer = csv.DictWriter(fh, fieldnames=SWEEP_CSV_FIELDS)
        writer.writeheader()
        for r in rows:
            writer.writerow({f: getattr(r, f) for f in SWEEP_CSV_FIELDS})


def read_sweep_csv(path):
    rows = []
    with open(path, newline="") as fh:
        for rec in csv.DictReader(fh):
            rows.append(SweepRow(in_channels=int(rec["in_channels"]), out_channels=int(rec["out_channels"]),
                                 kernel=int(rec["kernel"]), stride=int(rec["stride"]),
                                 batch_size=int(rec["batch_size"]), height=int(rec["height"]),
                                 width=int(rec["width"]),
                                 median_forward_backward_s=float(rec["median_forward_backward_s"]),
                                 flops_per_layer=int(rec["flops_per_layer"]), flops_per_s=float(rec["flops_per_s"])))
    return rows


def top_k_by_throughput(rows, k):
    if k > len(rows):
        raise ValueError(f"k={k} exceeds {len(rows)} rows")
    return sorted(rows, key=lambda r: -r.flops_per_s)[:k]


def build_prior(rows, k, beta=0.5):
    """Add-one-smoothed frequency of each conv hyper-parameter value among the
    top-k rows by throughput; support = every value seen in `rows` (bench.py:147-165)."""
    top = top_k_by_throughput(rows, k)
    prior = {}
    for hp in ("out_channels", "kernel", "stride"):
        support = sorted({getattr(r, hp) for r in rows})
        counts = {v: 1 for v in support}
        for r in top:
            counts[getattr(r, hp)] += 1
        total = sum(counts.values())
        prior[hp] = {v: c / total for v, c in counts.items()}
    return ThroughputPrior(out_channels=prior["out_channels"], kernel=prior["kernel"], stride=prior["stride"],
                           beta=beta)


# ------------------------------------------------------------------ timing distribution
@dataclass
class TimingSummary:
    bin_edges: np.ndarray
    counts: np.ndarray
    modes: int
    mode_centers: tuple
    separation_stat: float


def _two_means_1d(values):
    """SSE-optimal split of sorted values into two clusters (prefix-sum scan)."""
    x = np.sort(values)
    n = len(x)
    csum, csq = np.cumsum(x), np.cumsum(x * x)
    best = (np.inf, 1)
    for t in range(1, n):
        sa, qa = csum[t - 1], csq[t - 1]
        sb, qb = csum[-1] - sa, csq[-1] - qa
        sse = (qa - sa * sa / t) + (qb - sb * sb / (n - t))
        if sse < best[0]:
            best = (sse, t)
    a, b = x[:best[1]], x[best[1]:]
    return float(a.mean()), float(b.mean()), float(a.std()), float(b.std())


def timing_distribution(samples, bins=30):
    """Histogram + two-cluster test: 2 modes when |c2 - c1| / (s1 + s2) > 2 (bench.py:196-229)."""
    values = np.asarray([getattr(s, "epoch_time_s", s) for s in samples], dtype=np.float64)
    if len(values) < 30:
        raise ValueError(f"need >= 30 samples, got {len(values)}")
    counts, edges = np.histogram(values, bins=bins)
    if np.ptp(values) == 0.0:
        return TimingSummary(edges, counts, 1, (float(values[0]),), 0.0)
    c1, c2, s1, s2 = _two_means_1d(values)
    spread = s1 + s2
    stat = float("inf") if spread == 0.0 else (c2 - c1) / spread
    if stat > 2.0:
        return TimingSummary(edges, counts, 2, (c1, c2), stat)
    return TimingSummary(edges, counts, 1, (float(values.mean()),), stat)


def write_histogram_csv(summary, path):
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(["bin_lo", "bin_hi", "count"])
        for lo, hi, c in zip(summary.bin_edges[:-1], summary.bin_edges[1:], summary.counts):
            writer.writerow([lo, hi, int(c)])
