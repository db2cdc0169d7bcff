#!/usr/bin/env python
"""bench.py — candidate CNNs evaluated per hour on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): the population of 16
bootstrap-random genomes issued by Master(SearchSpace(), capacity=16,
max_evaluations=16, seed=0); each candidate is trained for 2 epochs (batch =
its genome's batch size) on the 4,000 synthetic 100x100x3 TIL-style train
patches, scored on the 400 validation patches (F1 / AUC) and timed for
inference latency (1 warm-up + 5 device-timed forwards of a 64-patch batch),
i.e. one full `evaluate()` per candidate. A "step" is one evaluation of the
whole population. At N GPUs (torchrun, one process per GPU) the 16*N genomes
of Master(capacity=16N, seed=0) are statically sharded longest-estimated-first
(no data-path collective; weak scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0. `value` = candidates/h over the device-timed
steps with the train/val sets resident in HBM; `e2e` re-runs the same steps
through the public API with the data sets re-uploaded from pinned host memory
every step. `roofline` comes from a profiling pass over the same population
(per-kernel CUDA events on the launching stream); `cpu_baseline` times the
numpy oracle port (oracle/cnn_ref.py) on a bounded sample on this host.
"""

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

POP_PER_GPU = 16
METRIC = "candidate_cnns_evaluated_per_hour"
UNIT = "candidates/h"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--slots", type=int, default=4, help="candidates packed per GPU (streams)")
    ap.add_argument("--order", choices=["lpt", "two_ended", "fifo"], default="two_ended",
                    help="dispatch order of the pre-issued population")
    ap.add_argument("--big-slots", type=int, default=1,
                    help="two_ended: slots per GPU that take the longest remaining candidate")
    ap.add_argument("--precision", choices=["bf16", "fp32"], default="bf16")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return {k: float(p[k]) for k in FALLBACK_PEAKS}, "measured"
    except Exception:
        return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


def population(world):
    from paper_1909_12291_b200 import EvolutionSettings, Master, ObjectiveConfig, SearchSpace
    m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0),
               EvolutionSettings(capacity=POP_PER_GPU * world, max_evaluations=POP_PER_GPU * world), seed=0)
    return [m.issue("bench") for _ in range(POP_PER_GPU * world)]


def objective():
    from paper_1909_12291_b200 import ObjectiveConfig
    return ObjectiveConfig("measured_latency", -0.2, 1e-5, 1e-2)


# ------------------------------------------------------------------ CPU (oracle port)
def cpu_candidate_seconds(genome, splits, budget, sample_batch=8):
    """Extrapolated seconds for one candidate evaluate() on the CPU oracle:
    one timed train step and one timed forward at `sample_batch` patches,
    scaled to the candidate's full step count, val set and latency reps."""
    from oracle.cnn_ref import OracleNet
    from paper_1909_12291_b200.network import instantiate
    n = len(splits.train)
    bs = min(genome.learn.batch_size, n)
    sb = min(sample_batch, bs)
    net = instantiate(genome, splits.train.input_shape, seed=0)
    oracle = OracleNet.from_network(net)
    x = splits.train.pixels[:sb].astype(np.float32) / np.float32(255.0)
    y = splits.train.labels[:sb].astype(np.int64)
    t0 = time.perf_counter()
    oracle.train_batch(x, y, genome.learn.lr, genome.learn.momentum)
    t_step = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.forward(x, keep=False)
    t_fwd = time.perf_counter() - t0
    steps = budget.epochs * (n // bs)
    per_patch_fwd = t_fwd / sb
    return steps * t_step * (bs / sb) + per_patch_fwd * (len(splits.val) + 6 * 64)


def cpu_rate(genomes, splits, budget):
    secs = [cpu_candidate_seconds(g, splits, budget) for g in genomes]
    return len(genomes) / sum(secs) * 3600.0, sum(secs)


def run_reference(args, rank, out_fd):
    """--impl reference: the oracle port of the reference's CPU path, rank 0 only."""
    if rank != 0:
        return 0
    from paper_1909_12291_b200 import TrainBudget
    from paper_1909_12291_b200.patches import default_splits
    splits = default_splits()
    genomes = population(1)
    budget = TrainBudget(epochs=2)
    times, extrapolated = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _, secs = cpu_rate(genomes, splits, budget)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            extrapolated.append(secs)
    value = len(genomes) / statistics.fmean(extrapolated) * 3600.0
    cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.fmean(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": workload_config(args, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": "every step: all 16 genomes of the C2 population, 1 train step + 1 "
                                       "forward at batch 8 each on the numpy oracle (OpenBLAS, all host threads), "
                                       "extrapolated to each candidate's 2 epochs + val + latency"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line, out_fd)
    return 0


def workload_config(args, world):
    return {"workload": "C2 population evaluate(): 16 random genomes/GPU (Master seed 0), 2 epochs on 4000 "
                        "synthetic 100x100x3 patches, val F1/AUC on 400, device-timed latency (64-patch batch)",
            "population_per_gpu": POP_PER_GPU, "slots_per_gpu": args.slots, "precision": args.precision,
            "sharding": "static LPT over ranks" if world > 1 else "none",
            "l2": "flushed (256 MiB write) before every timed step"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        if os.environ.get("BENCH_NO_CLOCKS"):  # diagnostics only: the contract requires the sample
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ GPU arm
def emit(line, out_fd):
    """Write the single JSON result line to the real stdout (fd saved at start)."""
    os.write(out_fd, (json.dumps(line) + "\n").encode())


def main():
    args = parse_args()
    rank, world, local = dist_env()
    # Libraries (NCCL's version banner, ptxas, warnings) may print to stdout;
    # the contract is ONE JSON line there, so route fd 1 to stderr for the run.
    sys.stdout.flush()
    out_fd = os.dup(1)
    os.dup2(2, 1)
    if args.impl == "reference":
        return run_reference(args, rank, out_fd)
    import torch
    from paper_1909_12291_b200 import TrainBudget, native
    from paper_1909_12291_b200.candidate import DATASETS
    from paper_1909_12291_b200.patches import PatchSet, Splits, default_splits
    from paper_1909_12291_b200.population import estimate_cost, evaluate_population, shard_lpt

    device = local
    torch.cuda.set_device(device)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", device))

    def barrier():
        if dist is not None:
            dist.barrier()

    def allreduce(vals, op="max"):
        if dist is None:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return t.tolist()

    splits = default_splits()
    # pinned host copies: the e2e leg uploads these every step
    def pinned(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        return t.numpy()
    splits = Splits(*(PatchSet(pinned(p.pixels), pinned(p.labels), p.name) for p in
                      (splits.train, splits.val, splits.test)))
    budget = TrainBudget(epochs=2)
    obj = objective()
    genomes = population(world)
    n_train = len(splits.train)
    mine = shard_lpt(genomes, world, lambda g: estimate_cost(g, n_train, budget))[rank]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    last_trace = []
    last_window = [0.0]

    def step(profile=False):
        recs, report = evaluate_population(mine, splits, budget, obj, seed=0, devices=(device,),
                                           slots_per_gpu=1 if profile else args.slots, precision=args.precision,
                                           profile=profile, order=args.order, big_slots=args.big_slots)
        last_trace[:] = getattr(report, "trace", [])
        last_window[0] = getattr(report, "latency_window_s", 0.0)
        return recs

    def timed(n_steps, e2e=False):
        times, launches, recs = [], 0, None
        for _ in range(n_steps):
            flush.fill_(1)
            if e2e:
                DATASETS.clear()
            torch.cuda.synchronize()
            barrier()
            l0 = native.launch_count()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            recs = step()
            torch.cuda.synchronize()
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b))
            launches += native.launch_count() - l0
            barrier()
        return times, launches, recs

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(device)
    clocks.start()
    gc.collect()
    gc.disable()  # no collector pauses inside the timed steps (host objects are few and short-lived)
    try:
        times, launches, recs = timed(args.steps)
    finally:
        gc.enable()
    clock_info = clocks.stop()
    if os.environ.get("BENCH_TRACE"):  # per-candidate timeline of the last timed step (stderr)
        t0 = min(t[2] for t in last_trace)
        idx = {g.id: i for i, g in enumerate(mine)}
        for gid, wid, a, b in sorted(last_trace, key=lambda t: t[2]):
            print(f"trace {wid} g{idx.get(gid, -1):02d} start {1000 * (a - t0):8.1f} ms  dur {1000 * (b - a):8.1f} ms",
                  file=sys.stderr)
        print(f"trace latency window {1000 * last_window[0]:.1f} ms", file=sys.stderr)
    ms = allreduce([statistics.fmean(times)])[0]
    launches = int(allreduce([launches], "sum")[0])
    total_candidates = POP_PER_GPU * world
    value = total_candidates / (ms * 1e-3) * 3600.0
    ok = sum(1 for r in recs if r is not None and r.ok)
    train_imgs = sum(r.extras.get("train_steps", 0) * r.extras.get("train_batch", 0) for r in recs if r and r.ok)
    train_imgs = allreduce([train_imgs], "sum")[0]

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": workload_config(args, world),
            "train_img_per_s": train_imgs / (ms * 1e-3),
            "candidates_ok": int(allreduce([ok], "sum")[0]),
            "failures": [r.failure_reason[:120] for r in recs if r is not None and not r.ok],
            "gpu_launches": launches, "clocks": clock_info,
            "step_ms": [round(t, 1) for t in times]}

    if not args.no_e2e:
        e_times, _, _ = timed(max(1, args.steps), e2e=True)
        e_ms = allreduce([statistics.fmean(e_times)])[0]
        h2d = sum(p.pixels.nbytes + p.labels.nbytes for p in (splits.train, splits.val))
        from paper_1909_12291_b200.network import Network, build_layers
        d2h = 0
        for g in mine:
            shape = splits.train.input_shape
            n_params = Network(g, shape, build_layers(g, shape), []).param_count()
            steps = budget.epochs * (n_train // min(g.learn.batch_size, n_train))
            h2d += 4 * n_params + 4 * budget.epochs * n_train + 4 * 64 * int(np.prod(shape))
            d2h += 4 * steps + 16 * len(splits.val) + 8 * 5
        line["e2e"] = {"value": total_candidates / (e_ms * 1e-3) * 3600.0, "unit": UNIT,
                       "h2d_bytes_per_step": int(allreduce([h2d], "sum")[0]),
                       "d2h_bytes_per_step": int(allreduce([d2h], "sum")[0]),
                       "path": "evaluate_population() with train/val re-uploaded from pinned host memory"}

    if not args.no_profile:
        line["roofline"] = roofline(step(profile=True), ms)
        line["kernel_classes"] = line["roofline"].pop("classes")

    if not args.no_cpu_baseline and rank == 0 and world == 1:
        sample = mine
        t0 = time.perf_counter()
        rate, _ = cpu_rate(sample, splits, budget)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                                "sample": f"all {len(sample)} genomes of the population: 1 train step + 1 "
                                          "forward at batch 8 each on the numpy oracle (all host threads), "
                                          "extrapolated to each candidate's 2 epochs + val + latency; "
                                          f"{time.perf_counter() - t0:.1f} s of CPU work"}
    if rank == 0:
        emit(line, out_fd)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def roofline(recs, step_ms):
    """Dominant kernel class of the profiling pass vs the measured peaks."""
    peaks, src = load_peaks()
    tot = {}
    for r in recs:
        if r is None or not r.ok:
            continue
        for name, (n, ms, fl, by) in r.extras.get("kernel_profile", {}).items():
            t = tot.setdefault(name, [0, 0.0, 0.0, 0.0])
            t[0] += n
            t[1] += ms
            t[2] += fl
            t[3] += by
    if not tot:
        return {"bound": None, "achieved": None, "peak": None, "unit": None, "frac": None, "traffic": None,
                "classes": {}}
    name, (n, ms, fl, by) = max(tot.items(), key=lambda kv: kv[1][1])
    ai = fl / by if by else 0.0
    ridge = peaks["bf16_tflops_sustained"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    if fl > 0 and ai >= ridge:
        achieved, peak, unit, bound = fl / (ms * 1e-3) / 1e12, peaks["bf16_tflops_sustained"], "TFLOP/s", "tensor"
    else:
        achieved, peak, unit, bound = by / (ms * 1e-3) / 1e9, peaks["hbm_gbs"], "GB/s", "hbm"
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(name)
        except Exception:
            traffic = None
    classes = {k: {"launches": v[0], "ms": round(v[1], 3), "tflops": round(v[2] / (v[1] * 1e-3) / 1e12, 2) if v[1] else 0,
                   "gbs": round(v[3] / (v[1] * 1e-3) / 1e9, 1) if v[1] else 0} for k, v in tot.items()}
    return {"kernel": name, "bound": bound, "achieved": achieved, "peak": peak, "peak_source": src, "unit": unit,
            "frac": achieved / peak, "traffic": traffic, "algorithmic_flops_per_launch": fl / n,
            "algorithmic_bytes_per_launch": by / n, "avg_launch_ms": ms / n, "launches": n,
            "share_of_profiled_time": ms / sum(v[1] for v in tot.values()), "classes": classes}


if __name__ == "__main__":
    sys.exit(main())
