#!/usr/bin/env python
"""bench.py — candidate CNNs evaluated per hour on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): the population of 16
bootstrap-random genomes issued by Master(SearchSpace(), capacity=16,
max_evaluations=16, seed=0); each candidate is trained for 2 epochs (batch =
its genome's batch size) on the 4,000 synthetic 100x100x3 TIL-style train
patches, scored on the 400 validation patches (F1 / AUC) and timed for
inference latency (1 warm-up + 5 device-timed forwards of a 64-patch batch),
i.e. one full `evaluate()` per candidate. A "step" is one evaluation of the
whole population. At N GPUs (torchrun, one process per GPU) the step is N
copies of that generation (so the work per GPU is fixed and the per-N lines
compare: weak scaling), dealt to every (GPU, slot) worker from ONE shared
longest-first queue through TCPStore counters (work stealing; no NCCL, no
data-path collective). `--workload c5` runs the 512-genome C5 generation over
all GPUs instead (strong scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0. `value` = candidates/h over the device-timed
steps with the train/val sets resident in HBM; `e2e` re-runs the same steps
through the public API with the data sets re-uploaded from pinned host memory
every step. `roofline` comes from a profiling pass over the same population
(per-kernel CUDA events on the launching stream); `population_roofline` is
SURVEY §8(d)'s sum of per-launch max(F/P, B/BW) over the step time;
`cpu_baseline` times the numpy oracle port (oracle/cnn_ref.py) as the
reference deploys it: W = nproc single-threaded pool workers, a bounded
sample per genome (oracle/cpu_pool.py).
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
C5_POP = 512
METRIC = "candidate_cnns_evaluated_per_hour"
UNIT = "candidates/h"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c2", "c5"], default="c2",
                    help="c2: the 16-genome C2 generation per GPU (weak scaling); "
                         "c5: the 512-genome C5 generation over all GPUs (strong scaling)")
    ap.add_argument("--slots", type=int, default=4, help="candidates packed per GPU (streams)")
    ap.add_argument("--big-slots", type=int, default=1,
                    help="slots per GPU that take the longest remaining candidate (two-ended dispatch)")
    ap.add_argument("--precision", choices=["bf16", "fp32"], default="bf16")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--profile-only", action="store_true",
                    help="run only the per-kernel profiling pass (for an ncu capture of the same launch mix)")
    ap.add_argument("--profile-batches", type=int, default=None,
                    help="with --profile-only: batches per epoch (one epoch); the per-step launch mix is the same")
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


def population(n):
    """The first n bootstrap genomes of Master(seed=0)."""
    from paper_1909_12291_b200 import EvolutionSettings, Master, ObjectiveConfig, SearchSpace
    m = Master(SearchSpace(), ObjectiveConfig("flop_proxy", -0.2, 1.0, 2.0),
               EvolutionSettings(capacity=n, max_evaluations=n), seed=0)
    return [m.issue("bench") for _ in range(n)]


def workload_genomes(workload, world):
    """The generation one bench step evaluates, identical on every rank.

    c2: N copies of the 16-genome C2 generation (replica r > 0 renames the ids),
        so the work per GPU is the same at every N (weak scaling) and the
        per-N lines compare; the copies are dealt from one shared queue.
    c5: the 512-genome C5 generation, total work fixed (strong scaling)."""
    import dataclasses
    if workload == "c5":
        return population(C5_POP)
    base = population(POP_PER_GPU)
    return [g if r == 0 else dataclasses.replace(g, id=f"{g.id}-r{r}") for r in range(world) for g in base]


def objective():
    from paper_1909_12291_b200 import ObjectiveConfig
    return ObjectiveConfig("measured_latency", -0.2, 1e-5, 1e-2)


# ------------------------------------------------------------------ CPU (oracle pool)
def cpu_leg(genomes, samples):
    """The reference's CPU path on this host: W = nproc single-threaded oracle
    workers (oracle/cpu_pool.py); returns (rate per sample, wall per sample, info)."""
    from oracle.cpu_pool import CpuPool, host_info
    pool = CpuPool(genomes)
    try:
        rates, walls, last = [], [], None
        for _ in range(samples):
            wall, sample = pool.sample()
            rates.append(pool.rate(sample))
            walls.append(wall)
            last = sample
        batches = sorted({v[2] for v in last.values()})
    finally:
        pool.close()
    info = host_info()
    info["workers"] = pool.workers
    info["sample_batches"] = batches
    return rates, walls, info


def cpu_sample_text(info):
    return (f"every genome of the generation on a pool of {info['workers']} single-threaded oracle workers "
            "(OPENBLAS_NUM_THREADS=1, W = nproc, as convevo's WorkerPool): per genome one forward+backward on "
            f"a {min(info['sample_batches'])}-{max(info['sample_batches'])}-patch sample, the full momentum-SGD "
            "update and one inference forward; extrapolated to 2 epochs at the genome's batch + 400 val + 6x64 "
            "latency patches; LPT makespan over the workers")


def run_reference(args, rank, out_fd):
    """--impl reference: the oracle port of the reference's CPU path, rank 0 only."""
    if rank != 0:
        return 0
    genomes = population(POP_PER_GPU) if args.workload == "c2" else population(C5_POP)
    rates, walls, info = cpu_leg(genomes, args.warmup + args.steps)
    rates, walls = rates[args.warmup:], walls[args.warmup:]
    value = statistics.fmean(rates)
    cfg = workload_config(args, 1)
    cfg["precision"] = "f32"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.fmean(walls),
            "higher_is_better": True, "scaling": "weak" if args.workload == "c2" else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["workers"], "kind": "port",
                             "sample": cpu_sample_text(info), "host": info},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line, out_fd)
    return 0


def workload_config(args, world):
    if args.workload == "c5":
        text = (f"C5 generation evaluate(): the {C5_POP} bootstrap genomes of Master seed 0 over all GPUs, 2 epochs "
                "on 4000 synthetic 100x100x3 patches, val F1/AUC on 400, device-timed latency (64-patch batch)")
    else:
        text = ("C2 population evaluate(): 16 random genomes/GPU (Master seed 0), 2 epochs on 4000 synthetic "
                "100x100x3 patches, val F1/AUC on 400, device-timed latency (64-patch batch)")
    return {"workload": text, "population": POP_PER_GPU * world if args.workload == "c2" else C5_POP,
            "slots_per_gpu": args.slots, "precision": args.precision,
            "sharding": ("one shared longest-first queue over all ranks (TCPStore counters, work stealing)"
                         if world > 1 else "none"),
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


def transfer_bytes(recs, genomes_by_id, splits, budget, datasets_uploaded):
    """Host<->device bytes of one e2e step, counted from what is actually
    copied: the train/val sets (re-uploaded every e2e step), each training
    run's epoch permutations (int32) and loss trajectory, the val scores and
    preds, and the latency batch + timings. Weights are drawn on the device
    (PCG64) and never cross PCIe."""
    n_train, n_val = len(splits.train), len(splits.val)
    h2d = datasets_uploaded * sum(p.pixels.nbytes + p.labels.nbytes for p in (splits.train, splits.val))
    d2h = 0
    lat_batch = 4 * 64 * int(np.prod(splits.train.input_shape))
    for r in recs:
        if r is None:
            continue
        g = genomes_by_id[r.genome_id]
        steps = budget.epochs * (n_train // min(g.learn.batch_size, n_train))
        runs = 2 if "bf16_failure" in r.extras else 1
        h2d += runs * 4 * budget.epochs * n_train
        d2h += runs * 4 * steps
        if r.ok:
            d2h += 16 * n_val
            if r.latency is not None:
                h2d += lat_batch
                d2h += 8 * r.latency.reps
    return h2d, d2h


def main():
    args = parse_args()
    if os.environ.get("CE_HANG_DUMP"):  # diagnostics: every thread's stack after N seconds (stderr)
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["CE_HANG_DUMP"]), repeat=True)
    rank, world, local = dist_env()
    # Libraries (ptxas, warnings) may print to stdout; the contract is ONE JSON
    # line there, so route fd 1 to stderr for the run.
    sys.stdout.flush()
    out_fd = os.dup(1)
    os.dup2(2, 1)
    if args.impl == "reference":
        return run_reference(args, rank, out_fd)
    import torch
    from paper_1909_12291_b200 import TrainBudget, native
    from paper_1909_12291_b200.candidate import DATASETS
    from paper_1909_12291_b200.patches import PatchSet, Splits, default_splits
    from paper_1909_12291_b200.population import (LocalCounter, SharedQueueMaster, StoreCounter, estimate_cost,
                                                  evaluate_population)
    from paper_1909_12291_b200.scheduler import is_big_slot

    device = local
    torch.cuda.set_device(device)
    dist, store = None, None
    if world > 1:
        # host-side plumbing only (barriers, max-over-ranks timings, the shared
        # work counters); candidates are independent, so no NCCL and no
        # collective on the data path (north_star)
        import torch.distributed as dist
        dist.init_process_group("gloo")
        store = dist.distributed_c10d._get_default_store()

    def barrier():
        if dist is not None:
            dist.barrier()

    def allreduce(vals, op="max"):
        if dist is None:
            return vals
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return t.tolist()

    splits = default_splits()

    def pinned(a):  # pinned host copies: the e2e leg uploads these every step
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    splits = Splits(*(PatchSet(pinned(p.pixels), pinned(p.labels), p.name) for p in
                      (splits.train, splits.val, splits.test)))
    budget = TrainBudget(epochs=2)
    obj = objective()
    genomes = workload_genomes(args.workload, world)
    by_id = {g.id: g for g in genomes}
    n_train = len(splits.train)

    def cost(g):
        return estimate_cost(g, n_train, budget)
    peaks, peak_src = load_peaks()
    native.set_prof_peaks(peaks["bf16_tflops_sustained"] * 1e12, peaks["hbm_gbs"] * 1e9)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    generation = [0]
    last_report = [None]

    def step(profile=False, pbudget=None):
        if profile:  # serial per-kernel profiling pass over the base generation (same genomes every rank)
            base = genomes[:POP_PER_GPU] if args.workload == "c2" else genomes
            recs, _ = evaluate_population(base, splits, pbudget or budget, obj, seed=0, devices=(device,),
                                          slots_per_gpu=1,
                                          precision=args.precision, profile=True, order="lpt")
            return recs
        generation[0] += 1
        counter = StoreCounter(store, f"gen{generation[0]}") if store is not None else LocalCounter()
        master = SharedQueueMaster(genomes, counter, cost, big_worker=lambda wid: is_big_slot(wid, args.big_slots))
        recs, report = evaluate_population(None, splits, budget, obj, seed=0, devices=(device,),
                                           slots_per_gpu=args.slots, precision=args.precision, master=master)
        last_report[0] = report
        return recs

    if args.profile_only:  # one profiling pass; prints the bracket count per class (ncu traffic denominators)
        pb = TrainBudget(epochs=1, max_batches_per_epoch=args.profile_batches) if args.profile_batches else None
        recs = step(profile=True, pbudget=pb)
        torch.cuda.synchronize()
        counts = {}
        for r in recs:
            for name, vals in (r.extras.get("kernel_profile", {}) if r is not None and r.ok else {}).items():
                counts[name] = counts.get(name, 0) + int(vals[0])
        print(json.dumps({"profile_only": True, "class_launches": counts,
                          "ok": sum(1 for r in recs if r is not None and r.ok), "candidates": len(recs)}))
        return 0

    def timed(n_steps, e2e=False):
        times, launches, all_recs = [], 0, []
        h2d = d2h = 0
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
            times.append(allreduce([a.elapsed_time(b)])[0])  # the step ends when the slowest rank does
            launches += native.launch_count() - l0
            if e2e:
                hb, db = transfer_bytes(recs, by_id, splits, budget, 1)
                h2d, d2h = h2d + hb, d2h + db
            all_recs = recs
            barrier()
        return times, launches, all_recs, h2d / max(1, n_steps), d2h / max(1, n_steps)

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(device)
    clocks.start()
    gc.collect()
    gc.disable()  # no collector pauses inside the timed steps (host objects are few and short-lived)
    try:
        times, launches, recs, _, _ = timed(args.steps)
    finally:
        gc.enable()
    clock_info = clocks.stop()
    if os.environ.get("BENCH_TRACE") and last_report[0] is not None:  # timeline of the last timed step (stderr)
        rep = last_report[0]
        t0 = min(t[2] for t in rep.trace)
        for gid, wid, a, b in sorted(rep.trace, key=lambda t: t[2]):
            r = next((x for x in recs if x is not None and x.genome_id == gid), None)
            extra = "" if r is None else f" {'fp32-confirmed' if 'bf16_failure' in r.extras else ''}"
            print(f"trace r{rank} {wid} {gid[:16]} start {1e3 * (a - t0):8.1f} ms dur {1e3 * (b - a):8.1f} ms"
                  f"{extra}", file=sys.stderr)
        print(f"trace r{rank} latency window {1e3 * getattr(rep, 'latency_window_s', 0.0):.1f} ms", file=sys.stderr)
    ms = statistics.fmean(times)
    launches = int(allreduce([launches], "sum")[0])
    total_candidates = len(genomes)
    value = total_candidates / (ms * 1e-3) * 3600.0
    ok = sum(1 for r in recs if r is not None and r.ok)
    train_imgs = sum(r.extras.get("train_steps", 0) * r.extras.get("train_batch", 0) for r in recs if r and r.ok)
    n_done, ok, train_imgs = allreduce([len(recs), ok, train_imgs], "sum")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if args.workload == "c2" else "strong",
            "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": workload_config(args, world),
            "train_img_per_s": train_imgs / (ms * 1e-3),
            "candidates_ok": int(ok), "candidates_done": int(n_done),
            "candidates_this_rank": len(recs),
            "failures": [r.failure_reason[:120] for r in recs if r is not None and not r.ok],
            "fp32_confirmed": sum(1 for r in recs if r is not None and "bf16_failure" in r.extras),
            "gpu_launches": launches, "clocks": clock_info,
            "step_ms": [round(t, 1) for t in times]}

    if not args.no_e2e:
        e_times, _, _, h2d, d2h = timed(max(1, args.steps), e2e=True)
        h2d, d2h = allreduce([h2d, d2h], "sum")
        line["e2e"] = {"value": total_candidates / (statistics.fmean(e_times) * 1e-3) * 3600.0, "unit": UNIT,
                       "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                       "path": "evaluate_population() with train/val re-uploaded from pinned host memory every step"}

    if not args.no_profile:
        line["roofline"] = roofline(step(profile=True), ms, peaks, peak_src,
                                    POP_PER_GPU if args.workload == "c2" else total_candidates, total_candidates)
        line["kernel_classes"] = line["roofline"].pop("classes")
        line["population_roofline"] = line["roofline"].pop("population")

    if not args.no_cpu_baseline and rank == 0 and world == 1:
        t0 = time.perf_counter()
        rates, _, info = cpu_leg(genomes[:POP_PER_GPU] if args.workload == "c2" else genomes, 1)
        line["cpu_baseline"] = {"value": rates[0], "unit": UNIT, "cores": info["workers"], "kind": "port",
                                "sample": cpu_sample_text(info) + f"; {time.perf_counter() - t0:.1f} s on this host",
                                "host": info}
    if rank == 0:
        emit(line, out_fd)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def roofline(recs, step_ms, peaks, src, profiled, total):
    """Dominant kernel class of the profiling pass (per-launch CUDA events on the
    launching stream) against the measured peaks, plus the population roofline
    SURVEY §8(d) defines: the sum over launches of max(F/P, B/BW) (sustained
    bf16 peak, HBM copy bandwidth) divided by the measured step time."""
    tot = {}
    for r in recs:
        if r is None or not r.ok:
            continue
        for name, vals in r.extras.get("kernel_profile", {}).items():
            t = tot.setdefault(name, [0, 0.0, 0.0, 0.0, 0.0])
            for i, v in enumerate(vals):
                t[i] += v
    if not tot:
        return {"bound": None, "achieved": None, "peak": None, "unit": None, "frac": None, "traffic": None,
                "classes": {}, "population": None}
    name, (n, ms, fl, by, _) = max(tot.items(), key=lambda kv: kv[1][1])
    ai = fl / by if by else 0.0
    ridge = peaks["bf16_tflops_sustained"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    if fl > 0 and ai >= ridge:
        achieved, peak, unit, bound = fl / (ms * 1e-3) / 1e12, peaks["bf16_tflops_sustained"], "TFLOP/s", "tensor"
    else:
        achieved, peak, unit, bound = by / (ms * 1e-3) / 1e9, peaks["hbm_gbs"], "GB/s", "hbm"
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic_r02.json")
    if os.path.exists(tfile):
        try:
            with open(tfile) as fh:
                traffic = json.load(fh)["classes"].get(name, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    classes = {k: {"launches": v[0], "ms": round(v[1], 3),
                   "tflops": round(v[2] / (v[1] * 1e-3) / 1e12, 2) if v[1] else 0,
                   "gbs": round(v[3] / (v[1] * 1e-3) / 1e9, 1) if v[1] else 0,
                   "ideal_ms": round(v[4], 3)} for k, v in tot.items()}
    scale = total / profiled
    ideal = sum(v[4] for v in tot.values()) * scale
    prof_ms = sum(v[1] for v in tot.values())
    population = {"ideal_ms": ideal, "measured_ms": step_ms, "frac": ideal / step_ms,
                  "profiled_serial_ms": prof_ms * scale,
                  "rule": "sum over kernel launches of max(flops / sustained bf16 peak, algorithmic bytes / HBM "
                          "peak) from the profiling pass (1 slot, eager), scaled to the step's candidate count, "
                          "divided by ms_per_step"}
    return {"kernel": name, "bound": bound, "achieved": achieved, "peak": peak, "peak_source": src, "unit": unit,
            "frac": achieved / peak, "traffic": traffic, "algorithmic_flops_per_launch": fl / n,
            "algorithmic_bytes_per_launch": by / n, "avg_launch_ms": ms / n, "launches": n,
            "share_of_profiled_time": ms / prof_ms, "classes": classes, "population": population}


if __name__ == "__main__":
    sys.exit(main())
