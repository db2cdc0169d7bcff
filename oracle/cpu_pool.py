"""CPU ORACLE POOL — TEST / BASELINE INFRASTRUCTURE ONLY.

Times the reference's CPU path the way the reference deploys it: a
WorkerPool of W = nproc workers (convevo/workers.py:151-205), each evaluating
whole candidates single-threaded (OPENBLAS_NUM_THREADS=1),
here as W processes running oracle/cnn_ref.py (the numpy restatement of
convevo/nn.py + evaluator.py pinned by tests/test_oracle_golden.py).

A bounded sample per genome and per bench step: forward + backward on a
sample batch sized so it takes about `budget_s` (the genome's own batch when
that fits), the real momentum-SGD update over every parameter, and an
inference forward of the sample batch. One training step at the genome's
batch is t_fwd_bwd * batch / sample + t_sgd (the tensor work scales with the
batch, the parameter update does not); the full-budget candidate time is
steps * t_step + t_fwd_per_patch * (400 val + 6 * 64 latency patches), and
the generation's makespan is the LPT schedule of those times over the W
workers (the reference pool pulls FIFO; LPT is the CPU's
best case). Only bench.py's cpu_baseline / --impl reference legs use this.
"""

import multiprocessing as mp
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MIN_SAMPLE = 8


def _worker(conn, genome_texts, budget_s, seed):
    sys.path.insert(0, ROOT)
    from oracle.cnn_ref import OracleNet, softmax_xent
    from paper_1909_12291_b200.genes import parse_genome
    from paper_1909_12291_b200.network import instantiate
    from paper_1909_12291_b200.patches import default_splits
    train = default_splits().train
    rng = np.random.default_rng(seed)
    nets = []
    for text in genome_texts:  # untimed set-up: host Kaiming draw, as instantiate() does once per candidate
        g = parse_genome(text)
        bs = min(g.learn.batch_size, len(train))
        idx = rng.permutation(len(train))[:bs]
        x = train.pixels[idx].astype(np.float32) / np.float32(255.0)
        y = train.labels[idx].astype(np.int64)
        net = OracleNet.from_network(instantiate(g, train.input_shape, seed=0))
        t0 = time.perf_counter()  # calibration: one sample's forward+backward
        _fwd_bwd(net, x[:1], y[:1], softmax_xent)
        t1 = time.perf_counter() - t0
        # at least 8 patches: tiny batches are dominated by per-call overheads and would overstate the CPU time
        sb = int(min(bs, max(MIN_SAMPLE, budget_s // max(t1, 1e-6))))
        nets.append((g, net, x, y, bs, sb))
    conn.send("ready")
    while True:
        msg = conn.recv()
        if msg is None:
            return
        out = {}
        for g, net, x, y, bs, sb in nets:
            t0 = time.perf_counter()
            _fwd_bwd(net, x[:sb], y[:sb], softmax_xent)
            t1 = time.perf_counter()
            net.step(g.learn.lr, g.learn.momentum)
            t2 = time.perf_counter()
            net.forward(x[:sb], keep=False)
            t3 = time.perf_counter()
            # forward/backward work scales with the batch, the momentum-SGD pass does not
            out[g.id] = ((t1 - t0) * bs / sb + (t2 - t1), (t3 - t2) / sb, sb)
        conn.send(out)


def _fwd_bwd(net, x, y, xent):
    loss, g = xent(net.forward(x), y)
    net.backward(g)
    return loss


def _lpt_makespan(times, workers):
    loads = np.zeros(workers)
    for t in sorted(times, reverse=True):
        loads[np.argmin(loads)] += t
    return float(loads.max())


class CpuPool:
    """W single-threaded oracle worker processes holding their genomes' nets."""

    def __init__(self, genomes, workers=None, n_train=4000, epochs=2, seed=0, budget_s=1.5):
        from paper_1909_12291_b200.genes import format_genome
        from paper_1909_12291_b200.population import estimate_cost
        self.workers = workers or os.cpu_count()
        self.genomes = list(genomes)
        self.n_train, self.epochs = n_train, epochs
        shards = [[] for _ in range(min(self.workers, len(self.genomes)))]
        loads = np.zeros(len(shards))
        for g in sorted(self.genomes, key=lambda g: -estimate_cost(g)):
            k = int(np.argmin(loads))
            shards[k].append(format_genome(g))
            loads[k] += estimate_cost(g) + 1e-3
        ctx = mp.get_context("spawn")
        saved = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
        os.environ.update(OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1")
        try:
            self.procs, self.conns = [], []
            for i, shard in enumerate(shards):
                a, b = ctx.Pipe()
                p = ctx.Process(target=_worker, args=(b, shard, budget_s, seed + i), daemon=True)
                p.start()
                self.procs.append(p)
                self.conns.append(a)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        for c in self.conns:
            assert c.recv() == "ready"

    def sample(self):
        """One bounded sample of every genome in parallel; returns (wall s, {id: (t_step, t_fwd)})."""
        t0 = time.perf_counter()
        for c in self.conns:
            c.send("go")
        out = {}
        for c in self.conns:
            out.update(c.recv())
        return time.perf_counter() - t0, out

    def candidate_seconds(self, sample):
        secs = []
        for g in self.genomes:
            t_step, t_fwd, _ = sample[g.id]
            bs = min(g.learn.batch_size, self.n_train)
            steps = self.epochs * (self.n_train // bs)
            secs.append(steps * t_step + t_fwd * (400 + 6 * 64))
        return secs

    def rate(self, sample):
        """Candidates/h of the generation on W workers (LPT makespan of the extrapolated times)."""
        secs = self.candidate_seconds(sample)
        return len(secs) / _lpt_makespan(secs, self.workers) * 3600.0

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except Exception:
                pass
        for p in self.procs:
            p.join(timeout=10)
            if p.is_alive():
                p.kill()


def host_info():
    model = platform.processor()
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = "unknown"
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name', '?')} {b.get('version', '?')}"
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "numpy": np.__version__, "blas": blas}
