"""Worker process of ProcessGpuPool: `slots` socket workers on one GPU.

    python -m paper_1909_12291_b200.gpu_worker --port P --device D --slots K --config JSON

config keys (all optional): budget {epochs, max_batches_per_epoch},
objective {kind, alpha, lo, hi}, seed, precision, data {total, seed}. Worker
ids are g{D}s{k} like the in-process GpuPool. The process owns its CUDA
context, so a sticky device fault ends this process only; the master reissues
its in-flight candidates (scheduler.SocketPool)."""

import argparse
import json
import os
import sys
import threading

from .candidate import TrainBudget, evaluate
from .patches import default_splits
from .scheduler import run_socket_worker
from .scoring import ObjectiveConfig


def make_evaluate(config, device):
    data = config.get("data", {})
    splits = default_splits(data.get("total", 4800), data.get("seed", 0))
    budget = TrainBudget(**config.get("budget", {}))
    objective = ObjectiveConfig(**config.get("objective", {}))
    seed = int(config.get("seed", 0))
    precision = config.get("precision", "bf16")

    def evaluate_fn(genome, worker_id):
        return evaluate(genome, splits, budget, objective, seed, worker_id=worker_id, precision=precision,
                        device=device)
    return evaluate_fn


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--host", default="127.0.0.1")
    ap.add_argument("--port", type=int, required=True)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--slots", type=int, default=1)
    ap.add_argument("--config", default="{}")
    args = ap.parse_args(argv)
    fn = make_evaluate(json.loads(args.config), args.device)

    def on_sticky(err):  # the context is poisoned: end the process, the master reissues its work
        sys.stderr.write(f"gpu_worker device {args.device}: sticky CUDA fault, exiting: {err}\n")
        sys.stderr.flush()
        os._exit(3)

    threads = [threading.Thread(target=run_socket_worker,
                                args=(args.host, args.port, f"g{args.device}s{k}", fn, on_sticky))
               for k in range(args.slots)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()


if __name__ == "__main__":
    main()
