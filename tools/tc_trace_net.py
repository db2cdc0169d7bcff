"""Pipeline timeline of the LAST tcgen05 launch of an inference pass over a
genome (debug build, CE_LIB=trace): with a one-conv genome the last tcgen05
launch is that conv's forward, which reaches the paths the kernel ABI does not
(the implicit packed first layer, fused pools):

    CE_LIB=trace python tools/tc_trace_net.py "f0=conv:oc=32,k=4,s=2,relu=1" [batch]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CE_LIB"] = "trace"
from paper_1909_12291_b200 import native, parse_genome  # noqa: E402
from paper_1909_12291_b200.candidate import predict_scores  # noqa: E402
from paper_1909_12291_b200.network import instantiate  # noqa: E402
from paper_1909_12291_b200.patches import PatchSet  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import tc_trace  # noqa: E402


def main():
    feats = sys.argv[1]
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    g = parse_genome(f"id=trace0000000000 parents= lr=0.001 momentum=0.9 batch_size={batch} {feats}")
    net = instantiate(g, (3, 100, 100), seed=0)
    net.to_device(0, "bf16", max_batch=batch)
    rng = np.random.default_rng(0)
    ps = PatchSet(rng.integers(0, 256, (batch, 3, 100, 100), dtype=np.uint8),
                  rng.integers(0, 2, batch).astype(np.uint8), name="trace")
    lib = native.load()
    predict_scores(net, ps, batch_size=batch)  # warm-up
    tc_trace.read_trace(lib)
    predict_scores(net, ps, batch_size=batch)
    arr, cnt = tc_trace.read_trace(lib)
    ev = tc_trace.decode(arr, cnt, 0)
    full = [e[0] for e in ev if e[1] == "mma_full"]
    iss = {(e[2], e[3]): e[0] for e in ev if e[1] == "prod_issue"}
    ld = {(e[2], e[3]): e[0] for e in ev if e[1] == "prod_loaded"}
    mi = {(e[2], e[3]): e[0] for e in ev if e[1] == "mma_issued"}
    ful = {(e[2], e[3]): e[0] for e in ev if e[1] == "mma_full"}
    es = {e[2]: e[0] for e in ev if e[1] == "epi_start"}
    ed = {e[2]: e[0] for e in ev if e[1] == "epi_done"}
    out = {"genome": feats, "batch": batch, "events": len(ev), "span_cycles": ev[-1][0] if ev else 0,
           "stages": len(full),
           "cycles_per_stage": round((full[-1] - full[0]) / max(1, len(full) - 1), 1) if full else None,
           "load_call_cycles": float(np.median([ld[k] - iss[k] for k in ld if k in iss])) if ld else None,
           "mma_issue_cycles": float(np.median([mi[k] - ful[k] for k in mi if k in ful])) if mi else None,
           "epilogue_cycles_per_tile": [ed[t] - es[t] for t in sorted(es) if t in ed][:6],
           "tiles": len(es)}
    print(json.dumps(out))
    if "dump" in sys.argv:
        for e in ev[:200]:
            print(e)


if __name__ == "__main__":
    main()
