"""Pipeline timeline of one tcgen05 conv launch from the -DCE_TC_TRACE debug
library (build: python -m paper_1909_12291_b200.build --trace; run with
CE_LIB=trace). For CTA 0 it prints, per k-block, when the producer found the
stage free and issued its copies, when the MMA thread saw the stage full, and
per tile when the epilogue got and released the accumulator, as SM cycles
from the first event; then the average gaps:

    CE_LIB=trace python tools/tc_trace.py 64,128,46,128,3,1 [fwd|dgrad|wgrad] [pool=2,2]
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CE_LIB"] = "trace"
from paper_1909_12291_b200 import native  # noqa: E402

KIND = {1: "prod_wait", 2: "prod_issue", 3: "mma_full", 4: "mma_acc_free", 5: "epi_start", 6: "epi_done",
        7: "prod_loaded", 8: "mma_issued", 9: "epi_chunk", 10: "epi_converted", 11: "epi_stored"}


def read_trace(lib):
    buf = (C.c_ulonglong * (4 * 3 * 4096))()
    cnt = (C.c_uint * 12)()
    assert lib.ce_debug_trace(buf, cnt) == 0
    arr = np.frombuffer(buf, dtype=np.uint64).reshape(4, 3, 4096)
    n = np.frombuffer(cnt, dtype=np.uint32).reshape(4, 3)
    return arr, n


def decode(arr, n, cta):
    ev = []
    for role in range(3):
        for v in arr[cta, role, :min(int(n[cta, role]), 4096)]:
            v = int(v)
            ev.append((v & 0xFFFFFFFF, KIND[v >> 60], (v >> 46) & 0x3FFF, (v >> 32) & 0x3FFF))
    if not ev:
        return []
    t0 = min(e[0] for e in ev)
    return sorted(((e[0] - t0) & 0xFFFFFFFF, e[1], e[2], e[3]) for e in ev)


def main():
    args = sys.argv[1:]
    shape = tuple(int(v) for v in (args[0] if args else "64,128,46,128,3,1").split(","))
    p = next((a for a in args if a in ("fwd", "dgrad", "wgrad")), "fwd")
    n, c, h, co, k, s = shape
    oh = (h - k) // s + 1
    lib = native.load()
    desc = native.conv_desc(n, c, h, h, co, k, s, "bf16")
    x = torch.randn(n, h, h, c, device="cuda").to(torch.bfloat16)
    w = (torch.randn(co, k, k, c, device="cuda") * 0.05).to(torch.bfloat16)
    b = torch.zeros(co, device="cuda")
    y = torch.empty(n, oh, oh, co, device="cuda", dtype=torch.bfloat16)
    dy = torch.randn(n, oh, oh, co, device="cuda").to(torch.bfloat16)
    dx = torch.empty_like(x)
    dw = torch.empty(co, k, k, c, device="cuda")
    db = torch.empty(co, device="cuda")
    ws = torch.empty(native.conv_workspace_bytes(desc), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    pool = next((tuple(int(v) for v in a.split("=")[1].split(",")) for a in args if a.startswith("pool=")), None)
    if pool:
        ph = (oh - pool[0]) // pool[1] + 1
        yp = torch.empty(n, ph, ph, co, device="cuda", dtype=torch.bfloat16)
        ap = torch.empty(n, ph, ph, co, device="cuda", dtype=torch.uint8)

    def run():
        if p == "fwd" and pool:
            native.conv_fwd(desc, x.data_ptr(), w.data_ptr(), b.data_ptr(), 1, yp.data_ptr(), st, pool=pool,
                            arg=ap.data_ptr())
        elif p == "fwd":
            native.conv_fwd(desc, x.data_ptr(), w.data_ptr(), b.data_ptr(), 1, y.data_ptr(), st)
        elif p == "dgrad":
            native.conv_dgrad(desc, dy.data_ptr(), w.data_ptr(), 0, dx.data_ptr(), ws.data_ptr(), ws.numel(), st)
        else:
            native.conv_wgrad(desc, x.data_ptr(), dy.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(),
                              ws.numel(), st)
    if "fake" in args:  # producers skip the copies: the MMA / barrier rate alone
        assert lib.ce_debug_fake_load(1) == 0
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    read_trace(lib)  # reset
    run()
    torch.cuda.synchronize()
    arr, cnt = read_trace(lib)
    ev = decode(arr, cnt, 0)
    out = {"shape": shape, "pass": p, "events": len(ev), "counts": cnt.tolist()}
    issue = [e[0] for e in ev if e[1] == "prod_issue"]
    full = [e[0] for e in ev if e[1] == "mma_full"]
    waits = [(e[0], e[2], e[3]) for e in ev if e[1] == "prod_wait"]
    iss = {(e[2], e[3]): e[0] for e in ev if e[1] == "prod_issue"}
    ful = {(e[2], e[3]): e[0] for e in ev if e[1] == "mma_full"}
    lat = [ful[kk] - iss[kk] for kk in ful if kk in iss]
    stall = [iss[(t, kb)] - w0 for (w0, t, kb) in waits if (t, kb) in iss]
    tiles = sorted({e[2] for e in ev if e[1] == "epi_start"})
    es = {e[2]: e[0] for e in ev if e[1] == "epi_start"}
    ed = {e[2]: e[0] for e in ev if e[1] == "epi_done"}
    af = {e[2]: e[0] for e in ev if e[1] == "mma_acc_free"}
    out["span_cycles"] = ev[-1][0] if ev else 0
    out["kblocks"] = len(issue)
    out["cycles_per_kblock_mma"] = round((full[-1] - full[0]) / max(1, len(full) - 1), 1) if full else None
    out["load_latency_cycles_issue_to_full"] = {"median": float(np.median(lat)) if lat else None,
                                                "p90": float(np.percentile(lat, 90)) if lat else None}
    out["producer_stall_cycles_waiting_free_stage"] = {"median": float(np.median(stall)) if stall else None,
                                                       "total": int(sum(stall))}
    out["epilogue_cycles_per_tile"] = [ed[t] - es[t] for t in tiles if t in ed]
    out["mma_waits_for_acc_cycles"] = [af[t] - (ed.get(t, 0)) for t in tiles if t in af][:8]
    ld = {(e[2], e[3]): e[0] for e in ev if e[1] == "prod_loaded"}
    lc = [ld[kk] - iss[kk] for kk in ld if kk in iss]
    out["load_call_cycles"] = {"median": float(np.median(lc)) if lc else None,
                               "first": lc[:6]}
    mi = {(e[2], e[3]): e[0] for e in ev if e[1] == "mma_issued"}
    mc = [mi[kk] - ful[kk] for kk in mi if kk in ful]
    out["mma_issue_cycles"] = {"median": float(np.median(mc)) if mc else None, "first": mc[:6]}
    out["first_issue"] = issue[0] if issue else None
    out["first_full"] = full[0] if full else None
    print(json.dumps(out))
    if "dump" in args:
        for e in ev[:400]:
            print(e)


if __name__ == "__main__":
    main()
