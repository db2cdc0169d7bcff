"""Conv pass microbenchmark through the kernel-level ABI (CUDA events on the
launching stream, L2 flushed between reps), with nvidia-smi clocks and
throttle reasons sampled during the timed reps (bench.ClockSampler).

    python tools/conv_bench.py [shape ...] [fwd|dgrad|wgrad] [vgg] [pool=k,s]
        shape = n,c,h,co,k,s
Default: the SWEET layer (256->256, k4, s1, 97x97 -> 94x94, B=64);
`vgg` adds every VGG16STYLE conv layer with C_out >= 128 at B=64.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import ClockSampler  # noqa: E402
from paper_1909_12291_b200 import native  # noqa: E402

SWEET = (64, 256, 97, 256, 4, 1)
# VGG16STYLE conv layers with C_out >= 128 at B=64: (n, c_in, h_in, c_out, k, s)
VGG = [(64, 64, 48, 128, 3, 1), (64, 128, 46, 128, 3, 1), (64, 128, 22, 256, 3, 1), (64, 256, 20, 256, 3, 1),
       (64, 256, 18, 256, 3, 1), (64, 256, 8, 256, 3, 1), (64, 256, 6, 256, 3, 1)]


def bench_shape(shape, reps=10, passes=("fwd", "dgrad", "wgrad")):
    n, c, h, co, k, s = shape
    oh = (h - k) // s + 1
    desc = native.conv_desc(n, c, h, h, co, k, s, "bf16")
    x = torch.randn(n, h, h, c, device="cuda").to(torch.bfloat16)
    w = (torch.randn(co, k, k, c, device="cuda") * 0.05).to(torch.bfloat16)
    b = torch.zeros(co, device="cuda")
    y = torch.empty(n, oh, oh, co, device="cuda", dtype=torch.bfloat16)
    dy = torch.randn(n, oh, oh, co, device="cuda").to(torch.bfloat16)
    dx = torch.empty_like(x)
    dw = torch.empty(co, k, k, c, device="cuda")
    db = torch.empty(co, device="cuda")
    wsb = native.conv_workspace_bytes(desc)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    flops = 2.0 * n * oh * oh * co * k * k * c
    calls = {
        "fwd": lambda: native.conv_fwd(desc, x.data_ptr(), w.data_ptr(), b.data_ptr(), 1, y.data_ptr(), st),
        "dgrad": lambda: native.conv_dgrad(desc, dy.data_ptr(), w.data_ptr(), None, dx.data_ptr(), ws.data_ptr(),
                                           wsb, st),
        "wgrad": lambda: native.conv_wgrad(desc, x.data_ptr(), dy.data_ptr(), dw.data_ptr(), db.data_ptr(),
                                           ws.data_ptr(), wsb, st),
    }
    out = {"shape": shape, "gflop": flops / 1e9}
    for p in passes:
        fn = calls[p]
        for _ in range(3):
            fn()
        ts = []
        for _ in range(reps):
            flush.fill_(1)
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            e.record()
            e.synchronize()
            ts.append(a.elapsed_time(e))
        ms = sorted(ts)[len(ts) // 2]
        out[p] = {"ms": round(ms, 4), "tflops": round(flops / (ms * 1e-3) / 1e12, 1)}
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    shapes = [tuple(int(v) for v in a.split(",")) for a in args if "," in a and "=" not in a]
    if "vgg" in args:
        shapes += VGG
    shapes = shapes or [SWEET]
    only = [a for a in args if a in ("fwd", "dgrad", "wgrad")]
    reps = int(next((a.split("=")[1] for a in args if a.startswith("reps=")), 10))
    # bring the SM clock up before the first timed shape (a cold GPU starts below max clocks)
    a_ = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    for _ in range(60):
        a_ @ a_
    torch.cuda.synchronize()
    del a_
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    rows = [bench_shape(sh, reps=reps, passes=tuple(only) or ("fwd", "dgrad", "wgrad")) for sh in shapes]
    info = clocks.stop()
    for r in rows:
        r["clocks"] = info
        print(json.dumps(r), flush=True)
