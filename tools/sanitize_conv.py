"""One small launch of each tcgen05 conv pass (fwd, fwd+max-pool epilogue,
dgrad, wgrad) and of the dense tcgen05 passes through the kernel ABI, for
compute-sanitizer (racecheck / synccheck / memcheck on the mbarrier + TMEM
pipelines):

    compute-sanitizer --tool racecheck python tools/sanitize_conv.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_12291_b200 import native  # noqa: E402


def main():
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(0)
    # (n, c, h, co, k, s): TMA im2col path (C % 64 == 0), gather path, strided dgrad classes
    for (n, c, h, co, k, s) in [(2, 64, 12, 128, 3, 1), (2, 16, 13, 32, 4, 2)]:
        oh = (h - k) // s + 1
        desc = native.conv_desc(n, c, h, h, co, k, s, "bf16")
        x = torch.from_numpy(rng.standard_normal((n, h, h, c)).astype(np.float32)).cuda().to(torch.bfloat16)
        w = torch.from_numpy(rng.standard_normal((co, k, k, c)).astype(np.float32) * 0.1).cuda().to(torch.bfloat16)
        b = torch.zeros(co, device="cuda")
        y = torch.empty(n, oh, oh, co, device="cuda", dtype=torch.bfloat16)
        dy = torch.randn(n, oh, oh, co, device="cuda").to(torch.bfloat16)
        dx = torch.empty_like(x)
        dw = torch.empty(co, k, k, c, device="cuda")
        db = torch.empty(co, device="cuda")
        wsb = native.conv_workspace_bytes(desc)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        native.conv_fwd(desc, x.data_ptr(), w.data_ptr(), b.data_ptr(), 1, y.data_ptr(), st)
        ph = (oh - 2) // 2 + 1
        yp = torch.empty(n, ph, ph, co, device="cuda", dtype=torch.bfloat16)
        ap = torch.empty(n, ph, ph, co, device="cuda", dtype=torch.uint8)
        native.conv_fwd(desc, x.data_ptr(), w.data_ptr(), b.data_ptr(), 1, yp.data_ptr(), st, pool=(2, 2),
                        arg=ap.data_ptr())
        native.conv_dgrad(desc, dy.data_ptr(), w.data_ptr(), x.data_ptr(), dx.data_ptr(), ws.data_ptr(), wsb, st)
        native.conv_wgrad(desc, x.data_ptr(), dy.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(), wsb, st)
    # dense tcgen05 forward / backward with the fused SGD
    B, I, O = 64, 512, 96
    d = native.dense_desc(B, I, O, "bf16")
    xb = torch.randn(B, I, device="cuda").to(torch.bfloat16)
    wf = torch.randn(O, I, device="cuda") * 0.05
    w16 = wf.to(torch.bfloat16)
    bias = torch.zeros(O, device="cuda")
    yd = torch.empty(B, O, device="cuda")
    wsb = native.dense_workspace_bytes(d)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    native.dense_fwd(d, xb.data_ptr(), wf.data_ptr(), w16.data_ptr(), bias.data_ptr(), yd.data_ptr(), ws.data_ptr(),
                     wsb, st)
    gy = torch.randn(B, O, device="cuda")
    dxd = torch.empty(B, I, device="cuda", dtype=torch.bfloat16)
    dwd = torch.empty(O, I, device="cuda")
    dbd = torch.empty(O, device="cuda")
    vw, vb = torch.zeros_like(wf), torch.zeros_like(bias)
    native.dense_bwd(d, xb.data_ptr(), gy.data_ptr(), wf.data_ptr(), w16.data_ptr(), bias.data_ptr(), dxd.data_ptr(),
                     None, dwd.data_ptr(), dbd.data_ptr(), (0.01, 0.9, vw.data_ptr(), vb.data_ptr()), ws.data_ptr(),
                     wsb, st)
    torch.cuda.synchronize()
    print("sanitize_conv: all launches completed")


if __name__ == "__main__":
    main()
