"""T1 kernel parity through the kernel-level C ABI on bf16-exact inputs.

Inputs and weights are rounded to bf16 first, so the oracle (float64 on the
same values) and the tcgen05 kernels see identical operands; the remaining
error is fp32 accumulation + the bf16 rounding of stored outputs. This is the
per-kernel bar of north_star (rel <= 1e-2 bf16, <= 1e-5 fp32 check mode);
pooling is exact.
"""

import numpy as np
import pytest

from oracle import cnn_ref as O
from paper_1909_12291_b200 import native

from parity_util import rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

# (n, c, h, c_out, k, s): FIXED layers (c padded 3->8), SWEET-like, random-genome-like
SHAPES = [(4, 8, 100, 32, 4, 2), (4, 32, 49, 64, 4, 1), (4, 64, 23, 128, 4, 1), (2, 256, 19, 256, 4, 1),
          (3, 16, 33, 8, 1, 2), (2, 8, 40, 24, 7, 3), (2, 128, 16, 256, 2, 3), (5, 64, 17, 16, 5, 2),
          (2, 32, 12, 64, 3, 3), (1, 16, 9, 128, 6, 1), (2, 24, 11, 40, 3, 2),
          (2, 96, 10, 64, 3, 1)]  # C % 64 == 32: the 32-channel (SWIZZLE_64B) im2col fwd / wgrad


def _round(a, precision):
    if precision == "fp32":
        return a.astype(np.float32)
    return torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).float().numpy()


def _dev(a_nhwc, precision):
    t = torch.from_numpy(np.ascontiguousarray(a_nhwc, dtype=np.float32)).cuda()
    return t.to(torch.bfloat16).contiguous() if precision == "bf16" else t.contiguous()


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("shape", SHAPES, ids=[str(s) for s in SHAPES])
def test_conv_passes(shape, precision):
    n, c, h, co, k, s = shape
    rng = np.random.default_rng(sum(shape))
    x = _round(rng.standard_normal((n, c, h, h)), precision)
    w = _round(rng.uniform(-0.2, 0.2, (co, c, k, k)), precision)
    b = rng.uniform(-0.1, 0.1, co).astype(np.float32)
    oh = (h - k) // s + 1
    dy = _round(rng.standard_normal((n, co, oh, oh)), precision)
    mask_src = rng.standard_normal((n, c, h, h)).astype(np.float32)
    # oracle in float64 on the same (rounded) values
    y_ref = O.conv_forward(x.astype(np.float64), w.astype(np.float64), b.astype(np.float64), s)
    y_ref = np.maximum(y_ref, 0)
    dx_ref, dw_ref, db_ref = O.conv_backward(x.astype(np.float64), w.astype(np.float64), s, dy.astype(np.float64))
    dx_ref = dx_ref * (mask_src > 0)

    desc = native.conv_desc(n, c, h, h, co, k, s, precision)
    xd = _dev(x.transpose(0, 2, 3, 1), precision)
    wd = _dev(w.transpose(0, 2, 3, 1), precision)           # [o][kh][kw][c]
    bd = torch.from_numpy(b).cuda()
    yd = torch.empty((n, oh, oh, co), dtype=xd.dtype, device="cuda")
    dyd = _dev(dy.transpose(0, 2, 3, 1), precision)
    maskd = _dev(mask_src.transpose(0, 2, 3, 1), precision)
    dxd = torch.empty_like(xd)
    dwd = torch.empty((co, k, k, c), dtype=torch.float32, device="cuda")
    dbd = torch.empty(co, dtype=torch.float32, device="cuda")
    wsb = native.conv_workspace_bytes(desc)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    native.conv_fwd(desc, xd.data_ptr(), wd.data_ptr(), bd.data_ptr(), 1, yd.data_ptr(), st)
    native.conv_dgrad(desc, dyd.data_ptr(), wd.data_ptr(), maskd.data_ptr(), dxd.data_ptr(), ws.data_ptr(), wsb, st)
    native.conv_wgrad(desc, xd.data_ptr(), dyd.data_ptr(), dwd.data_ptr(), dbd.data_ptr(), ws.data_ptr(), wsb, st)
    torch.cuda.synchronize()
    tol = 1e-2 if precision == "bf16" else 1e-5
    y = yd.float().cpu().numpy().transpose(0, 3, 1, 2)
    dx = dxd.float().cpu().numpy().transpose(0, 3, 1, 2)
    dw = dwd.cpu().numpy().transpose(0, 3, 1, 2)
    assert rel(y, y_ref) <= tol, f"fwd rel err {rel(y, y_ref):.3e}"
    assert rel(dx, dx_ref) <= tol, f"dgrad rel err {rel(dx, dx_ref):.3e}"
    assert rel(dw, dw_ref) <= tol, f"wgrad rel err {rel(dw, dw_ref):.3e}"
    assert rel(dbd.cpu().numpy(), db_ref) <= tol


# (n, c, h, c_out, k, s, pool window, pool stride, relu): packed-like C=8, gather C=16/32, C%64==0,
# ragged pooled edges, stride > window gaps, more windows than one wave of tiles
POOL_SHAPES = [(4, 32, 49, 64, 4, 1, 2, 2, 1), (3, 8, 40, 24, 3, 1, 3, 3, 1), (2, 16, 33, 40, 3, 2, 2, 3, 1),
               (2, 64, 30, 128, 3, 1, 2, 2, 1), (3, 24, 29, 16, 5, 1, 3, 3, 0), (2, 256, 20, 256, 3, 1, 3, 3, 1),
               (16, 32, 49, 64, 4, 1, 2, 2, 1)]


@pytest.mark.parametrize("shape", POOL_SHAPES, ids=[str(s) for s in POOL_SHAPES])
def test_conv_pool_epilogue(shape):
    """ce_conv_fwd with the max-pool epilogue == conv then ce_maxpool_fwd, bit for bit (same bf16
    values compared, same first-max rule), and == the oracle's conv+ReLU+MaxPool (nn.py:82-150)."""
    n, c, h, co, k, s, pk, ps, relu = shape
    rng = np.random.default_rng(sum(shape))
    x = _round(rng.standard_normal((n, c, h, h)), "bf16")
    w = _round(rng.uniform(-0.2, 0.2, (co, c, k, k)), "bf16")
    b = rng.uniform(-0.1, 0.1, co).astype(np.float32)
    oh = (h - k) // s + 1
    ph = (oh - pk) // ps + 1
    desc = native.conv_desc(n, c, h, h, co, k, s, "bf16")
    xd = _dev(x.transpose(0, 2, 3, 1), "bf16")
    wd = _dev(w.transpose(0, 2, 3, 1), "bf16")
    bd = torch.from_numpy(b).cuda()
    yfull = torch.empty((n, oh, oh, co), dtype=torch.bfloat16, device="cuda")
    yp = torch.full((n, ph, ph, co), 7.0, dtype=torch.bfloat16, device="cuda")
    argp = torch.full((n, ph, ph, co), 77, dtype=torch.uint8, device="cuda")
    yu = torch.empty_like(yp)
    argu = torch.empty_like(argp)
    st = torch.cuda.current_stream().cuda_stream
    native.conv_fwd(desc, xd.data_ptr(), wd.data_ptr(), bd.data_ptr(), relu, yp.data_ptr(), st, pool=(pk, ps),
                    arg=argp.data_ptr())
    native.conv_fwd(desc, xd.data_ptr(), wd.data_ptr(), bd.data_ptr(), relu, yfull.data_ptr(), st)
    pdesc = native.conv_desc(n, co, oh, oh, 0, pk, ps, "bf16")
    native.maxpool_fwd(pdesc, yfull.data_ptr(), yu.data_ptr(), argu.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(yp, yu), "fused pooled values differ from conv + pool"
    a_f, a_u = argp.cpu().numpy(), argu.cpu().numpy()
    dead = a_f == 0xFF
    if relu:
        assert np.all(yu.float().cpu().numpy()[dead] == 0.0)
    else:
        assert not dead.any()
    np.testing.assert_array_equal(a_f[~dead], a_u[~dead])
    y_ref = O.conv_forward(x.astype(np.float64), w.astype(np.float64), b.astype(np.float64), s)
    if relu:
        y_ref = np.maximum(y_ref, 0)
    p_ref, _ = O.pool_forward(y_ref, pk, ps)
    got = yp.float().cpu().numpy().transpose(0, 3, 1, 2)
    assert rel(got, p_ref) <= 1e-2, f"pooled rel err {rel(got, p_ref):.3e}"


def test_conv_pool_epilogue_rejects_overlap():
    desc = native.conv_desc(1, 8, 10, 10, 8, 3, 1, "bf16")
    t = torch.zeros(1024, device="cuda")
    with pytest.raises(Exception):
        native.conv_fwd(desc, t.data_ptr(), t.data_ptr(), t.data_ptr(), 1, t.data_ptr(), 0, pool=(3, 2),
                        arg=t.data_ptr())


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("size,stride", [(2, 1), (2, 2), (2, 3), (3, 1), (3, 2), (3, 3)])
@pytest.mark.parametrize("variant", ["rand", "ties"])
def test_pool_exact(size, stride, variant, precision):
    rng = np.random.default_rng(size * 7 + stride)
    n, c, h = 3, 16, 13
    if variant == "rand":
        x = _round(rng.standard_normal((n, c, h, h)), precision)
    else:
        x = rng.integers(0, 3, size=(n, c, h, h)).astype(np.float32)
    oh = (h - size) // stride + 1
    dy = _round(rng.standard_normal((n, c, oh, oh)), precision)
    y_ref, arg_ref = O.pool_forward(x, size, stride)
    dx_ref = O.pool_backward(dy.astype(np.float64), arg_ref, x.shape, size, stride)
    desc = native.conv_desc(n, c, h, h, 0, size, stride, precision)
    xd = _dev(x.transpose(0, 2, 3, 1), precision)
    yd = torch.empty((n, oh, oh, c), dtype=xd.dtype, device="cuda")
    argd = torch.empty((n, oh, oh, c), dtype=torch.uint8, device="cuda")
    dyd = _dev(dy.transpose(0, 2, 3, 1), precision)
    dxd = torch.empty_like(xd)
    native.maxpool_fwd(desc, xd.data_ptr(), yd.data_ptr(), argd.data_ptr())
    native.maxpool_bwd(desc, dyd.data_ptr(), argd.data_ptr(), None, dxd.data_ptr())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(yd.float().cpu().numpy().transpose(0, 3, 1, 2), y_ref)
    np.testing.assert_array_equal(argd.cpu().numpy().transpose(0, 3, 1, 2), arg_ref)
    dx = dxd.float().cpu().numpy().transpose(0, 3, 1, 2)
    if precision == "fp32" or size <= stride:  # no overlap: a single term per input, exact
        assert rel(dx, dx_ref) <= 1e-6
    else:  # overlapping windows accumulate in fp32 then round to bf16
        assert rel(dx, dx_ref) <= 1e-2


def test_wgrad_multiwave_splits():
    """Long reductions take the multi-wave split count (conv_wgrad_splits: 8x256x94x94 k4 has
    32 M tiles and 1,036 k-blocks -> 9 splits, 288 units on 148 SMs); checked against a
    PyTorch fp32 (no TF32) weight gradient on the same bf16 operands."""
    n, c, h, co, k, s = 8, 256, 94, 256, 4, 1
    oh = h - k + 1
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(n, c, h, h, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(n, co, oh, oh, device="cuda", generator=g).to(torch.bfloat16)
    prev = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False
    try:
        dw_ref = torch.nn.grad.conv2d_weight(x.float(), (co, c, k, k), dy.float(), stride=s)
    finally:
        torch.backends.cudnn.allow_tf32 = prev
    desc = native.conv_desc(n, c, h, h, co, k, s, "bf16")
    xd = x.permute(0, 2, 3, 1).contiguous()
    dyd = dy.permute(0, 2, 3, 1).contiguous()
    dwd = torch.empty((co, k, k, c), dtype=torch.float32, device="cuda")
    dbd = torch.empty(co, dtype=torch.float32, device="cuda")
    wsb = native.conv_workspace_bytes(desc)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    native.conv_wgrad(desc, xd.data_ptr(), dyd.data_ptr(), dwd.data_ptr(), dbd.data_ptr(), ws.data_ptr(), wsb, st)
    torch.cuda.synchronize()
    dw = dwd.permute(0, 3, 1, 2).cpu().numpy()
    assert rel(dw, dw_ref.cpu().numpy()) <= 1e-2, f"wgrad rel err {rel(dw, dw_ref.cpu().numpy()):.3e}"
    db_ref = dy.float().sum(dim=(0, 2, 3)).cpu().numpy()
    assert rel(dbd.cpu().numpy(), db_ref) <= 1e-2


@pytest.mark.parametrize("shape", [(64, 256, 97, 256, 4, 1), (64, 128, 46, 128, 3, 1)], ids=["sweet_b64", "vgg_l3_b64"])
def test_conv_passes_full_size(shape):
    """SWEET and a VGG16STYLE layer at B=64: thousands of 128-row tiles, so
    every persistent CTA runs many tiles (TMEM accumulator flip, mbarrier phase wrap). fwd /
    dgrad / wgrad vs PyTorch fp32 (TF32 off) on the same bf16-exact operands, <= 1e-2."""
    import torch.nn.functional as F
    n, c, h, co, k, s = shape
    oh = (h - k) // s + 1
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(n, c, h, h, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(co, c, k, k, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    b = torch.randn(co, device="cuda", generator=g) * 0.1
    dy = torch.randn(n, co, oh, oh, device="cuda", generator=g).to(torch.bfloat16)
    desc = native.conv_desc(n, c, h, h, co, k, s, "bf16")
    xd, wd = x.permute(0, 2, 3, 1).contiguous(), w.permute(0, 2, 3, 1).contiguous()
    dyd = dy.permute(0, 2, 3, 1).contiguous()
    yd = torch.empty(n, oh, oh, co, device="cuda", dtype=torch.bfloat16)
    dxd = torch.empty_like(xd)
    dwd = torch.empty(co, k, k, c, device="cuda")
    dbd = torch.empty(co, device="cuda")
    wsb = native.conv_workspace_bytes(desc)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    native.conv_fwd(desc, xd.data_ptr(), wd.data_ptr(), b.data_ptr(), 0, yd.data_ptr(), st)
    native.conv_dgrad(desc, dyd.data_ptr(), wd.data_ptr(), None, dxd.data_ptr(), ws.data_ptr(), wsb, st)
    native.conv_wgrad(desc, xd.data_ptr(), dyd.data_ptr(), dwd.data_ptr(), dbd.data_ptr(), ws.data_ptr(), wsb, st)
    torch.cuda.synchronize()
    prev = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False
    try:
        y_ref = F.conv2d(x.float(), w.float(), b, stride=s)
        dx_ref = torch.nn.grad.conv2d_input(x.shape, w.float(), dy.float(), stride=s)
        dw_ref = torch.nn.grad.conv2d_weight(x.float(), w.shape, dy.float(), stride=s)
    finally:
        torch.backends.cudnn.allow_tf32 = prev

    def trel(a, r):
        return float((a.float() - r).norm() / r.norm())
    assert trel(yd.permute(0, 3, 1, 2), y_ref) <= 1e-2
    assert trel(dxd.permute(0, 3, 1, 2), dx_ref) <= 1e-2
    assert trel(dwd.permute(0, 3, 1, 2), dw_ref) <= 1e-2
    assert trel(dbd, dy.float().sum(dim=(0, 2, 3))) <= 1e-2
