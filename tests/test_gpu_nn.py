"""Operator-level drop-in (paper_1909_12291_b200.nn, mirroring convevo/nn.py)
and the kernel-level C ABI entries it sits on (gather, dense, xent, SGD,
PCG64, flatten permutation), against the CPU oracle (oracle/cnn_ref.py).

Tolerances (norm-wise ||a-b||/||b||, SURVEY.md section 8(c) tier T1/T2):
fp32 mode <= 1e-5, bf16 mode <= 1e-2 (1.5e-2 for bf16 grads that pass
through a bf16-rounded activation); integer / RNG / permutation / SGD work is
bit-exact."""

import numpy as np
import pytest
import torch

from oracle import cnn_ref as ref
from paper_1909_12291_b200 import native
from paper_1909_12291_b200 import nn
from paper_1909_12291_b200.faults import ShapeError

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "bf16": 1e-2}
DT = {"fp32": np.float32, "bf16": "bf16"}


def rel(a, b):
    a = a.detach().float().cpu().numpy() if torch.is_tensor(a) else np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def host(t):
    return t.detach().float().cpu().numpy()


def stream():
    return torch.cuda.current_stream().cuda_stream


# ---------------------------------------------------------------- kernel-level entries
def test_pcg64_uniform_bit_exact():
    rng = np.random.default_rng(1234)
    st = rng.bit_generator.state["state"]
    out = torch.empty(10000, dtype=torch.float32, device="cuda")
    native.pcg64_uniform(st["state"], st["inc"], 777, -0.25, 0.75, out.data_ptr(), out.numel(), stream())
    rng.bit_generator.advance(777)
    want = rng.uniform(-0.25, 0.75, size=10000).astype(np.float32)
    np.testing.assert_array_equal(host(out), want)


def test_kaiming_init_matches_reference_draws():
    rng_dev, rng_host = np.random.default_rng(7), np.random.default_rng(7)
    conv = nn.Conv2d(3, 16, 5, 2, rng=rng_dev)
    dense = nn.Dense(40, 10, rng=rng_dev)
    lim_c, lim_d = np.sqrt(6.0 / 75), np.sqrt(6.0 / 40)
    wc = rng_host.uniform(-lim_c, lim_c, size=(16, 3, 5, 5)).astype(np.float32)
    wd = rng_host.uniform(-lim_d, lim_d, size=(10, 40)).astype(np.float32)
    np.testing.assert_array_equal(host(conv.params["w"]), wc)
    np.testing.assert_array_equal(host(dense.params["w"]), wd)
    # the host generator is left where the reference's draws leave it
    assert rng_dev.bit_generator.state == rng_host.bit_generator.state


def test_permute_flatten_round_trip():
    rows, c, cs, hw = 5, 3, 8, 7 * 6
    rng = np.random.default_rng(0)
    src = rng.standard_normal((rows, c * hw)).astype(np.float32)
    s = torch.from_numpy(src).cuda()
    dev = torch.empty(rows, hw * cs, device="cuda")
    back = torch.empty(rows, c * hw, device="cuda")
    native.permute_flatten_weights(s.data_ptr(), rows, c, cs, hw, 0, dev.data_ptr(), stream())
    native.permute_flatten_weights(dev.data_ptr(), rows, c, cs, hw, 1, back.data_ptr(), stream())
    want = np.zeros((rows, hw, cs), np.float32)
    want[:, :, :c] = src.reshape(rows, c, hw).transpose(0, 2, 1)
    np.testing.assert_array_equal(host(dev), want.reshape(rows, -1))
    np.testing.assert_array_equal(host(back), src)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_gather_u8_normalize(prec):
    rng = np.random.default_rng(3)
    pix = rng.integers(0, 256, size=(10, 3, 5, 7), dtype=np.uint8)
    idx = np.array([3, 0, 9, 3], np.int32)
    p = torch.from_numpy(pix).cuda()
    i = torch.from_numpy(idx).cuda()
    out = torch.empty(4, 5, 7, 8, dtype=torch.bfloat16 if prec == "bf16" else torch.float32, device="cuda")
    native.gather_u8_normalize(p.data_ptr(), 3, 5, 7, i.data_ptr(), 4, 8, prec, out.data_ptr(), stream())
    want = np.zeros((4, 5, 7, 8), np.float32)
    want[..., :3] = (pix[idx].astype(np.float32) / np.float32(255)).transpose(0, 2, 3, 1)
    if prec == "bf16":
        want = torch.from_numpy(want).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(host(out), want)


def test_sgd_momentum_bit_exact_and_validation():
    rng = np.random.default_rng(5)
    w, v, g = (rng.standard_normal(1001).astype(np.float32) for _ in range(3))
    tw, tv, tg = (torch.from_numpy(a.copy()).cuda() for a in (w, v, g))
    for _ in range(2):
        native.sgd_momentum(tw.data_ptr(), tv.data_ptr(), tg.data_ptr(), 1001, 0.01, 0.9, stream())
        w, v = ref.sgd(w, v, g, 0.01, 0.9)
    np.testing.assert_array_equal(host(tw), w)
    np.testing.assert_array_equal(host(tv), v)
    with pytest.raises(ValueError):
        native.sgd_momentum(tw.data_ptr(), tv.data_ptr(), tg.data_ptr(), 1001, 0.0, 0.9, stream())
    with pytest.raises(ValueError):
        native.sgd_momentum(tw.data_ptr(), tv.data_ptr(), tg.data_ptr(), 1001, 0.1, 1.0, stream())


def test_softmax_cross_entropy():
    rng = np.random.default_rng(9)
    logits = (rng.standard_normal((37, 2)) * 4).astype(np.float32)
    labels = rng.integers(0, 2, 37)
    loss, grad = nn.softmax_cross_entropy(torch.from_numpy(logits).cuda(), labels)
    rl, rg = ref.softmax_xent(logits, labels)
    assert abs(loss - rl) <= 1e-6 * max(1.0, abs(rl))
    assert rel(grad, rg) <= 1e-6
    with pytest.raises(ValueError):
        nn.softmax_cross_entropy(torch.from_numpy(logits).cuda(), np.full(37, 2))


# ---------------------------------------------------------------- layers vs oracle
CONV_CASES = [  # (n, c_in, h, w, c_out, k, s)
    (4, 3, 20, 20, 16, 4, 2),
    (2, 16, 11, 13, 32, 3, 1),
    (3, 8, 9, 9, 12, 2, 3),     # c_out not a multiple of 8, k < s (dgrad holes)
    (2, 24, 7, 7, 8, 7, 1),     # 1x1 output
]


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("case", CONV_CASES)
def test_conv2d_layer(prec, case):
    n, c, h, w, co, k, s = case
    rng = np.random.default_rng(sum(case))
    layer = nn.Conv2d(c, co, k, s, rng=np.random.default_rng(1), dtype=DT[prec])
    layer.params["b"].copy_(torch.from_numpy(rng.standard_normal(co).astype(np.float32)))
    x = rng.random((n, c, h, w), dtype=np.float32)
    if prec == "bf16":  # compare on the bf16-representable input the device consumes
        x = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    W, b = host(layer.params["w"]), host(layer.params["b"])
    y = layer.forward(torch.from_numpy(x).cuda())
    ry = ref.conv_forward(x, W, b, s)
    assert tuple(y.shape) == ry.shape
    assert rel(y, ry) <= TOL[prec]
    gy = rng.standard_normal(ry.shape).astype(np.float32)
    if prec == "bf16":
        gy = torch.from_numpy(gy).to(torch.bfloat16).float().numpy()
    dx = layer.backward(torch.from_numpy(gy).cuda())
    rdx, rdw, rdb = ref.conv_backward(x, W, s, gy)
    assert tuple(dx.shape) == x.shape
    assert rel(dx, rdx) <= TOL[prec]
    assert rel(layer.grads["w"], rdw) <= TOL[prec]
    assert rel(layer.grads["b"], rdb) <= TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("size,stride", [(2, 1), (2, 2), (2, 3), (3, 1), (3, 2), (3, 3)])
def test_maxpool_layer(prec, size, stride):
    rng = np.random.default_rng(size * 10 + stride)
    x = rng.integers(0, 6, size=(2, 16, 11, 10)).astype(np.float32)  # many ties
    if prec == "bf16":
        xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    else:
        xt = torch.from_numpy(x).cuda()
    pool = nn.MaxPool(size, stride)
    y = pool.forward(xt)
    ry, rarg = ref.pool_forward(x, size, stride)
    np.testing.assert_array_equal(host(y), ry)
    np.testing.assert_array_equal(pool.argmax_indices.cpu().numpy(), rarg)
    gy = rng.integers(-4, 5, size=ry.shape).astype(np.float32)  # exact in bf16, exact sums
    gyt = torch.from_numpy(gy).cuda()
    dx = pool.backward(gyt.to(torch.bfloat16) if prec == "bf16" else gyt)
    np.testing.assert_array_equal(host(dx), ref.pool_backward(gy, rarg, x.shape, size, stride))


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("n,i,o", [(32, 300, 20), (16, 1000, 2), (64, 77, 13), (5, 4096, 64)])
def test_dense_layer(prec, n, i, o):
    rng = np.random.default_rng(n + i + o)
    layer = nn.Dense(i, o, rng=np.random.default_rng(2), dtype=DT[prec])
    layer.params["b"].copy_(torch.from_numpy(rng.standard_normal(o).astype(np.float32)))
    x = rng.standard_normal((n, i)).astype(np.float32)
    W, b = host(layer.params["w"]), host(layer.params["b"])
    xr = x
    if prec == "bf16":
        xr = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
        Wr = torch.from_numpy(W).to(torch.bfloat16).float().numpy()
    else:
        Wr = W
    y = layer.forward(torch.from_numpy(x).cuda())
    assert rel(y, ref.dense_forward(xr, Wr, b)) <= TOL[prec]
    gy = rng.standard_normal((n, o)).astype(np.float32)
    dx = layer.backward(torch.from_numpy(gy).cuda())
    rdx, rdw, rdb = ref.dense_backward(xr, Wr, gy)
    assert rel(dx, rdx) <= TOL[prec]
    assert rel(layer.grads["w"], rdw) <= TOL[prec]
    assert rel(layer.grads["b"], rdb) <= 1e-6
    with pytest.raises(ShapeError):
        layer.forward(torch.zeros(n, i + 1, device="cuda"))


def _fixed_like(dtype, rng):
    """A small FIXED-shaped stack (nn.py layer API) on 3x24x24 inputs."""
    return [nn.Conv2d(3, 8, 4, 2, rng=rng, dtype=dtype), nn.ReLU(),
            nn.Conv2d(8, 16, 3, 1, rng=rng, dtype=dtype), nn.ReLU(), nn.MaxPool(2, 2),
            nn.Flatten(), nn.Dense(16 * 4 * 4, 12, rng=rng, dtype=dtype), nn.Dense(12, 2, rng=rng, dtype=dtype)]


def _oracle_of(layers):
    spec, params = [], []
    i = 0
    while i < len(layers):
        L = layers[i]
        if isinstance(L, nn.Conv2d):
            relu = i + 1 < len(layers) and isinstance(layers[i + 1], nn.ReLU)
            spec.append(("conv", L.stride, relu))
            params.append((host(L.params["w"]), host(L.params["b"])))
            i += 2 if relu else 1
            continue
        if isinstance(L, nn.MaxPool):
            spec.append(("pool", L.size, L.stride))
        elif isinstance(L, nn.Dense):
            spec.append(("dense",))
            params.append((host(L.params["w"]), host(L.params["b"])))
        i += 1
    return ref.OracleNet(spec, params)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_network_train_batch_matches_oracle(prec):
    net = nn.Network(_fixed_like(DT[prec], np.random.default_rng(0)), input_shape=(3, 24, 24))
    oracle = _oracle_of(net.layers)
    rng = np.random.default_rng(4)
    x = rng.random((16, 3, 24, 24), dtype=np.float32)
    y = rng.integers(0, 2, 16)
    tol = 1e-5 if prec == "fp32" else 3e-2
    for step in range(3):
        loss = nn.train_batch(net, torch.from_numpy(x).cuda(), y, 0.01, 0.9)
        rl = oracle.train_batch(x, y, 0.01, 0.9)
        assert abs(loss - rl) <= tol * max(1.0, abs(rl)), (step, loss, rl)
    # parameters() yields b before w per layer (nn.py:280-284)
    names = [name for _, name, _ in net.parameters()]
    params = [p for _, _, p in net.parameters()]
    flat = [t for pair in oracle.params for t in (pair[1], pair[0])]
    for name, got, want in zip(names, params, flat):
        # biases start at 0, so after k steps they ARE the cumulative update:
        # bf16 routing/rounding differences show up there undiluted (T3 drift)
        bound = tol if (prec == "fp32" or name == "w") else 0.1
        assert rel(got, want) <= bound, name


def test_network_validation():
    rng = np.random.default_rng(0)
    with pytest.raises(ValueError):
        nn.Network([nn.Conv2d(3, 8, 3, rng=rng)])
    with pytest.raises(ValueError):
        nn.Network([nn.Dense(4, 3, rng=rng)], class_count=2)
    net = nn.Network(_fixed_like(np.float32, rng), input_shape=(3, 24, 24))
    with pytest.raises(ShapeError):
        net.forward(torch.zeros(2, 3, 25, 24, device="cuda"))
    with pytest.raises(ShapeError) as e:
        nn.infer_shapes([nn.Conv2d(3, 8, 5, rng=rng), nn.MaxPool(3), nn.Conv2d(8, 8, 5, rng=rng)], (3, 10, 10))
    assert e.value.layer_index == 2
    with pytest.raises(ValueError):
        nn.sgd_step(net, 0.0)
    with pytest.raises(ValueError):
        nn.Conv2d(3, 8, 0)


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("shape", [(4, 8, 13, 13), (3, 5), (1, 7, 1, 1)])
def test_relu_native_exact(dtype, shape):
    """Operator-API ReLU runs the library kernel (ce_relu_fwd/bwd) and matches
    nn.py:178-183 exactly: where(x > 0, x, 0) and grad * (x > 0)."""
    rng = np.random.default_rng(len(shape))
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = torch.from_numpy(rng.standard_normal(shape).astype(np.float32)).to(tdt).cuda()
    x.view(-1)[0] = 0.0  # x == 0 is not > 0
    g = torch.from_numpy(rng.standard_normal(shape).astype(np.float32)).to(tdt).cuda()
    layer = nn.ReLU()
    y = layer.forward(x)
    dx = layer.backward(g)
    torch.cuda.synchronize()
    xr = x.float().cpu().numpy()
    np.testing.assert_array_equal(y.float().cpu().numpy(), np.where(xr > 0, xr, 0))
    np.testing.assert_array_equal(dx.float().cpu().numpy(), g.float().cpu().numpy() * (xr > 0))
    assert y.dtype == tdt and dx.dtype == tdt and layer._mask.dtype == torch.uint8
