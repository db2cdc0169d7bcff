"""Kernel- and step-level parity of the B200 path against the CPU oracle
(SURVEY §8(c) tiers T1 and T2), called through the C ABI.

T1: per-layer activations and logits of one forward, and every parameter
    gradient of one backward, for identical inputs and weights.
T2: loss, weights and velocities after one train_batch.
Tolerances are norm-wise ||a-b||/||b||: 1e-5 in the fp32 check mode for every
tensor; 1e-2 in bf16 for activations, logits and loss (north_star). In bf16
the backward chain stores every activation/gradient in bf16, so ReLU masks and
max-pool argmax routing flip on near-ties and the deep-layer gradients drift
by up to ~0.15 (measured identically with the CUDA-core kernels, so it is the
storage precision, not a kernel defect; per-kernel bf16 parity on bf16-exact
inputs is held to 1e-2 in test_gpu_kernels.py). Those gradients get a sanity
bound only (GRAD_DRIFT_BF16), which still catches routing / layout bugs.
"""

import numpy as np
import pytest

from oracle.cnn_ref import OracleNet
from paper_1909_12291_b200.network import instantiate

from parity_util import CASES, TOL, case_genome, make_batch, rel

pytestmark = pytest.mark.gpu

N = 8
GRAD_DRIFT_BF16 = 0.25


def _layer_shapes(net):
    shapes = []
    for layer in net.layers:
        shapes.append(layer.out_shape if hasattr(layer, "out_shape") else (layer.out_units,))
    return shapes


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("name,text,shape", CASES, ids=[c[0] for c in CASES])
def test_forward_backward_step(name, text, shape, precision):
    genome = case_genome(text)
    net = instantiate(genome, shape, seed=3)
    oracle = OracleNet.from_network(net)
    x, y = make_batch(N, shape, seed=11)
    tol = TOL[precision]
    dev = net.to_device(0, precision, max_batch=N)
    dev.keep_grads()
    try:
        # ---- T1 forward: every layer output and the logits
        logits = dev.forward(x)
        ref_logits = oracle.forward(x)
        for li, lshape in enumerate(_layer_shapes(net)):
            if not dev.materialized(li):  # conv fused with its max-pool: checked through the pool output
                continue
            got = dev.activation(li, N, lshape)
            err = rel(got, oracle.outs[li])
            assert err <= tol, f"layer {li} activation rel err {err:.3e}"
        assert rel(logits, ref_logits) <= tol, f"logits rel err {rel(logits, ref_logits):.3e}"

        # ---- T1 backward + T2 step
        lr, mu = 1e-3, 0.9
        loss = dev.train_batch(x, y, lr, mu)
        ref_loss = oracle.train_batch(x, y, lr, mu)
        assert abs(loss - ref_loss) <= tol * max(1.0, abs(ref_loss)), (loss, ref_loss)
        gtol = GRAD_DRIFT_BF16 if precision == "bf16" else tol
        for p, (w, b) in enumerate(net.weights):
            gw, gb = dev.get_grads(p, w.shape, b.shape)
            rgw, rgb = oracle.grads[p]
            assert rel(gw, rgw) <= gtol, f"param layer {p} dW rel err {rel(gw, rgw):.3e}"
            assert rel(gb, rgb) <= gtol, f"param layer {p} db rel err {rel(gb, rgb):.3e}"
            nw, nb, vw, vb = dev.get_params(p, w.shape, b.shape)
            (rw, rb), (rvw, rvb) = oracle.params[p], oracle.vel[p]
            wtol = 1e-3 if precision == "bf16" else tol
            assert rel(nw, rw) <= wtol, f"param layer {p} W after step rel err {rel(nw, rw):.3e}"
            assert rel(vw, rvw) <= gtol, f"param layer {p} V after step rel err {rel(vw, rvw):.3e}"
            assert rel(nb, rb) <= gtol or np.abs(nb - rb).max() < 1e-7
    finally:
        net.release()


def test_sgd_bit_exact_fp32():
    """With identical gradients the update is the reference's fp32 arithmetic:
    checked via a 1-sample, single-dense network where dW = g x^T is exact."""
    genome = case_genome("id=case0000000009 parents= lr=0.01 momentum=0.9 batch_size=1 f0=pool:size=2,s=2")
    net = instantiate(genome, (3, 4, 4), seed=0)
    oracle = OracleNet.from_network(net)
    x, y = make_batch(2, (3, 4, 4), seed=5)
    dev = net.to_device(0, "fp32", max_batch=2)
    try:
        for _ in range(3):
            dev.train_batch(x[:1], y[:1], 0.01, 0.9)
            oracle.train_batch(x[:1], y[:1], 0.01, 0.9)
        w, b = net.weights[0]
        nw, nb, vw, vb = dev.get_params(0, w.shape, b.shape)
        assert rel(nw, oracle.params[0][0]) < 1e-6
    finally:
        net.release()


@pytest.mark.parametrize("name,text,shape", CASES, ids=[c[0] for c in CASES])
def test_device_init_bit_exact(name, text, shape):
    """ce_net_init_uniform (device PCG64 jump-ahead) == the host Kaiming draw, bit for bit."""
    genome = case_genome(text)
    lazy = instantiate(genome, shape, seed=17)            # weights drawn on the device
    dev = lazy.to_device(0, "bf16", max_batch=4)
    host = instantiate(genome, shape, seed=17, lazy=False)  # weights drawn by numpy
    try:
        for p, (w, b) in enumerate(host.weights):
            dw, db, vw, vb = dev.get_params(p, w.shape, b.shape)
            np.testing.assert_array_equal(dw, w)
            assert not db.any() and not vw.any() and not vb.any()
    finally:
        lazy.release()
