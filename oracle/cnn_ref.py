"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain numpy restatement of the reference's candidate-evaluation arithmetic
(convevo, /root/reference/pkg/src/convevo), used as the parity checker for the
B200 path and as the `cpu_baseline` / `--impl reference` leg of bench.py.
Only tests/, __graft_entry__.smoke() and bench.py may import this module; the
product path (paper_1909_12291_b200) never does and has no CPU fallback.

Pinned: tests/test_oracle_golden.py checks every function here against golden
vectors produced by running the reference itself in the build container
(tests/golden/make_golden.py -> tests/golden/*.npz, numpy 2.3.5 / OpenBLAS
0.3.30). Each function cites the reference lines it restates.

Layouts follow the reference: activations NCHW, conv W (out, in, kh, kw),
dense W (out, in), flatten in (c, h, w) order.
"""

import math
import time

import numpy as np


# ------------------------------------------------------------------ layers
def conv_forward(x, w, b, stride):
    """Valid cross-correlation, taps outer / channels inner (nn.py:82-94)."""
    n, c, h, wd = x.shape
    co, ci, k, _ = w.shape
    oh, ow = (h - k) // stride + 1, (wd - k) // stride + 1
    acc = np.zeros((n, oh, ow, co), dtype=x.dtype)
    for i in range(k):
        for j in range(k):
            tap = x[:, :, i:i + stride * oh:stride, j:j + stride * ow:stride]
            acc += np.tensordot(tap, w[:, :, i, j], axes=([1], [1]))
    return np.ascontiguousarray(acc.transpose(0, 3, 1, 2) + b[None, :, None, None])


def conv_backward(x, w, stride, gy):
    """(dx, dw, db) of conv_forward (nn.py:96-116)."""
    n, c, h, wd = x.shape
    co, ci, k, _ = w.shape
    oh, ow = gy.shape[2], gy.shape[3]
    g = gy.transpose(0, 2, 3, 1)
    dw = np.zeros_like(w)
    dx = np.zeros_like(x)
    for i in range(k):
        for j in range(k):
            tap = x[:, :, i:i + stride * oh:stride, j:j + stride * ow:stride]
            dw[:, :, i, j] = np.tensordot(g, tap, axes=([0, 1, 2], [0, 2, 3]))
            dx[:, :, i:i + stride * oh:stride, j:j + stride * ow:stride] += \
                np.tensordot(g, w[:, :, i, j], axes=([3], [0])).transpose(0, 3, 1, 2)
    return dx, dw, gy.sum(axis=(0, 2, 3))


def pool_forward(x, size, stride):
    """Max over windows; argmax = first max in row-major order (nn.py:140-150)."""
    n, c, h, wd = x.shape
    oh, ow = (h - size) // stride + 1, (wd - size) // stride + 1
    views = np.stack([x[:, :, i:i + stride * oh:stride, j:j + stride * ow:stride]
                      for i in range(size) for j in range(size)], axis=0)
    return views.max(axis=0), views.argmax(axis=0)


def pool_backward(gy, arg, in_shape, size, stride):
    """Route each output grad to its argmax, accumulating on overlap (nn.py:156-167)."""
    oh, ow = gy.shape[2], gy.shape[3]
    gx = np.zeros(in_shape, dtype=gy.dtype)
    for idx in range(size * size):
        i, j = divmod(idx, size)
        gx[:, :, i:i + stride * oh:stride, j:j + stride * ow:stride] += gy * (arg == idx)
    return gx


def relu_forward(x):
    mask = x > 0
    return np.where(mask, x, np.zeros((), dtype=x.dtype)), mask  # nn.py:178-180


def dense_forward(x, w, b):
    return x @ w.T + b  # nn.py:225-231


def dense_backward(x, w, gy):
    return gy @ w, gy.T @ x, gy.sum(axis=0)  # (dx, dw, db), nn.py:233-240


def softmax_xent(logits, labels):
    """Mean cross-entropy and its logits gradient (nn.py:287-303)."""
    labels = np.asarray(labels)
    n, k = logits.shape
    if labels.min() < 0 or labels.max() >= k:
        raise ValueError(f"labels must lie in [0, {k - 1}]")
    z = logits - logits.max(axis=1, keepdims=True)
    logp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    loss = -logp[np.arange(n), labels].mean()
    grad = np.exp(logp)
    grad[np.arange(n), labels] -= 1.0
    grad /= n
    return float(loss), grad.astype(logits.dtype)


def sgd(w, v, g, lr, momentum):
    """v <- mu v - lr g ; w <- w + v   in the array dtype (nn.py:306-322)."""
    v = momentum * v - lr * g
    return w + v, v


# ------------------------------------------------------------------ network
class OracleNet:
    """Executes a paper_1909_12291_b200.network.Network description on the CPU.

    layers: list of ("conv", stride, relu) / ("pool", size, stride) /
    ("dense",) entries; params: list of [w, b] per parameterised layer.
    """

    def __init__(self, layers, params, dtype=np.float32):
        self.layers = layers
        self.params = [[np.array(w, dtype=dtype), np.array(b, dtype=dtype)] for w, b in params]
        self.vel = [[np.zeros_like(w), np.zeros_like(b)] for w, b in self.params]
        self.grads = [[None, None] for _ in self.params]
        self.dtype = dtype

    @classmethod
    def from_network(cls, net, dtype=np.float32):
        from paper_1909_12291_b200.network import ConvLayer, PoolLayer  # description only
        layers = []
        for layer in net.layers:
            if isinstance(layer, ConvLayer):
                layers.append(("conv", layer.stride, layer.relu))
            elif isinstance(layer, PoolLayer):
                layers.append(("pool", layer.size, layer.stride))
            else:
                layers.append(("dense",))
        return cls(layers, net.weights, dtype)

    def forward(self, x, keep=True):
        """Returns logits; keeps per-layer caches (and outputs in self.outs)."""
        cache, outs = [], []
        p = 0
        for spec in self.layers:
            if spec[0] == "conv":
                w, b = self.params[p]
                y = conv_forward(x, w, b, spec[1])
                mask = None
                if spec[2]:
                    y, mask = relu_forward(y)
                cache.append((x, mask, p))
                p += 1
            elif spec[0] == "pool":
                y, arg = pool_forward(x, spec[1], spec[2])
                cache.append((x.shape, arg))
            else:
                flat_shape = None
                if x.ndim == 4:  # implicit Flatten, (c, h, w) order (nn.py:197-199)
                    flat_shape = x.shape
                    x = x.reshape(x.shape[0], -1)
                w, b = self.params[p]
                y = dense_forward(x, w, b)
                cache.append((x, p, flat_shape))
                p += 1
            outs.append(y)
            x = y
        if keep:
            self.cache, self.outs = cache, outs
        return x

    def backward(self, g):
        for spec, c in zip(reversed(self.layers), reversed(self.cache)):
            if spec[0] == "dense":
                x, p, flat_shape = c
                w = self.params[p][0]
                g, gw, gb = dense_backward(x, w, g)
                self.grads[p] = [gw, gb]
                if flat_shape is not None:
                    g = g.reshape(flat_shape)
            elif spec[0] == "conv":
                x, mask, p = c
                if mask is not None:
                    g = g * mask
                w = self.params[p][0]
                g, gw, gb = conv_backward(x, w, spec[1], g)
                self.grads[p] = [gw, gb]
            else:
                in_shape, arg = c
                g = pool_backward(g, arg, in_shape, spec[1], spec[2])
        return g

    def step(self, lr, momentum):
        for p, ((w, b), (vw, vb), (gw, gb)) in enumerate(zip(self.params, self.vel, self.grads)):
            w, vw = sgd(w, vw, gw, lr, momentum)
            b, vb = sgd(b, vb, gb, lr, momentum)
            self.params[p], self.vel[p] = [w, b], [vw, vb]

    def train_batch(self, x, y, lr, momentum):
        """One fwd -> xent -> bwd -> SGD step; returns the pre-step loss (nn.py:325-331)."""
        loss, g = softmax_xent(self.forward(x), y)
        self.backward(g)
        self.step(lr, momentum)
        return loss


# ------------------------------------------------------------------ candidate (evaluator.py)
def train_short(net, genome, train_set, epochs, seed, max_batches_per_epoch=None, dtype=np.float32):
    """evaluator.py:145-171 on the oracle net; returns (losses, seconds)."""
    x = train_set.pixels.astype(dtype) / dtype(255.0)
    y = train_set.labels.astype(np.int64)
    n = len(train_set)
    bs = min(genome.learn.batch_size, n)
    rng = np.random.default_rng([seed, 0xDA7A])
    losses = []
    t0 = time.monotonic()
    for epoch in range(epochs):
        perm = rng.permutation(n)
        for bi, start in enumerate(range(0, n - bs + 1, bs)):
            if max_batches_per_epoch is not None and bi >= max_batches_per_epoch:
                break
            idx = perm[start:start + bs]
            loss = net.train_batch(x[idx], y[idx], genome.learn.lr, genome.learn.momentum)
            losses.append(loss)
            if not math.isfinite(loss):
                return losses, time.monotonic() - t0, (loss, epoch, bi)
    return losses, time.monotonic() - t0, None


def predict_scores(net, pset, batch_size=128, dtype=np.float32):
    """evaluator.py:174-186."""
    x = pset.pixels.astype(dtype) / dtype(255.0)
    scores = np.empty(len(pset), dtype=np.float64)
    preds = np.empty(len(pset), dtype=np.int64)
    for start in range(0, len(pset), batch_size):
        logits = net.forward(x[start:start + batch_size], keep=False)
        z = logits - logits.max(axis=1, keepdims=True)
        p = np.exp(z)
        p /= p.sum(axis=1, keepdims=True)
        scores[start:start + len(logits)] = p[:, 1]
        preds[start:start + len(logits)] = logits.argmax(axis=1)
    return scores, preds


def measure_latency(net, input_shape, batch_size=64, reps=5, warmup=1, seed=0):
    """evaluator.py:189-210 (wall-clock seconds per batch)."""
    batch = np.random.default_rng(seed).random((batch_size, *input_shape), dtype=np.float32)
    for _ in range(warmup):
        net.forward(batch, keep=False)
    times = []
    for _ in range(reps):
        t0 = time.monotonic()
        net.forward(batch, keep=False)
        times.append(time.monotonic() - t0)
    return float(np.median(times)), min(times), max(times)
