"""Operator-level drop-in for the reference layer API (convevo/nn.py).

Same names, argument meaning and error behaviour as nn.py:18-380 -- Layer,
Conv2d, MaxPool, ReLU, Flatten, Dense, Network, softmax_cross_entropy,
sgd_step, train_batch, infer_shapes -- with the arithmetic on the B200 through
the kernel-level C ABI of libmenndl_sm100 (include/menndl_sm100.h):

  Conv2d.forward / backward  -> ce_conv_fwd / ce_conv_wgrad / ce_conv_dgrad
  MaxPool.forward / backward -> ce_maxpool_fwd / ce_maxpool_bwd
  Dense.forward / backward   -> ce_dense_fwd / ce_dense_bwd
  softmax_cross_entropy      -> ce_softmax_xent
  sgd_step                   -> ce_sgd_momentum (bit-exact fp32)
  Kaiming init               -> ce_pcg64_uniform (bit-exact numpy PCG64 draws)

Tensors are torch CUDA tensors in the reference's logical layouts (NCHW
activations, (o, c, k, k) conv weights, (out, in) dense weights); numpy inputs
are moved to the device. Feature-map outputs are NCHW *views* of the NHWC
buffers the kernels write, so a chain of layers moves no data between them.

Precision is per layer, like the reference's dtype argument:
  np.float32 / "fp32"        FFMA kernels, float32 activations (parity mode)
  "bf16" / torch.bfloat16    tcgen05 tensor cores, bf16 activations, fp32
                             master weights, gradients and optimiser state.
float64 networks (used by the reference only for grad_check, nn.py:334-367)
are not offered on the device: grad_check runs on the CPU oracle.

ReLU and Flatten are pure data movement here (torch elementwise / reshape);
the candidate runtime (libmenndl ce_train) fuses them into the conv epilogue
and the first dense layer's column order instead.
"""

import numpy as np
import torch

from . import native
from .faults import ShapeError

__all__ = ["Layer", "Conv2d", "MaxPool", "ReLU", "Flatten", "Dense", "Network", "softmax_cross_entropy",
           "sgd_step", "train_batch", "infer_shapes", "precision_of"]


def _out_dim(size, k, stride):
    return (size - k) // stride + 1


def _pad8(v):
    return (v + 7) // 8 * 8


def precision_of(dtype):
    """Map a reference-style dtype to the kernel precision ("fp32" | "bf16")."""
    if dtype in ("bf16", torch.bfloat16):
        return "bf16"
    if dtype in ("fp32", torch.float32):
        return "fp32"
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "fp32"
    raise ValueError(f"unsupported dtype {dtype!r}: the device layers run fp32 or bf16 "
                     "(float64 grad-checks run on the CPU oracle)")


def _act_dtype(prec):
    return torch.bfloat16 if prec == "bf16" else torch.float32


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1909_12291_b200.nn needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _as_tensor(x, dtype=None):
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    x = x.to(_device())
    return x if dtype is None else x.to(dtype)


def _ptr(t):
    return None if t is None else t.data_ptr()


def _precision_of(t):
    """Kernel precision of a device tensor: bf16 stays bf16, everything else runs as float32."""
    return "bf16" if t.dtype == torch.bfloat16 else "fp32"


def _to_nhwc(x, c_store, dtype):
    """NCHW (possibly a view of NHWC storage) -> contiguous NHWC with channels
    zero-padded to c_store, in the kernel's activation type."""
    x = _as_tensor(x, dtype)
    h = x.permute(0, 2, 3, 1)
    c = h.shape[3]
    if c < c_store:
        h = torch.nn.functional.pad(h, (0, c_store - c))
    return h.contiguous()


def _nchw_view(y_nhwc, c):
    return y_nhwc.permute(0, 3, 1, 2)[:, :c]


def _workspace(nbytes):
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=_device())


def _kaiming_uniform(rng, shape, fan_in):
    """rng.uniform(-l, l, size=shape).astype(float32) drawn on the device from
    the generator's PCG64 position (nn.py:44-46); the host generator is then
    advanced past the draws, exactly as the reference's call leaves it."""
    limit = float(np.sqrt(6.0 / fan_in))
    count = int(np.prod(shape))
    st = rng.bit_generator.state
    if st["bit_generator"] != "PCG64":
        raise ValueError("Kaiming init needs a PCG64-backed numpy Generator")
    out = torch.empty(count, dtype=torch.float32, device=_device())
    native.pcg64_uniform(st["state"]["state"], st["state"]["inc"], 0, -limit, limit, out.data_ptr(), count, _stream())
    rng.bit_generator.advance(count)
    return out.view(*shape)


class Layer:
    """Base class: parameter-free by default (nn.py:22-41)."""

    def __init__(self):
        self.params = {}
        self.grads = {}
        self._vel = {}

    def forward(self, x):
        raise NotImplementedError

    def backward(self, grad_out):
        raise NotImplementedError

    def output_shape(self, in_shape):
        raise NotImplementedError


class Conv2d(Layer):
    """Valid-mode cross-correlation with per-output-channel bias (nn.py:49-116)."""

    def __init__(self, in_channels, out_channels, kernel, stride=1, rng=None, dtype=np.float32):
        super().__init__()
        if kernel < 1 or stride < 1:
            raise ValueError(f"kernel and stride must be >= 1, got k={kernel} s={stride}")
        self.in_channels, self.out_channels = in_channels, out_channels
        self.kernel, self.stride = kernel, stride
        self.precision = precision_of(dtype)
        self.dtype = np.dtype(np.float32)  # parameters are fp32 masters in both modes
        rng = rng or np.random.default_rng(0)
        fan_in = in_channels * kernel * kernel
        self.params["w"] = _kaiming_uniform(rng, (out_channels, in_channels, kernel, kernel), fan_in)
        self.params["b"] = torch.zeros(out_channels, dtype=torch.float32, device=_device())
        self._x = None
        self._desc = None

    def output_shape(self, in_shape):
        c, h, w = in_shape
        if c != self.in_channels:
            raise ShapeError(f"conv expects {self.in_channels} input channels, got {c}", dimension="channels")
        k, s = self.kernel, self.stride
        if h < k or w < k:
            raise ShapeError(f"conv kernel {k} exceeds input {h}x{w}", dimension="rows" if h < k else "cols")
        return (self.out_channels, _out_dim(h, k, s), _out_dim(w, k, s))

    def _stores(self):
        return _pad8(self.in_channels), _pad8(self.out_channels)

    def _kernel_weight(self):
        """(o, c, k, k) fp32 master -> device layout [o_store][k][k][c_store]."""
        cs, os_ = self._stores()
        w = self.params["w"].permute(0, 2, 3, 1)
        w = torch.nn.functional.pad(w, (0, cs - self.in_channels, 0, 0, 0, 0, 0, os_ - self.out_channels))
        return w.to(_act_dtype(self.precision)).contiguous()

    def _bias(self):
        _, os_ = self._stores()
        return torch.nn.functional.pad(self.params["b"].float(), (0, os_ - self.out_channels)).contiguous()

    def forward(self, x):
        n, c, h, w = x.shape
        _, oh, ow = self.output_shape((c, h, w))
        cs, os_ = self._stores()
        dt = _act_dtype(self.precision)
        xs = _to_nhwc(x, cs, dt)
        self._desc = native.conv_desc(n, cs, h, w, os_, self.kernel, self.stride, self.precision)
        y = torch.empty(n, oh, ow, os_, dtype=dt, device=xs.device)
        # operands stay referenced across the call: a temporary freed before the
        # launch could be handed to the next allocation by the caching allocator
        wk, bias = self._kernel_weight(), self._bias()
        native.conv_fwd(self._desc, xs.data_ptr(), wk.data_ptr(), bias.data_ptr(), 0, y.data_ptr(), _stream())
        self._x = xs
        return _nchw_view(y, self.out_channels)

    def backward(self, grad_out):
        xs = self._x
        n, h, w, _ = xs.shape
        k, s = self.kernel, self.stride
        expect = (n, self.out_channels, _out_dim(h, k, s), _out_dim(w, k, s))
        if tuple(grad_out.shape) != expect:
            raise ShapeError(f"conv grad shape {tuple(grad_out.shape)}, expected {expect}")
        cs, os_ = self._stores()
        dt = _act_dtype(self.precision)
        dy = _to_nhwc(grad_out, os_, dt)
        ws = _workspace(native.conv_workspace_bytes(self._desc))
        dw = torch.empty(os_, k, k, cs, dtype=torch.float32, device=xs.device)
        db = torch.empty(os_, dtype=torch.float32, device=xs.device)
        native.conv_wgrad(self._desc, xs.data_ptr(), dy.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(),
                          ws.numel(), _stream())
        dx = torch.empty(n, h, w, cs, dtype=dt, device=xs.device)
        wk = self._kernel_weight()
        native.conv_dgrad(self._desc, dy.data_ptr(), wk.data_ptr(), None, dx.data_ptr(), ws.data_ptr(), ws.numel(),
                          _stream())
        self.grads["w"] = dw[:self.out_channels, :, :, :self.in_channels].permute(0, 3, 1, 2).contiguous()
        self.grads["b"] = db[:self.out_channels].contiguous()
        return _nchw_view(dx, self.in_channels)


class MaxPool(Layer):
    """Max pooling; ties go to the first window element in row-major order (nn.py:119-167)."""

    def __init__(self, size, stride=None, dtype=None):
        super().__init__()
        if size < 1:
            raise ValueError(f"pool size must be >= 1, got {size}")
        self.size = size
        self.stride = stride if stride is not None else size
        # like the reference (dtype follows the input), unless pinned
        self.precision = None if dtype is None else precision_of(dtype)
        self._arg = None
        self._in_shape = None
        self._desc = None

    def output_shape(self, in_shape):
        c, h, w = in_shape
        if h < self.size or w < self.size:
            raise ShapeError(f"pool window {self.size} exceeds input {h}x{w}",
                             dimension="rows" if h < self.size else "cols")
        return (c, _out_dim(h, self.size, self.stride), _out_dim(w, self.size, self.stride))

    def forward(self, x):
        n, c, h, w = x.shape
        _, oh, ow = self.output_shape((c, h, w))
        cs = _pad8(c)
        prec = self.precision or ("bf16" if x.dtype == torch.bfloat16 else "fp32")
        dt = _act_dtype(prec)
        xs = _to_nhwc(x, cs, dt)
        self._desc = native.conv_desc(n, cs, h, w, cs, self.size, self.stride, prec)
        y = torch.empty(n, oh, ow, cs, dtype=dt, device=xs.device)
        self._arg = torch.empty(n, oh, ow, cs, dtype=torch.uint8, device=xs.device)
        native.maxpool_fwd(self._desc, xs.data_ptr(), y.data_ptr(), self._arg.data_ptr(), _stream())
        self._in_shape = (n, c, h, w)
        return _nchw_view(y, c)

    @property
    def argmax_indices(self):
        """Window-relative argmax i*size+j per output element (NCHW, int64)."""
        if self._arg is None:
            return None
        return _nchw_view(self._arg, self._in_shape[1]).to(torch.int64)

    def backward(self, grad_out):
        if self._arg is None:
            raise ShapeError(f"pool grad shape {tuple(grad_out.shape)} does not match forward output")
        n, c, h, w = self._in_shape
        expect = (n, c, self._arg.shape[1], self._arg.shape[2])
        if tuple(grad_out.shape) != expect:
            raise ShapeError(f"pool grad shape {tuple(grad_out.shape)} does not match forward output")
        cs = self._arg.shape[3]
        dt = _act_dtype("bf16" if self._desc.precision == native.PREC_BF16 else "fp32")
        dy = _to_nhwc(grad_out, cs, dt)
        dx = torch.empty(n, h, w, cs, dtype=dt, device=dy.device)
        native.maxpool_bwd(self._desc, dy.data_ptr(), self._arg.data_ptr(), None, dx.data_ptr(), _stream())
        return _nchw_view(dx, c)


class ReLU(Layer):
    """max(x, 0) with the (x > 0) mask kept for backward (nn.py:170-183)."""

    def __init__(self):
        super().__init__()
        self._mask = None

    def output_shape(self, in_shape):
        return in_shape

    def forward(self, x):
        x = _as_tensor(x).contiguous()
        if x.dtype not in (torch.bfloat16, torch.float32):
            x = x.float()
        y = torch.empty_like(x)
        self._mask = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
        native.relu_fwd(x.data_ptr(), x.numel(), _precision_of(x), y.data_ptr(), self._mask.data_ptr(), _stream())
        return y

    def backward(self, grad_out):
        g = _as_tensor(grad_out).contiguous()
        if g.dtype not in (torch.bfloat16, torch.float32):
            g = g.float()
        if g.shape != self._mask.shape:
            raise ShapeError(f"relu backward: grad shape {tuple(g.shape)} != {tuple(self._mask.shape)}")
        dx = torch.empty_like(g)
        native.relu_bwd(g.data_ptr(), self._mask.data_ptr(), g.numel(), _precision_of(g), dx.data_ptr(), _stream())
        return dx


class Flatten(Layer):
    """(n, c, h, w) -> (n, c*h*w) in (c, h, w) order (nn.py:186-202)."""

    def __init__(self):
        super().__init__()
        self._shape = None

    def output_shape(self, in_shape):
        units = 1
        for d in in_shape:
            units *= d
        return (units,)

    def forward(self, x):
        x = _as_tensor(x)
        self._shape = tuple(x.shape)
        return x.reshape(x.shape[0], -1)

    def backward(self, grad_out):
        return grad_out.reshape(self._shape)


class Dense(Layer):
    """out = x @ W.T + b with W stored (out_units, in_units) (nn.py:205-240)."""

    def __init__(self, in_units, out_units, rng=None, dtype=np.float32):
        super().__init__()
        self.in_units, self.out_units = in_units, out_units
        self.precision = precision_of(dtype)
        self.dtype = np.dtype(np.float32)
        rng = rng or np.random.default_rng(0)
        self.params["w"] = _kaiming_uniform(rng, (out_units, in_units), in_units)
        self.params["b"] = torch.zeros(out_units, dtype=torch.float32, device=_device())
        self._x = None

    def output_shape(self, in_shape):
        if len(in_shape) != 1 or in_shape[0] != self.in_units:
            raise ShapeError(f"dense expects {self.in_units} input units, got {in_shape}", dimension="units")
        return (self.out_units,)

    def _desc(self, n):
        return native.dense_desc(n, self.in_units, self.out_units, self.precision)

    def _w16(self):
        pad = _pad8(self.in_units) - self.in_units
        return torch.nn.functional.pad(self.params["w"], (0, pad)).to(torch.bfloat16).contiguous()

    def _input(self, x):
        if self.precision == "bf16":
            x = _as_tensor(x, torch.bfloat16)
            return torch.nn.functional.pad(x, (0, _pad8(self.in_units) - self.in_units)).contiguous()
        return _as_tensor(x, torch.float32).contiguous()

    def forward(self, x):
        if x.ndim != 2 or x.shape[1] != self.in_units:
            raise ShapeError(f"dense expects (n, {self.in_units}) input, got {tuple(x.shape)}", dimension="units")
        n = x.shape[0]
        xs = self._input(x)
        d = self._desc(n)
        ws = _workspace(native.dense_workspace_bytes(d))
        y = torch.empty(n, self.out_units, dtype=torch.float32, device=xs.device)
        w16 = self._w16() if self.precision == "bf16" else None
        native.dense_fwd(d, xs.data_ptr(), self.params["w"].data_ptr(), _ptr(w16), self.params["b"].data_ptr(),
                         y.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
        self._x = xs
        return y

    def backward(self, grad_out):
        n = self._x.shape[0]
        if tuple(grad_out.shape) != (n, self.out_units):
            raise ShapeError(f"dense grad shape {tuple(grad_out.shape)}, expected ({n}, {self.out_units})")
        dy = _as_tensor(grad_out, torch.float32).contiguous()
        d = self._desc(n)
        ws = _workspace(native.dense_workspace_bytes(d))
        dt = _act_dtype(self.precision)
        dx = torch.empty(n, self.in_units, dtype=dt, device=dy.device)
        dw = torch.empty(self.out_units, self.in_units, dtype=torch.float32, device=dy.device)
        db = torch.empty(self.out_units, dtype=torch.float32, device=dy.device)
        w16 = self._w16() if self.precision == "bf16" else None
        native.dense_bwd(d, self._x.data_ptr(), dy.data_ptr(), self.params["w"].data_ptr(), _ptr(w16),
                         self.params["b"].data_ptr(), dx.data_ptr(), None, dw.data_ptr(), db.data_ptr(), None,
                         ws.data_ptr(), ws.numel(), _stream())
        self.grads["w"], self.grads["b"] = dw, db
        return dx


class Network:
    """An ordered layer stack ending in a Dense classifier head (nn.py:243-284)."""

    def __init__(self, layers, input_shape=None, class_count=2):
        if not layers or not isinstance(layers[-1], Dense):
            raise ValueError("network must end in a Dense layer")
        if layers[-1].out_units != class_count:
            raise ValueError(f"final Dense has {layers[-1].out_units} units, expected class_count={class_count}")
        self.layers = list(layers)
        self.input_shape = input_shape
        self.class_count = class_count

    @property
    def dtype(self):
        return np.dtype(np.float32)

    def forward(self, x):
        x = _as_tensor(x)
        if self.input_shape is not None and x.ndim == 4:
            if tuple(x.shape[1:]) != tuple(self.input_shape):
                raise ShapeError(f"network expects input {tuple(self.input_shape)}, got {tuple(x.shape[1:])}")
        for layer in self.layers:
            x = layer.forward(x)
        return x

    def backward(self, grad_logits):
        g = grad_logits
        for layer in reversed(self.layers):
            g = layer.backward(g)
        return g

    def parameters(self):
        """Yield (layer_index, name, tensor) with names sorted (b before w)."""
        for li, layer in enumerate(self.layers):
            for name in sorted(layer.params):
                yield li, name, layer.params[name]


def softmax_cross_entropy(logits, labels):
    """Mean cross-entropy and its gradient w.r.t. the logits (nn.py:287-303)."""
    logits = _as_tensor(logits, torch.float32).contiguous()
    n, k = logits.shape
    lab = _as_tensor(np.asarray(labels) if not torch.is_tensor(labels) else labels, torch.int64).contiguous()
    if int(lab.min()) < 0 or int(lab.max()) >= k:
        raise ValueError(f"labels must lie in [0, {k - 1}]")
    loss = torch.empty(1, dtype=torch.float32, device=logits.device)
    grad = torch.empty_like(logits)
    native.softmax_xent(logits.data_ptr(), lab.data_ptr(), n, k, loss.data_ptr(), grad.data_ptr(), _stream())
    return float(loss.item()), grad


def sgd_step(network, lr, momentum=0.0):
    """Classical momentum: v <- momentum*v - lr*g; w <- w + v (nn.py:306-322), in place."""
    if lr <= 0:
        raise ValueError(f"lr must be positive, got {lr}")
    if not 0.0 <= momentum < 1.0:
        raise ValueError(f"momentum must lie in [0, 1), got {momentum}")
    for layer in network.layers:
        for name, w in layer.params.items():
            g = layer.grads.get(name)
            if g is None:
                continue
            v = layer._vel.get(name)
            if v is None:
                v = torch.zeros_like(w)
                layer._vel[name] = v
            g = g.contiguous()
            native.sgd_momentum(w.data_ptr(), v.data_ptr(), g.data_ptr(), w.numel(), float(lr), float(momentum),
                                _stream())


def train_batch(network, batch, labels, lr, momentum=0.0):
    """One forward/backward/update step; returns the pre-step loss (nn.py:325-331)."""
    logits = network.forward(batch)
    loss, grad = softmax_cross_entropy(logits, labels)
    network.backward(grad)
    sgd_step(network, lr, momentum)
    return loss


def infer_shapes(layers, input_shape):
    """Per-layer output shapes for a single sample; raises ShapeError (nn.py:370-380)."""
    shape = tuple(input_shape)
    trace = []
    for idx, layer in enumerate(layers):
        try:
            shape = layer.output_shape(shape)
        except ShapeError as e:
            raise ShapeError(str(e), layer_index=idx, dimension=e.dimension) from None
        trace.append(shape)
    return trace
