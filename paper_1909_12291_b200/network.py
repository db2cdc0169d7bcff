"""Genome -> network builder.

`instantiate` mirrors convevo/genome.py:309-335: it validates the shape trace,
draws every weight from one PCG64 stream `default_rng(seed)` in layer order
(conv_0, conv_1, ..., head dense, final Dense(2)) with the reference's
Kaiming-uniform rule (nn.py:44-46: U(-sqrt(6/fan_in), +sqrt(6/fan_in)) drawn
as float64 then cast), zero biases, and returns a Network. The Network keeps
the host-side description (layer list, FLOP/param accounting) and owns a
device instance (libmenndl_sm100 ce_net) created on demand.
"""

from dataclasses import dataclass

import numpy as np

from . import native
from .faults import ShapeError
from .genes import ConvGene, PoolGene, validate_shapes


@dataclass(frozen=True)
class ConvLayer:
    in_channels: int
    out_channels: int
    kernel: int
    stride: int
    relu: bool
    out_shape: tuple  # (c, h, w)


@dataclass(frozen=True)
class PoolLayer:
    size: int
    stride: int
    out_shape: tuple


@dataclass(frozen=True)
class DenseLayer:
    in_units: int
    out_units: int


def _kaiming(rng, shape, fan_in, dtype, chunk=1 << 26, limit=None):
    """rng.uniform(-l, l, size=shape).astype(dtype), drawn in chunks so giant
    heads never materialise a float64 copy (same stream, same values)."""
    if limit is None:
        limit = np.sqrt(6.0 / fan_in)
    total = int(np.prod(shape))
    out = np.empty(total, dtype=dtype)
    for start in range(0, total, chunk):
        stop = min(total, start + chunk)
        out[start:stop] = rng.uniform(-limit, limit, size=stop - start)
    return out.reshape(shape)


class Network:
    """Host description of an instantiated genome plus its device instance.

    Weights are "lazy" when built by instantiate(): only the PCG64 stream
    position of each layer is kept, the device draws the values itself
    (ce_net_init_uniform) and the host arrays are materialised on first access
    to `weights` (same values, bit for bit)."""

    def __init__(self, genome, input_shape, layers, weights, class_count=2, streams=None):
        self.genome = genome
        self.input_shape = tuple(input_shape)
        self.layers = layers            # ConvLayer / PoolLayer / DenseLayer in execution order
        self._weights = weights         # [(W, b)] reference layout, or None while lazy
        self.streams = streams          # [(state, inc, limit, shape, dtype)] per parameterised layer
        self.class_count = class_count
        self._dev = None
        self._dev_key = None

    @property
    def weights(self):
        if self._weights is None:
            self._weights = [_draw_layer(*st) for st in self.streams]
        return self._weights

    @weights.setter
    def weights(self, value):
        self._weights = value

    # -- accounting (evaluator.py:116-136) ---------------------------------
    def parameters(self):
        """(param_layer_index, name, array) with names sorted (b before w), nn.py:280-284."""
        for i, (w, b) in enumerate(self.weights):
            yield i, "b", b
            yield i, "w", w

    def param_count(self):
        total = 0
        for layer in self.layers:
            if isinstance(layer, ConvLayer):
                total += layer.out_channels * (layer.in_channels * layer.kernel ** 2 + 1)
            elif isinstance(layer, DenseLayer):
                total += layer.out_units * (layer.in_units + 1)
        return total

    def flops_inference(self):
        """conv 2k^2 c_in c_out h w; dense 2 in out; pool and ReLU = output elements."""
        total = 0
        for layer in self.layers:
            if isinstance(layer, ConvLayer):
                c, h, w = layer.out_shape
                total += 2 * layer.kernel ** 2 * layer.in_channels * c * h * w
                if layer.relu:
                    total += c * h * w
            elif isinstance(layer, PoolLayer):
                c, h, w = layer.out_shape
                total += c * h * w
            else:
                total += 2 * layer.in_units * layer.out_units
        return int(total)

    # -- device ---------------------------------------------------------------
    def native_layers(self):
        specs = []
        for layer in self.layers:
            if isinstance(layer, ConvLayer):
                specs.append((native.LAYER_CONV, layer.out_channels, layer.kernel, layer.stride, int(layer.relu), 0))
            elif isinstance(layer, PoolLayer):
                specs.append((native.LAYER_POOL, 0, layer.size, layer.stride, 0, 0))
            else:
                specs.append((native.LAYER_DENSE, 0, 0, 0, 0, layer.out_units))
        return specs

    def to_device(self, device=0, precision="bf16", max_batch=256):
        """Create (or reuse) the device instance and upload the current weights."""
        key = (device, precision, max_batch)
        if self._dev is not None and self._dev_key == key:
            return self._dev
        self.release()
        net = native.Net(self.native_layers(), self.input_shape, max_batch, device, precision)
        try:
            if self._weights is None:
                for p, (state, inc, limit, _, _) in enumerate(self.streams):
                    net.init_uniform(p, state, inc, limit)
            else:
                for p, (w, b) in enumerate(self.weights):
                    net.set_params(p, w, b)
        except Exception:
            net.close()
            raise
        self._dev, self._dev_key = net, key
        return net

    @property
    def device_net(self):
        if self._dev is None:
            raise RuntimeError("network has no device instance; call to_device()")
        return self._dev

    def pull_weights(self):
        """Copy device weights (and velocities) back into the host description."""
        out = []
        for p, (w, b) in enumerate(self.weights):
            nw, nb, vw, vb = self.device_net.get_params(p, w.shape, b.shape)
            out.append((nw, nb, vw, vb))
        self.weights = [(o[0], o[1]) for o in out]
        return out

    def release(self):
        if self._dev is not None:
            self._dev.close()
            self._dev = None
            self._dev_key = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def build_layers(genome, input_shape):
    trace = validate_shapes(genome, input_shape)
    c = input_shape[0]
    layers = []
    for gene, shape in zip(genome.feature_layers, trace.feature_shapes):
        if isinstance(gene, ConvGene):
            layers.append(ConvLayer(c, gene.out_channels, gene.kernel, gene.stride, bool(gene.relu), shape))
            c = gene.out_channels
        elif isinstance(gene, PoolGene):
            layers.append(PoolLayer(gene.size, gene.stride, shape))
        else:
            raise ShapeError(f"unknown gene {gene!r}")
    units = trace.flat_units
    for gene in genome.head_layers:
        layers.append(DenseLayer(units, gene.units))
        units = gene.units
    layers.append(DenseLayer(units, 2))
    return layers


def _draw_layer(state, inc, limit, shape, dtype):
    """Host draw of one layer's Kaiming weights from a recorded PCG64 position."""
    bg = np.random.PCG64()
    bg.state = {"bit_generator": "PCG64", "state": {"state": state, "inc": inc}, "has_uint32": 0, "uinteger": 0}
    rng = np.random.Generator(bg)
    w = _kaiming(rng, shape, None, dtype, limit=limit)
    return w, np.zeros(shape[0], dtype=dtype)


def instantiate(genome, input_shape, seed, dtype=np.float32, lazy=True):
    """Build the network for `genome` with seeded Kaiming-uniform weights.

    Draw order and values follow genome.py:309-335 / nn.py:44-46 exactly. With
    lazy=True the host only records where each layer's draws start in the
    PCG64 stream (and advances past them); the values are produced on the
    device, or on the host when `weights` is first read."""
    layers = build_layers(genome, tuple(input_shape))
    rng = np.random.default_rng(seed)
    streams = []
    for layer in layers:
        if isinstance(layer, ConvLayer):
            fan_in = layer.in_channels * layer.kernel ** 2
            shape = (layer.out_channels, layer.in_channels, layer.kernel, layer.kernel)
        elif isinstance(layer, DenseLayer):
            fan_in = layer.in_units
            shape = (layer.out_units, layer.in_units)
        else:
            continue
        st = rng.bit_generator.state["state"]
        streams.append((st["state"], st["inc"], float(np.sqrt(6.0 / fan_in)), shape, dtype))
        rng.bit_generator.advance(int(np.prod(shape)))
    net = Network(genome, input_shape, layers, None, streams=streams)
    if not lazy:
        net.weights  # materialise now
    return net
