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


def _kaiming(rng, shape, fan_in, dtype, chunk=1 << 26):
    """rng.uniform(-l, l, size=shape).astype(dtype), drawn in chunks so giant
    heads never materialise a float64 copy (same stream, same values)."""
    limit = np.sqrt(6.0 / fan_in)
    total = int(np.prod(shape))
    out = np.empty(total, dtype=dtype)
    for start in range(0, total, chunk):
        stop = min(total, start + chunk)
        out[start:stop] = rng.uniform(-limit, limit, size=stop - start)
    return out.reshape(shape)


class Network:
    """Host description of an instantiated genome plus its device instance."""

    def __init__(self, genome, input_shape, layers, weights, class_count=2):
        self.genome = genome
        self.input_shape = tuple(input_shape)
        self.layers = layers            # ConvLayer / PoolLayer / DenseLayer in execution order
        self.weights = weights          # [(W, b)] reference layout, parameterised layers in order
        self.class_count = class_count
        self._dev = None
        self._dev_key = None

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


def instantiate(genome, input_shape, seed, dtype=np.float32):
    """Build the network for `genome` with seeded Kaiming-uniform weights."""
    layers = build_layers(genome, tuple(input_shape))
    rng = np.random.default_rng(seed)
    weights = []
    for layer in layers:
        if isinstance(layer, ConvLayer):
            fan_in = layer.in_channels * layer.kernel ** 2
            w = _kaiming(rng, (layer.out_channels, layer.in_channels, layer.kernel, layer.kernel), fan_in, dtype)
            weights.append((w, np.zeros(layer.out_channels, dtype=dtype)))
        elif isinstance(layer, DenseLayer):
            w = _kaiming(rng, (layer.out_units, layer.in_units), layer.in_units, dtype)
            weights.append((w, np.zeros(layer.out_units, dtype=dtype)))
    return Network(genome, input_shape, layers, weights)
