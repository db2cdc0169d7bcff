"""MNDL model files (convevo/model_io.py:1-152), byte-compatible.

Container (little-endian): b"MNDL", u32 version (1), u32 layer count, then
per layer a u8 tag (1 Conv2d, 2 MaxPool, 3 ReLU, 4 Flatten, 5 Dense), its u32
hyper-parameters (Conv2d: in, out, kernel, stride; MaxPool: size, stride;
Dense: in, out) and, for Conv2d / Dense, the weight then bias tensors as
u32 ndim, u32 dims, float32 data. Weights round-trip bit-exactly; errors
raise FormatError with the byte offset (model_io.py:70-152).

Three views of the same file:
  read_mndl / write_mndl     host-only layer specs (numpy), no device needed
  load_network / save_network  the operator-level drop-in (nn.Network on the
                             B200), same signatures as the reference; save also
                             accepts a candidate network (network.Network)
  load_candidate             the fast candidate runtime (ce_predict /
                             ce_predict_stream) for predict_cmd
"""

import struct

import numpy as np

from .faults import FormatError

MAGIC = b"MNDL"
VERSION = 1
TAG_CONV, TAG_POOL, TAG_RELU, TAG_FLATTEN, TAG_DENSE = 1, 2, 3, 4, 5


# ------------------------------------------------------------------ host container
def _pack_tensor(arr):
    arr = np.ascontiguousarray(arr, dtype="<f4")
    return struct.pack("<I", arr.ndim) + struct.pack(f"<{arr.ndim}I", *arr.shape) + arr.tobytes()


def encode_mndl(specs):
    """specs: [("conv", cin, cout, k, s, w, b) | ("pool", size, stride) | ("relu",) |
    ("flatten",) | ("dense", in, out, w, b)] -> bytes."""
    chunks = [MAGIC, struct.pack("<II", VERSION, len(specs))]
    for sp in specs:
        kind = sp[0]
        if kind == "conv":
            _, cin, cout, k, s, w, b = sp
            chunks += [struct.pack("<BIIII", TAG_CONV, cin, cout, k, s), _pack_tensor(w), _pack_tensor(b)]
        elif kind == "pool":
            chunks.append(struct.pack("<BII", TAG_POOL, sp[1], sp[2]))
        elif kind == "relu":
            chunks.append(struct.pack("<B", TAG_RELU))
        elif kind == "flatten":
            chunks.append(struct.pack("<B", TAG_FLATTEN))
        elif kind == "dense":
            _, n_in, n_out, w, b = sp
            chunks += [struct.pack("<BII", TAG_DENSE, n_in, n_out), _pack_tensor(w), _pack_tensor(b)]
        else:
            raise ValueError(f"cannot serialize layer type {kind!r}")
    return b"".join(chunks)


def write_mndl(specs, path):
    with open(path, "wb") as fh:
        fh.write(encode_mndl(specs))


class _Reader:
    def __init__(self, data):
        self.data, self.pos = data, 0

    def take(self, n, what):
        if self.pos + n > len(self.data):
            raise FormatError(f"truncated file while reading {what}: expected {n} bytes at offset {self.pos}, "
                              f"only {len(self.data) - self.pos} available", offset=self.pos)
        chunk = self.data[self.pos:self.pos + n]
        self.pos += n
        return chunk

    def u32(self, what):
        return struct.unpack("<I", self.take(4, what))[0]

    def u8(self, what):
        return self.take(1, what)[0]

    def tensor(self, what):
        ndim = self.u32(f"{what} ndim")
        if ndim > 8:
            raise FormatError(f"implausible tensor rank {ndim} for {what}", offset=self.pos - 4)
        shape = struct.unpack(f"<{ndim}I", self.take(4 * ndim, f"{what} dims"))
        count = int(np.prod(shape)) if ndim else 1
        return np.frombuffer(self.take(4 * count, f"{what} data"), dtype="<f4").reshape(shape).astype(np.float32)


def decode_mndl(data):
    """bytes -> layer specs (see encode_mndl); validation as model_io.py:104-152."""
    r = _Reader(data)
    if r.take(4, "magic") != MAGIC:
        raise FormatError("bad magic: not an MNDL model file", offset=0)
    version = r.u32("version")
    if version != VERSION:
        raise FormatError(f"unsupported format version {version}", offset=4)
    specs = []
    for i in range(r.u32("layer count")):
        tag = r.u8(f"layer {i} tag")
        if tag == TAG_CONV:
            cin, cout, k, s = (r.u32(n) for n in ("in_channels", "out_channels", "kernel", "stride"))
            w = r.tensor("conv weights")
            b = r.tensor("conv bias")
            if w.shape != (cout, cin, k, k):
                raise FormatError(f"conv weight shape {w.shape} does not match header ({cout}, {cin}, {k}, {k})",
                                  offset=r.pos)
            specs.append(("conv", cin, cout, k, s, w, b))
        elif tag == TAG_POOL:
            size = r.u32("pool size")
            specs.append(("pool", size, r.u32("pool stride")))
        elif tag == TAG_RELU:
            specs.append(("relu",))
        elif tag == TAG_FLATTEN:
            specs.append(("flatten",))
        elif tag == TAG_DENSE:
            n_in = r.u32("in_units")
            n_out = r.u32("out_units")
            specs.append(("dense", n_in, n_out, r.tensor("dense weights"), r.tensor("dense bias")))
        else:
            raise FormatError(f"unknown layer tag {tag}", offset=r.pos - 1)
    if r.pos != len(r.data):
        raise FormatError(f"{len(r.data) - r.pos} trailing bytes after last layer", offset=r.pos)
    return specs


def read_mndl(path):
    with open(path, "rb") as fh:
        return decode_mndl(fh.read())


# ------------------------------------------------------------------ network views
def _host(t):
    return t.detach().float().cpu().numpy() if hasattr(t, "detach") else np.asarray(t, np.float32)


def specs_of(network):
    """Layer specs of an nn.Network (operator API) or a candidate network.Network."""
    from . import nn
    from .network import ConvLayer, DenseLayer, PoolLayer
    specs = []
    if isinstance(network, nn.Network):
        for L in network.layers:
            if isinstance(L, nn.Conv2d):
                specs.append(("conv", L.in_channels, L.out_channels, L.kernel, L.stride,
                              _host(L.params["w"]), _host(L.params["b"])))
            elif isinstance(L, nn.MaxPool):
                specs.append(("pool", L.size, L.stride))
            elif isinstance(L, nn.ReLU):
                specs.append(("relu",))
            elif isinstance(L, nn.Flatten):
                specs.append(("flatten",))
            elif isinstance(L, nn.Dense):
                specs.append(("dense", L.in_units, L.out_units, _host(L.params["w"]), _host(L.params["b"])))
            else:
                raise ValueError(f"cannot serialize layer type {type(L).__name__}")
        return specs
    # candidate network: Conv2d (+ReLU) / MaxPool ..., Flatten, Dense ... (genome.py:316-335)
    if network._dev is not None:
        network.pull_weights()
    params = iter(network.weights)
    flattened = False
    for L in network.layers:
        if isinstance(L, ConvLayer):
            w, b = next(params)
            specs.append(("conv", L.in_channels, L.out_channels, L.kernel, L.stride, _host(w), _host(b)))
            if L.relu:
                specs.append(("relu",))
        elif isinstance(L, PoolLayer):
            specs.append(("pool", L.size, L.stride))
        elif isinstance(L, DenseLayer):
            if not flattened:
                specs.append(("flatten",))
                flattened = True
            w, b = next(params)
            specs.append(("dense", L.in_units, L.out_units, _host(w), _host(b)))
    return specs


def save_network(network, path):
    """Write an MNDL file (model_io.py:48-68)."""
    write_mndl(specs_of(network), path)


def load_network(path, dtype=np.float32, class_count=None):
    """MNDL -> nn.Network on the device (model_io.py:104-152): the trailing
    Dense defines class_count unless overridden."""
    from . import nn
    import torch
    specs = read_mndl(path)
    layers = []
    rng = np.random.default_rng(0)  # init draws are overwritten by the file's tensors
    for sp in specs:
        if sp[0] == "conv":
            _, cin, cout, k, s, w, b = sp
            L = nn.Conv2d(cin, cout, k, s, rng=rng, dtype=dtype)
            L.params["w"] = torch.from_numpy(w).cuda()
            L.params["b"] = torch.from_numpy(b).cuda()
        elif sp[0] == "pool":
            L = nn.MaxPool(sp[1], sp[2])
        elif sp[0] == "relu":
            L = nn.ReLU()
        elif sp[0] == "flatten":
            L = nn.Flatten()
        else:
            _, n_in, n_out, w, b = sp
            L = nn.Dense(n_in, n_out, rng=rng, dtype=dtype)
            L.params["w"] = torch.from_numpy(w).cuda()
            L.params["b"] = torch.from_numpy(b).cuda()
        layers.append(L)
    if class_count is None:
        if not layers or not isinstance(layers[-1], nn.Dense):
            raise FormatError("model does not end in a Dense layer", offset=None)
        class_count = layers[-1].out_units
    return nn.Network(layers, input_shape=None, class_count=class_count)


def genome_of_specs(specs, model_id="mndl"):
    """The genome an MNDL layer sequence encodes (Conv2d [+ReLU] / MaxPool
    features, Flatten, Dense heads, final Dense(classes)), for the candidate
    runtime. Learning parameters are irrelevant for inference."""
    from .genes import ConvGene, DenseGene, Genome, LearnParams, PoolGene
    feats, heads = [], []
    i = 0
    while i < len(specs) and specs[i][0] != "flatten":
        sp = specs[i]
        if sp[0] == "conv":
            relu = i + 1 < len(specs) and specs[i + 1][0] == "relu"
            feats.append(ConvGene(out_channels=sp[2], kernel=sp[3], stride=sp[4], relu=relu))
            i += 2 if relu else 1
            continue
        if sp[0] == "pool":
            feats.append(PoolGene(size=sp[1], stride=sp[2]))
        else:
            raise FormatError(f"layer {i} ({sp[0]}) is not expressible as a genome feature", offset=None)
        i += 1
    dense = [sp for sp in specs[i + 1:]]
    if not dense or any(sp[0] != "dense" for sp in dense):
        raise FormatError("candidate models are features, Flatten, then Dense layers only", offset=None)
    heads = [DenseGene(units=sp[2]) for sp in dense[:-1]]
    return Genome(id=model_id, parent_ids=(), feature_layers=tuple(feats), head_layers=tuple(heads),
                  learn=LearnParams(lr=1e-3, momentum=0.0, batch_size=64))


def load_candidate(path, input_shape, model_id="mndl"):
    """MNDL -> candidate network.Network (weights set, not yet on a device)."""
    from .network import Network, build_layers
    specs = read_mndl(path)
    genome = genome_of_specs(specs, model_id)
    layers = build_layers(genome, tuple(input_shape))
    weights = [(sp[5], sp[6]) if sp[0] == "conv" else (sp[3], sp[4]) for sp in specs if sp[0] in ("conv", "dense")]
    if layers[-1].out_units != weights[-1][0].shape[0]:
        raise FormatError("final Dense does not match the candidate's class count", offset=None)
    plain = [L for L in layers if not hasattr(L, "size")]  # conv + dense, in order
    if len(plain) != len(weights):
        raise FormatError("parameter layers do not match the layer sequence", offset=None)
    for L, (w, _) in zip(plain, weights):
        want = ((L.out_channels, L.in_channels, L.kernel, L.kernel) if hasattr(L, "kernel")
                else (L.out_units, L.in_units))
        if tuple(w.shape) != want:
            raise FormatError(f"weights {tuple(w.shape)} do not fit input {tuple(input_shape)} (expected {want})",
                              offset=None)
    return Network(genome, input_shape, layers, weights, class_count=layers[-1].out_units)
