"""ctypes binding of libmenndl_sm100.so (include/menndl_sm100.h).

ctypes releases the GIL for the duration of each foreign call, so worker
threads driving different nets (different GPUs / streams) run concurrently.
There is no fallback: if the library is missing the import of this module
fails loudly (build it with paper_1909_12291_b200.build).
"""

import ctypes as C
import os
import threading

import numpy as np

from . import build as _build
from .faults import CE_OK, status_to_exception

LAYER_CONV, LAYER_POOL, LAYER_DENSE = 1, 2, 3
PREC_BF16, PREC_FP32 = 0, 1
PRECISIONS = {"bf16": PREC_BF16, "fp32": PREC_FP32}


class LayerDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("out_channels", C.c_int), ("kernel", C.c_int),
                ("stride", C.c_int), ("relu", C.c_int), ("units", C.c_int)]


class NetDesc(C.Structure):
    _fields_ = [("in_c", C.c_int), ("in_h", C.c_int), ("in_w", C.c_int), ("n_layers", C.c_int),
                ("layers", C.POINTER(LayerDesc)), ("max_batch", C.c_int)]


class ConvDesc(C.Structure):
    _fields_ = [("n", C.c_int), ("c", C.c_int), ("h", C.c_int), ("w", C.c_int), ("c_out", C.c_int),
                ("kernel", C.c_int), ("stride", C.c_int), ("precision", C.c_int)]


class DenseDesc(C.Structure):
    _fields_ = [("n", C.c_int), ("in_units", C.c_int), ("out_units", C.c_int), ("precision", C.c_int)]


class SgdArgs(C.Structure):
    _fields_ = [("lr", C.c_float), ("momentum", C.c_float), ("vel_w", C.c_void_p), ("vel_b", C.c_void_p)]


_P = C.c_void_p
_F = C.POINTER(C.c_float)
_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)
_U8 = C.POINTER(C.c_uint8)

_SIGNATURES = {
    "ce_version": ([], C.c_int),
    "ce_last_error": ([], C.c_char_p),
    "ce_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "ce_dataset_create": ([C.c_int, _U8, _U8, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_P)], C.c_int),
    "ce_dataset_destroy": ([_P], C.c_int),
    "ce_net_create": ([C.POINTER(NetDesc), C.c_int, C.c_int, C.POINTER(_P)], C.c_int),
    "ce_net_destroy": ([_P], C.c_int),
    "ce_net_device_bytes": ([_P, C.POINTER(C.c_size_t)], C.c_int),
    "ce_net_set_priority": ([_P, C.c_int], C.c_int),
    "ce_net_num_param_layers": ([_P, C.POINTER(C.c_int)], C.c_int),
    "ce_net_set_params": ([_P, C.c_int, _F, _F], C.c_int),
    "ce_net_get_params": ([_P, C.c_int, _F, _F, _F, _F], C.c_int),
    "ce_net_init_uniform": ([_P, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double], C.c_int),
    "ce_net_keep_grads": ([_P, C.c_int], C.c_int),
    "ce_net_get_grads": ([_P, C.c_int, _F, _F], C.c_int),
    "ce_net_forward_host": ([_P, _F, C.c_int, _F], C.c_int),
    "ce_net_get_activation": ([_P, C.c_int, C.c_int, _F], C.c_int),
    "ce_net_layer_materialized": ([_P, C.c_int, C.POINTER(C.c_int)], C.c_int),
    "ce_net_train_batch_host": ([_P, _F, _I64, C.c_int, C.c_float, C.c_float, _F], C.c_int),
    "ce_train": ([_P, _P, _I32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_float, _F, _D], C.c_int),
    "ce_predict": ([_P, _P, C.c_int, _D, _I64], C.c_int),
    "ce_latency": ([_P, _F, C.c_int, C.c_int, C.c_int, _D], C.c_int),
    "ce_predict_stream": ([_P, _U8, C.c_longlong, C.c_int, _D, _I64, _D], C.c_int),
    "ce_conv_workspace_bytes": ([C.POINTER(ConvDesc)], C.c_size_t),
    "ce_conv_fwd": ([C.POINTER(ConvDesc), _P, _P, _P, C.c_int, C.c_int, C.c_int, _P, _P, _P], C.c_int),
    "ce_conv_dgrad": ([C.POINTER(ConvDesc), _P, _P, _P, _P, _P, C.c_size_t, _P], C.c_int),
    "ce_conv_wgrad": ([C.POINTER(ConvDesc), _P, _P, _P, _P, _P, C.c_size_t, _P], C.c_int),
    "ce_maxpool_fwd": ([C.POINTER(ConvDesc), _P, _P, _P, _P], C.c_int),
    "ce_maxpool_bwd": ([C.POINTER(ConvDesc), _P, _P, _P, _P, _P], C.c_int),
    "ce_gather_u8_normalize": ([_P, C.c_int, C.c_int, C.c_int, _P, C.c_int, C.c_int, C.c_int, _P, _P], C.c_int),
    "ce_dense_workspace_bytes": ([C.POINTER(DenseDesc)], C.c_size_t),
    "ce_dense_fwd": ([C.POINTER(DenseDesc), _P, _P, _P, _P, _P, _P, C.c_size_t, _P], C.c_int),
    "ce_dense_bwd": ([C.POINTER(DenseDesc), _P, _P, _P, _P, _P, _P, _P, _P, _P, C.POINTER(SgdArgs), _P,
                      C.c_size_t, _P], C.c_int),
    "ce_softmax_xent": ([_P, _P, C.c_int, C.c_int, _P, _P, _P], C.c_int),
    "ce_sgd_momentum": ([_P, _P, _P, C.c_size_t, C.c_float, C.c_float, _P], C.c_int),
    "ce_relu_fwd": ([_P, C.c_size_t, C.c_int, _P, _P, _P], C.c_int),
    "ce_relu_bwd": ([_P, _P, C.c_size_t, C.c_int, _P, _P], C.c_int),
    "ce_pcg64_uniform": ([C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_double, _P,
                          C.c_size_t, _P], C.c_int),
    "ce_permute_flatten_weights": ([_P, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P], C.c_int),
    "ce_launch_count": ([], C.c_longlong),
    "ce_prof_num_classes": ([], C.c_int),
    "ce_net_set_profiling": ([_P, C.c_int], C.c_int),
    "ce_net_prof_read": ([_P, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_longlong), _D, _D, _D], C.c_int),
    "ce_prof_set_peaks": ([C.c_double, C.c_double], C.c_int),
    "ce_net_prof_ideal": ([_P, C.c_int, _D], C.c_int),
    "ce_net_prof_layer": ([_P, C.c_int, C.c_int, C.POINTER(C.c_longlong), _D, _D, _D, _D], C.c_int),
}
EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


def library_path():
    # CE_LIB=trace: the -DCE_TC_TRACE debug build (tools/tc_trace.py), never the product
    variant = os.environ.get("CE_LIB")
    if variant == "trace":
        return _build.TRACE_LIB_PATH
    if variant:  # experiment builds: lib/libmenndl_sm100_<variant>.so (never the product)
        return os.path.join(os.path.dirname(_build.LIB_PATH), f"libmenndl_sm100_{variant}.so")
    return _build.LIB_PATH


def load(build_if_missing=True):
    """Load (building first if needed) and return the CDLL."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if path != _build.LIB_PATH:
            if not os.path.exists(path):
                raise OSError(f"{path} missing (experiment build)")
        elif not os.path.exists(path) or (build_if_missing and not _build.up_to_date()):
            if not build_if_missing:
                raise OSError(f"{path} missing; run python -m paper_1909_12291_b200.build")
            _build.build()
        lib = C.CDLL(path)
        for name, (argtypes, restype) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes, fn.restype = argtypes, restype
        _lib = lib
        return lib


def check(status):
    if status != CE_OK:
        msg = load().ce_last_error().decode(errors="replace")
        raise status_to_exception(status, msg)


def fptr(a):
    return a.ctypes.data_as(_F) if a is not None else None


def conv_desc(n, c, h, w, c_out, kernel, stride, precision):
    return ConvDesc(n, c, h, w, c_out, kernel, stride, PRECISIONS[precision])


def conv_workspace_bytes(desc):
    return int(load().ce_conv_workspace_bytes(C.byref(desc)))


def conv_fwd(desc, x, w, bias, relu, y, stream=0, pool=None, arg=None):
    """Kernel-level conv forward on device pointers (ints) of NHWC tensors.
    pool=(window, stride): max-pool epilogue, y/arg are the pooled map and its u8 argmax."""
    pk, ps = pool if pool else (0, 0)
    check(load().ce_conv_fwd(C.byref(desc), x, w, bias, int(relu), int(pk), int(ps), y, arg, stream))


def conv_dgrad(desc, dy, w, mask, dx, ws, ws_bytes, stream=0):
    check(load().ce_conv_dgrad(C.byref(desc), dy, w, mask, dx, ws, ws_bytes, stream))


def conv_wgrad(desc, x, dy, dw, db, ws, ws_bytes, stream=0):
    check(load().ce_conv_wgrad(C.byref(desc), x, dy, dw, db, ws, ws_bytes, stream))


def maxpool_fwd(desc, x, y, arg, stream=0):
    check(load().ce_maxpool_fwd(C.byref(desc), x, y, arg, stream))


def maxpool_bwd(desc, dy, arg, mask, dx, stream=0):
    check(load().ce_maxpool_bwd(C.byref(desc), dy, arg, mask, dx, stream))


def gather_u8_normalize(pixels, c, h, w, idx, n, c_store, precision, out, stream=0):
    """Kernel-level batch gather + /255 normalise (device pointers)."""
    check(load().ce_gather_u8_normalize(pixels, c, h, w, idx, n, c_store, PRECISIONS[precision], out, stream))


def dense_desc(n, in_units, out_units, precision):
    return DenseDesc(n, in_units, out_units, PRECISIONS[precision])


def dense_workspace_bytes(desc):
    return int(load().ce_dense_workspace_bytes(C.byref(desc)))


def dense_fwd(desc, x, w, w16, b, y, ws, ws_bytes, stream=0):
    check(load().ce_dense_fwd(C.byref(desc), x, w, w16, b, y, ws, ws_bytes, stream))


def dense_bwd(desc, x, dy, w, w16, b, dx, mask, dw, db, sgd, ws, ws_bytes, stream=0):
    """sgd: None or (lr, momentum, vel_w_ptr, vel_b_ptr) for the fused update."""
    args = None if sgd is None else C.byref(SgdArgs(sgd[0], sgd[1], sgd[2], sgd[3]))
    check(load().ce_dense_bwd(C.byref(desc), x, dy, w, w16, b, dx, mask, dw, db, args, ws, ws_bytes, stream))


def softmax_xent(logits, labels, n, k, loss, grad, stream=0):
    check(load().ce_softmax_xent(logits, labels, n, k, loss, grad, stream))


def relu_fwd(x, count, precision, y, mask, stream=0):
    check(load().ce_relu_fwd(x, count, PRECISIONS[precision], y, mask, stream))


def relu_bwd(dy, mask, count, precision, dx, stream=0):
    check(load().ce_relu_bwd(dy, mask, count, PRECISIONS[precision], dx, stream))


def sgd_momentum(w, vel, g, count, lr, momentum, stream=0):
    check(load().ce_sgd_momentum(w, vel, g, count, lr, momentum, stream))


def pcg64_uniform(state, inc, skip, low, high, out, count, stream=0):
    """numpy PCG64(state, inc) advanced by `skip`, .uniform(low, high, count) as float32 into device `out`."""
    m = (1 << 64) - 1
    check(load().ce_pcg64_uniform(state >> 64, state & m, inc >> 64, inc & m, skip, low, high, out, count, stream))


def permute_flatten_weights(src, rows, c, c_store, hw, direction, dst, stream=0):
    check(load().ce_permute_flatten_weights(src, rows, c, c_store, hw, direction, dst, stream))


def set_prof_peaks(flops_per_s, bytes_per_s):
    """Peaks the profiler uses for each launch's roofline time max(F/P, B/BW)."""
    check(load().ce_prof_set_peaks(float(flops_per_s), float(bytes_per_s)))


def launch_count():
    return int(load().ce_launch_count())


def device_count():
    n = C.c_int(0)
    check(load().ce_device_count(C.byref(n)))
    return n.value


class Dataset:
    """A PatchSet resident on one device (u8 pixels + labels)."""

    def __init__(self, pset, device=0):
        lib = load()
        px = np.ascontiguousarray(pset.pixels, dtype=np.uint8)
        lab = np.ascontiguousarray(pset.labels, dtype=np.uint8)
        n, c, h, w = px.shape
        self.n, self.shape, self.device = n, (c, h, w), device
        self.labels = lab
        h_ = _P()
        check(lib.ce_dataset_create(device, px.ctypes.data_as(_U8), lab.ctypes.data_as(_U8), n, c, h, w,
                                    C.byref(h_)))
        self._h = h_

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            load().ce_dataset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_thread = threading.local()


class stream_priority:
    """Context: nets created by this thread get a high-priority stream (priority > 0)."""

    def __init__(self, priority):
        self.priority = priority

    def __enter__(self):
        self.prev = getattr(_thread, "priority", 0)
        _thread.priority = self.priority
        return self

    def __exit__(self, *exc):
        _thread.priority = self.prev


class Net:
    """Owning wrapper of a ce_net handle."""

    def __init__(self, layers, input_shape, max_batch, device=0, precision="bf16"):
        lib = load()
        arr = (LayerDesc * len(layers))()
        for i, spec in enumerate(layers):
            arr[i] = LayerDesc(*spec)
        c, h, w = input_shape
        desc = NetDesc(c, h, w, len(layers), arr, int(max_batch))
        h_ = _P()
        check(lib.ce_net_create(C.byref(desc), int(device), PRECISIONS[precision], C.byref(h_)))
        self._h = h_
        if getattr(_thread, "priority", 0) > 0:
            check(lib.ce_net_set_priority(h_, 1))
        self.device, self.precision, self.max_batch = device, precision, max_batch

    def close(self):
        if self._h:
            load().ce_net_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def device_bytes(self):
        n = C.c_size_t(0)
        check(load().ce_net_device_bytes(self._h, C.byref(n)))
        return n.value

    def set_params(self, p, w, b):
        w = np.ascontiguousarray(w, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        check(load().ce_net_set_params(self._h, p, fptr(w), fptr(b)))

    def init_uniform(self, p, state, inc, limit):
        """Device Kaiming init from a PCG64 (state, inc) pair (128-bit ints)."""
        m = (1 << 64) - 1
        check(load().ce_net_init_uniform(self._h, p, (state >> 64) & m, state & m, (inc >> 64) & m, inc & m,
                                         float(limit)))

    def get_params(self, p, w_shape, b_shape):
        w, b = np.empty(w_shape, np.float32), np.empty(b_shape, np.float32)
        vw, vb = np.empty(w_shape, np.float32), np.empty(b_shape, np.float32)
        check(load().ce_net_get_params(self._h, p, fptr(w), fptr(b), fptr(vw), fptr(vb)))
        return w, b, vw, vb

    def keep_grads(self, on=True):
        check(load().ce_net_keep_grads(self._h, int(bool(on))))

    def get_grads(self, p, w_shape, b_shape):
        gw, gb = np.empty(w_shape, np.float32), np.empty(b_shape, np.float32)
        check(load().ce_net_get_grads(self._h, p, fptr(gw), fptr(gb)))
        return gw, gb

    def forward(self, x, classes=2):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty((len(x), classes), np.float32)
        check(load().ce_net_forward_host(self._h, fptr(x), len(x), fptr(out)))
        return out

    def materialized(self, layer):
        """False for a conv whose max-pool runs in its epilogue (no pre-pool activation exists)."""
        yes = C.c_int(0)
        check(load().ce_net_layer_materialized(self._h, layer, C.byref(yes)))
        return bool(yes.value)

    def activation(self, layer, n, shape):
        out = np.empty((n, *shape), np.float32)
        check(load().ce_net_get_activation(self._h, layer, n, fptr(out)))
        return out

    def train_batch(self, x, labels, lr, momentum):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.ascontiguousarray(labels, dtype=np.int64)
        loss = np.zeros(1, np.float32)
        check(load().ce_net_train_batch_host(self._h, fptr(x), y.ctypes.data_as(_I64), len(x),
                                             float(lr), float(momentum), fptr(loss)))
        return float(loss[0])

    def train(self, dataset, perms, steps_per_epoch, batch, lr, momentum):
        perms = np.ascontiguousarray(perms, dtype=np.int32)
        epochs, n_perm = perms.shape
        losses = np.zeros(epochs * steps_per_epoch, np.float32)
        ms = C.c_double(0.0)
        check(load().ce_train(self._h, dataset.handle, perms.ctypes.data_as(_I32), n_perm, epochs,
                              steps_per_epoch, batch, float(lr), float(momentum), fptr(losses), C.byref(ms)))
        return losses, ms.value

    def predict(self, dataset, batch=128):
        scores = np.empty(dataset.n, np.float64)
        preds = np.empty(dataset.n, np.int64)
        check(load().ce_predict(self._h, dataset.handle, batch, scores.ctypes.data_as(_D),
                                preds.ctypes.data_as(_I64)))
        return scores, preds

    def predict_stream(self, pixels, batch=128):
        """Streamed predict over host u8 NCHW patches; returns (scores, preds, device seconds)."""
        n = len(pixels)
        scores = np.empty(n, np.float64)
        preds = np.empty(n, np.int64)
        secs = C.c_double(0.0)
        if isinstance(pixels, np.ndarray):
            px = np.ascontiguousarray(pixels, dtype=np.uint8)
            ptr = px.ctypes.data_as(_U8)
        else:  # a (pinned) torch uint8 tensor on the host
            px = pixels.contiguous()
            ptr = C.cast(px.data_ptr(), _U8)
        check(load().ce_predict_stream(self._h, ptr, n, batch, scores.ctypes.data_as(_D),
                                       preds.ctypes.data_as(_I64), C.byref(secs)))
        return scores, preds, secs.value

    def set_profiling(self, on):
        check(load().ce_net_set_profiling(self._h, int(bool(on))))

    def profile(self):
        """Per kernel class: {name: (launches, ms, flops, bytes, ideal_ms)} accumulated by ce_train;
        ideal_ms = sum over launches of max(flops / P, bytes / BW) (set_prof_peaks)."""
        lib, out = load(), {}
        for cls in range(lib.ce_prof_num_classes()):
            name, n = C.c_char_p(), C.c_longlong()
            ms, fl, by, ideal = C.c_double(), C.c_double(), C.c_double(), C.c_double()
            check(lib.ce_net_prof_read(self._h, cls, C.byref(name), C.byref(n), C.byref(ms), C.byref(fl),
                                       C.byref(by)))
            check(lib.ce_net_prof_ideal(self._h, cls, C.byref(ideal)))
            out[name.value.decode()] = (n.value, ms.value, fl.value, by.value, ideal.value)
        return out

    def profile_layers(self, n_layers):
        """{(layer, class): (launches, ms, flops, bytes, ideal_ms)} for every layer (and -1) with launches."""
        lib, out = load(), {}
        names = [c for c in self.profile()]
        for layer in range(-1, n_layers):
            for cls, name in enumerate(names):
                n = C.c_longlong()
                ms, fl, by, ideal = C.c_double(), C.c_double(), C.c_double(), C.c_double()
                check(lib.ce_net_prof_layer(self._h, layer, cls, C.byref(n), C.byref(ms), C.byref(fl), C.byref(by),
                                            C.byref(ideal)))
                if n.value:
                    out[(layer, name)] = (n.value, ms.value, fl.value, by.value, ideal.value)
        return out

    def latency(self, x, warmup, reps):
        x = np.ascontiguousarray(x, dtype=np.float32)
        secs = np.zeros(reps, np.float64)
        check(load().ce_latency(self._h, fptr(x), len(x), warmup, reps, secs.ctypes.data_as(_D)))
        return secs
