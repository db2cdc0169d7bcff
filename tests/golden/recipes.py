"""Deterministic input recipes shared by make_golden.py (which runs the
reference) and the tests (which rebuild the same inputs instead of storing
them): only reference OUTPUTS are committed."""

import numpy as np


def conv_shapes():
    rng = np.random.default_rng(1234)
    shapes = []
    for _ in range(40):
        cin = int(rng.choice([3, 8, 16, 32]))
        cout = int(rng.choice([8, 16, 32, 64]))
        k = int(rng.integers(1, 8))
        s = int(rng.integers(1, 4))
        h = int(rng.integers(k, k + 14))
        shapes.append((cin, cout, k, s, h))
    shapes += [(3, 32, 4, 2, 40), (32, 64, 4, 1, 21), (64, 128, 4, 1, 13)]  # FIXED layer kinds, reduced extent
    return shapes


def conv_dtypes(ci):
    return (np.float32, np.float64) if ci % 4 == 0 else (np.float32,)


def conv_inputs(ci, shape, dt):
    """(x, w, b, gy_shape_fn): w from the reference Conv2d init with rng seed ci."""
    cin, cout, k, s, h = shape
    n = 2 if h > 30 else 3
    x = np.random.default_rng(ci + 99).standard_normal((n, cin, h, h)).astype(dt)
    b = np.random.default_rng(ci + 7).uniform(-0.1, 0.1, cout).astype(dt)
    lim = np.sqrt(6.0 / (cin * k * k))
    w = np.random.default_rng(ci).uniform(-lim, lim, size=(cout, cin, k, k)).astype(dt)
    oh = (h - k) // s + 1
    gy = np.random.default_rng(ci + 5).standard_normal((n, cout, oh, oh)).astype(dt)
    return x, w, b, gy


def pool_input(size, stride, variant):
    r = np.random.default_rng(size * 10 + stride)
    if variant == "rand":
        x = r.standard_normal((2, 3, 11, 13)).astype(np.float32)
    elif variant == "ties":
        x = r.integers(0, 3, size=(2, 3, 11, 13)).astype(np.float32)
    else:
        x = np.full((2, 3, 11, 13), 0.5, np.float32)
    oh, ow = (11 - size) // stride + 1, (13 - size) // stride + 1
    gy = r.standard_normal((2, 3, oh, ow)).astype(np.float32)
    return x, gy


DENSE_SHAPES = [(4096, 64, 4), (64, 2, 16), (300, 17, 5)]


def dense_inputs(di):
    nin, nout, n = DENSE_SHAPES[di]
    r = np.random.default_rng(di)
    lim = np.sqrt(6.0 / nin)
    w = r.uniform(-lim, lim, size=(nout, nin)).astype(np.float32)
    b = r.uniform(-0.1, 0.1, nout).astype(np.float32)
    x = r.standard_normal((n, nin)).astype(np.float32)
    gy = r.standard_normal((n, nout)).astype(np.float32)
    return x, w, b, gy
