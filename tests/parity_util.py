"""Shared helpers for parity tests: norm-wise relative error and the genome
cases exercised against the oracle."""

import numpy as np

from paper_1909_12291_b200.genes import FIXED, parse_genome


def rel(a, b):
    """Per-tensor ||a - b||_2 / ||b||_2 (elementwise is invalid)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b.ravel())
    num = np.linalg.norm((a - b).ravel())
    if den == 0.0:
        return num
    return num / den


# tolerance per precision for single-kernel tensors (T1) and one step (T2)
TOL = {"fp32": 1e-5, "bf16": 1e-2}

_BASE = "parents= lr=0.001 momentum=0.9 batch_size=8 "

# (name, genome text, input shape) — small inputs keep the CPU oracle fast
CASES = [
    ("fixed", FIXED, (3, 100, 100)),
    ("conv_relu_pool_dense", "id=case0000000001 " + _BASE +
     "f0=conv:oc=16,k=3,s=1,relu=1 f1=pool:size=2,s=2 f2=conv:oc=32,k=3,s=2,relu=1 h0=dense:units=24",
     (3, 32, 32)),
    ("pool_first_norelu", "id=case0000000002 " + _BASE +
     "f0=pool:size=3,s=2 f1=conv:oc=8,k=5,s=1,relu=0 f2=conv:oc=64,k=2,s=3,relu=1",
     (3, 40, 40)),
    ("overlap_pools", "id=case0000000003 " + _BASE +
     "f0=conv:oc=32,k=4,s=2,relu=1 f1=pool:size=3,s=1 f2=pool:size=2,s=1 f3=conv:oc=16,k=1,s=1,relu=1",
     (3, 36, 36)),
    ("pool_only", "id=case0000000004 " + _BASE + "f0=pool:size=2,s=2 h0=dense:units=16", (3, 20, 20)),
    ("stride3_k7", "id=case0000000005 " + _BASE +
     "f0=conv:oc=24,k=7,s=3,relu=1 f1=conv:oc=128,k=3,s=2,relu=1 f2=conv:oc=256,k=2,s=1,relu=0 "
     "h0=dense:units=40", (3, 48, 48)),
    ("odd_units", "id=case0000000006 " + _BASE +
     "f0=conv:oc=64,k=5,s=3,relu=1 h0=dense:units=37", (3, 40, 40)),
    # max-pool in the conv epilogue: packed first conv -> 3x3/3 (KK=9), gather conv -> 2x2 stride 3 (gaps)
    ("fused_pools", "id=case0000000007 " + _BASE +
     "f0=conv:oc=16,k=3,s=1,relu=1 f1=pool:size=3,s=3 f2=conv:oc=32,k=3,s=1,relu=1 f3=pool:size=2,s=3 "
     "h0=dense:units=24", (3, 50, 50)),
    # relu=0 conv before a fused pool (no dead windows), C=64 conv fused (gather instead of TMA im2col)
    ("fused_norelu_c64", "id=case0000000008 " + _BASE +
     "f0=conv:oc=64,k=5,s=1,relu=0 f1=pool:size=2,s=2 f2=conv:oc=128,k=3,s=1,relu=1 f3=pool:size=3,s=3",
     (3, 40, 40)),
    # sub-wave layers (few tiles, long K): split-K forward with the pooled reduce (f1 + f2) and
    # with the plain bias/ReLU reduce (f3)
    ("subwave_splitk", "id=case0000000010 " + _BASE +
     "f0=conv:oc=96,k=4,s=2,relu=1 f1=conv:oc=128,k=4,s=1,relu=1 f2=pool:size=2,s=2 "
     "f3=conv:oc=64,k=3,s=1,relu=1", (3, 40, 40)),
    # C2 population genome #15 (2d5ebb4eae1bf684): 262,144 -> 523 head
    ("c2_g15", "id=2d5ebb4eae1bf684 parents= lr=0.017072315886796932 momentum=0.5 batch_size=32 "
     "f0=conv:oc=256,k=5,s=3,relu=1 h0=dense:units=523", (3, 100, 100)),
]


def case_genome(text):
    return parse_genome(text)


def make_batch(n, shape, seed=0):
    rng = np.random.default_rng(seed)
    x = (rng.integers(0, 256, size=(n, *shape)).astype(np.float32) / np.float32(255.0))
    y = rng.integers(0, 2, size=n).astype(np.int64)
    y[0], y[1] = 0, 1
    return x, y
