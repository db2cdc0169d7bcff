"""The device initialiser (csrc/init.cuh) restates numpy's PCG64 (XSL-RR 128/64)
step, output and jump-ahead. This pins that restatement on the CPU against
numpy itself: same 64-bit outputs, same doubles, same uniform(-l, l) floats,
and advance() == skipping draws (what lets every device thread jump to its
own slice of the Kaiming stream)."""

import numpy as np

M128 = (1 << 128) - 1
MULT = 0x2360ED051FC65DA44385DF649FCCF645


def step(state, inc):
    return (state * MULT + inc) & M128


def output(state):
    hi, lo = state >> 64, state & ((1 << 64) - 1)
    x = hi ^ lo
    rot = state >> 122
    return ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)


def advance(state, inc, delta):
    acc_mult, acc_plus, cur_mult, cur_plus = 1, 0, MULT, inc
    while delta:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & M128
        cur_plus = ((cur_mult + 1) * cur_plus) & M128
        cur_mult = (cur_mult * cur_mult) & M128
        delta >>= 1
    return (acc_mult * state + acc_plus) & M128


def _state(rng):
    st = rng.bit_generator.state["state"]
    return st["state"], st["inc"]


def test_outputs_match_numpy():
    rng = np.random.default_rng(12345)
    s, inc = _state(rng)
    ref = rng.bit_generator.random_raw(64)
    got = []
    for _ in range(64):
        s = step(s, inc)
        got.append(output(s))
    assert [int(v) for v in ref] == got


def test_uniform_floats_match_numpy():
    rng = np.random.default_rng(7)
    s, inc = _state(rng)
    limit = np.sqrt(6.0 / 75)
    ref = rng.uniform(-limit, limit, size=200).astype(np.float32)
    vals = []
    for _ in range(200):
        s = step(s, inc)
        d = (output(s) >> 11) * (1.0 / 9007199254740992.0)
        vals.append(np.float32(-limit + (2 * limit) * d))
    np.testing.assert_array_equal(np.array(vals, np.float32), ref)


def test_advance_equals_skipping():
    rng = np.random.default_rng(99)
    s, inc = _state(rng)
    rng.bit_generator.advance(123457)
    s2 = advance(s, inc, 123457)
    assert s2 == _state(rng)[0]
    nxt = step(s2, inc)
    assert output(nxt) == int(rng.bit_generator.random_raw())
