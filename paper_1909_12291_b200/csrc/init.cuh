// Device-side Kaiming-uniform initialisation, bit-exact to the reference's host
// draws (nn.py:44-46 via genome.instantiate, genome.py:309-335).
//
// The reference draws every weight of a network from ONE numpy PCG64 stream
// (XSL-RR 128/64, default_rng(seed)) in layer order, as float64
// U(-l, l) = -l + (2l) * ((x >> 11) * 2^-53), then casts to float32. The host
// records the stream state at the start of each layer and skips over it with
// PCG64.advance(); here every thread jumps to its own chunk of the layer's
// draws (LCG jump-ahead) and writes the float32 values straight into the
// device layout. tests/test_pcg64.py pins the recurrence against numpy; the GPU
// parity test compares the device weights with the host draw bit for bit.
#pragma once
#include "kernels.cuh"

namespace ce {

typedef unsigned __int128 u128;

__host__ __device__ inline u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

__device__ inline u128 pcg_advance(u128 state, u128 inc, unsigned long long delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1ull) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ uint64_t pcg_next(u128& s, u128 inc) {
  s = s * pcg_mult() + inc;
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// Layout of the destination: where reference element r (C order of the
// reference weight shape) lands in the device weight array.
struct InitLayout {
  int kind;         // 0 = identity (dense after dense), 1 = conv, 2 = dense after features
  int co, cin, k;   // conv: reference (co, cin, k, k) -> device [co][k][k][cp]
  int cp;           // stored channels
  long long in_ref; // dense after features: reference columns (c, h, w)
  int hw;           // dense after features: h*w of the flattened input
  long long in_dev; // dense after features: device columns (h, w, cp)
};

__device__ __forceinline__ size_t init_dev_index(const InitLayout& L, size_t r) {
  if (L.kind == 1) {
    const int j = r % L.k;
    size_t t = r / L.k;
    const int i = t % L.k;
    t /= L.k;
    const int c = t % L.cin;
    const size_t o = t / L.cin;
    return ((o * L.k + i) * L.k + j) * L.cp + c;
  }
  if (L.kind == 2) {
    const size_t o = r / L.in_ref, col = r % L.in_ref;
    const size_t c = col / L.hw, px = col % L.hw;
    return o * L.in_dev + px * L.cp + c;
  }
  return r;
}

// draws per thread: each is one link of a dependent 128-bit LCG chain, so the chunk
// length bounds the kernel latency; the per-thread jump-ahead (~2 log2(n) u128
// multiply-adds) is amortised over it
constexpr int kInitChunk = 128;

// numpy Generator.uniform(lo, lo + range): lo + range * next_double, in double,
// then cast to float32 (the .astype of nn.py:46). Draw r of the stream (after
// `skip`) lands at init_dev_index(L, r). Kaiming: lo = -limit, range = 2*limit.
__global__ void kaiming_uniform_kernel(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                                       unsigned long long skip, size_t count, double lo, double range, InitLayout L,
                                       float* __restrict__ w) {
  const u128 state = ((u128)st_hi << 64) | st_lo;
  const u128 inc = ((u128)inc_hi << 64) | inc_lo;
  const size_t nchunks = (count + kInitChunk - 1) / kInitChunk;
  for (size_t ch = blockIdx.x * (size_t)blockDim.x + threadIdx.x; ch < nchunks;
       ch += (size_t)gridDim.x * blockDim.x) {
    u128 s = pcg_advance(state, inc, skip + (unsigned long long)(ch * kInitChunk));
    const size_t r1 = count < (ch + 1) * kInitChunk ? count : (ch + 1) * kInitChunk;
    for (size_t r = ch * kInitChunk; r < r1; ++r) {
      const uint64_t x = pcg_next(s, inc);
      const double d = (double)(x >> 11) * (1.0 / 9007199254740992.0);
      w[init_dev_index(L, r)] = __double2float_rn(__dadd_rn(lo, __dmul_rn(range, d)));
    }
  }
}

}  // namespace ce
