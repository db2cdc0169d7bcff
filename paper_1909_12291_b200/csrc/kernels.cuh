// Device kernels of the candidate training step (CUDA-core path).
//
// Layouts: activations NHWC (channels innermost, first-layer channels padded
// to a multiple of 8 with zeros); conv weights [o][kh][kw][c_pad]; dense
// weights [o][in] with `in` in (h, w, c_pad) flatten order. The reference
// flattens in (c, h, w) order (nn.py:197-199); the permutation is applied to
// the first dense layer's columns when parameters are loaded.
#pragma once
#include <type_traits>
#include "common.cuh"

namespace ce {

// ---------------------------------------------------------------- generic SIMT GEMM
// D[m, n] = sum_k A(m, k) * B(k, n) over k in the split's range; E(m, n, split, v)
// consumes each result (fp32 check mode). Tile (16*TM) x (16*TN), BK = 16, 256
// threads as 16 x 16, each thread TM consecutive rows x TN columns (columns
// tx*4+{0..3} and, for TN = 8, 64+tx*4+{0..3}: conflict-free float4 reads).
// Shared memory is double-buffered: the next K tile is fetched into registers
// while the current one is consumed, one barrier per tile.
constexpr int SG_BM = 64, SG_BN = 128, SG_BK = 16;

// Epilogues may consume 4 consecutive columns at once: `static constexpr bool
// VEC4 = true` plus store4(m, n, split, const float* v, count).
template <class E, class = void>
struct has_vec4 : std::false_type {};
template <class E>
struct has_vec4<E, std::void_t<decltype(E::VEC4)>> : std::bool_constant<E::VEC4> {};
// ... or in two phases (read-modify-write): Pre prefetch4(m, n, count) for the
// whole thread tile first, then commit4(m, n, v, count, pre).
template <class E, class = void>
struct has_prefetch : std::false_type {};
template <class E>
struct has_prefetch<E, std::void_t<typename E::Pre>> : std::true_type {};

inline int simt_tm(int M) { return M <= 32 ? 2 : 4; }
inline int simt_tn(int N) { return N <= 64 ? 4 : 8; }
// output tiles per K split, as launched by simt_gemm
inline long long simt_tiles(int M, int N) {
  return (long long)cdiv(M, 16 * simt_tm(M)) * cdiv(N, 16 * simt_tn(N));
}

template <int TM, int TN, class AF, class BF, class EP>
__global__ void __launch_bounds__(256, 2) simt_gemm_kernel(const AF A, const BF B, const EP E, int M, int N, int K,
                                                       int kchunk) {
  constexpr int BM = 16 * TM, BN = 16 * TN;
  constexpr int AL = BM * SG_BK / 256, BL = BN * SG_BK / 256;  // elements per thread per tile
  __shared__ __align__(16) float As[2][SG_BK][BM + 4];
  __shared__ __align__(16) float Bs[2][SG_BK][BN + 4];
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kbeg = blockIdx.z * kchunk;
  const int kend = min(K, kbeg + kchunk);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  // Separable operands (im2col: element offset = row part(m) + column part(k)):
  // each thread's rows (A) / column (B) are fixed across the K loop.
  size_t a_row[TM];
  bool a_ok[TM];
  if constexpr (AF::SEPARABLE) {
#pragma unroll
    for (int j = 0; j < TM; ++j) {
      const int m = m0 + ty + 16 * j;
      a_ok[j] = m < M;
      a_row[j] = a_ok[j] ? A.row(m) : 0;
    }
  }
  size_t b_col = 0;
  bool b_ok = false;
  if constexpr (BF::SEPARABLE) {
    const int n = n0 + (tid % BN);
    b_ok = n < N;
    b_col = b_ok ? B.col(n) : 0;
  }
  float ra[AL], rb[BL];
  auto fetch = [&](int k0) {
    if constexpr (AF::SEPARABLE) {  // column kk = tid % 16 of rows tid/16 + 16 j
      const int k = k0 + tx;
      const bool kok = k < kend;
      const size_t ko = kok ? A.col(k) : 0;
#pragma unroll
      for (int j = 0; j < AL; ++j) ra[j] = (kok && a_ok[j]) ? A.ld(a_row[j] + ko) : 0.f;
    } else {
#pragma unroll
      for (int j = 0; j < AL; ++j) {
        const int e = tid + 256 * j;
        const int mm = AF::M_FAST ? e % BM : e / SG_BK, kk = AF::M_FAST ? e / BM : e % SG_BK;
        const int m = m0 + mm, k = k0 + kk;
        ra[j] = (m < M && k < kend) ? A(m, k) : 0.f;
      }
    }
    if constexpr (BF::SEPARABLE) {  // column nn = tid % BN of rows tid/BN + (256/BN) j
#pragma unroll
      for (int j = 0; j < BL; ++j) {
        const int k = k0 + tid / BN + (256 / BN) * j;
        rb[j] = (b_ok && k < kend) ? B.ld(B.row(k) + b_col) : 0.f;
      }
    } else {
#pragma unroll
      for (int j = 0; j < BL; ++j) {
        const int e = tid + 256 * j;
        const int nn = BF::N_FAST ? e % BN : e / SG_BK, kk = BF::N_FAST ? e / BN : e % SG_BK;
        const int n = n0 + nn, k = k0 + kk;
        rb[j] = (n < N && k < kend) ? B(k, n) : 0.f;
      }
    }
  };
  auto stash = [&](int buf) {
    if constexpr (AF::SEPARABLE) {
#pragma unroll
      for (int j = 0; j < AL; ++j) As[buf][tx][ty + 16 * j] = ra[j];
    } else {
#pragma unroll
      for (int j = 0; j < AL; ++j) {
        const int e = tid + 256 * j;
        const int mm = AF::M_FAST ? e % BM : e / SG_BK, kk = AF::M_FAST ? e / BM : e % SG_BK;
        As[buf][kk][mm] = ra[j];
      }
    }
    if constexpr (BF::SEPARABLE) {
#pragma unroll
      for (int j = 0; j < BL; ++j) Bs[buf][tid / BN + (256 / BN) * j][tid % BN] = rb[j];
    } else {
#pragma unroll
      for (int j = 0; j < BL; ++j) {
        const int e = tid + 256 * j;
        const int nn = BF::N_FAST ? e % BN : e / SG_BK, kk = BF::N_FAST ? e / BN : e % SG_BK;
        Bs[buf][kk][nn] = rb[j];
      }
    }
  };
  if (kbeg < kend) {
    fetch(kbeg);
    stash(0);
  }
  __syncthreads();
  int buf = 0;
  for (int k0 = kbeg; k0 < kend; k0 += SG_BK) {
    const bool more = k0 + SG_BK < kend;
    if (more) fetch(k0 + SG_BK);
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[TM], b[TN];
      if constexpr (TM == 4) {
        const float4 v = *(const float4*)&As[buf][kk][ty * 4];
        a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
      } else {
        const float2 v = *(const float2*)&As[buf][kk][ty * 2];
        a[0] = v.x; a[1] = v.y;
      }
#pragma unroll
      for (int h = 0; h < TN / 4; ++h) {
        const float4 v = *(const float4*)&Bs[buf][kk][64 * h + tx * 4];
        b[4 * h] = v.x; b[4 * h + 1] = v.y; b[4 * h + 2] = v.z; b[4 * h + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty * TM + i;
    if (m >= M) continue;
#pragma unroll
    for (int h = 0; h < TN / 4; ++h) {
      const int n = n0 + 64 * h + tx * 4;
      if (n >= N) continue;
      if constexpr (has_prefetch<EP>::value) {
        continue;  // handled below: all loads first, then all updates
      } else if constexpr (has_vec4<EP>::value) {
        E.store4(m, n, blockIdx.z, &acc[i][4 * h], min(4, N - n));
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (n + j < N) E(m, n + j, blockIdx.z, acc[i][4 * h + j]);
      }
    }
  }
  if constexpr (has_prefetch<EP>::value) {
    // read-modify-write epilogues: issue every load of the thread's tile before
    // the first store (stores through the same pointers would otherwise pin
    // each group's loads behind the previous group's stores)
    typename EP::Pre pre[TM][TN / 4];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int h = 0; h < TN / 4; ++h) {
        const int m = m0 + ty * TM + i, n = n0 + 64 * h + tx * 4;
        if (m < M && n < N) pre[i][h] = E.prefetch4(m, n, min(4, N - n));
      }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int h = 0; h < TN / 4; ++h) {
        const int m = m0 + ty * TM + i, n = n0 + 64 * h + tx * 4;
        if (m < M && n < N) E.commit4(m, n, &acc[i][4 * h], min(4, N - n), pre[i][h]);
      }
  }
}

template <class AF, class BF, class EP>
inline void simt_gemm(const AF& A, const BF& B, const EP& E, int M, int N, int K, int splits, cudaStream_t st) {
  if (splits < 1) splits = 1;
  int kchunk = cdiv(K, splits);
  kchunk = cdiv(kchunk, SG_BK) * SG_BK;
  splits = cdiv(K, kchunk);
  if (splits < 1) splits = 1;
  const int tm = simt_tm(M), tn = simt_tn(N);
  dim3 grid(cdiv(M, 16 * tm), cdiv(N, 16 * tn), splits);
  if (tm == 2 && tn == 4)
    simt_gemm_kernel<2, 4><<<grid, 256, 0, st>>>(A, B, E, M, N, K, kchunk);
  else if (tm == 2)
    simt_gemm_kernel<2, 8><<<grid, 256, 0, st>>>(A, B, E, M, N, K, kchunk);
  else if (tn == 4)
    simt_gemm_kernel<4, 4><<<grid, 256, 0, st>>>(A, B, E, M, N, K, kchunk);
  else
    simt_gemm_kernel<4, 8><<<grid, 256, 0, st>>>(A, B, E, M, N, K, kchunk);
}

// Number of K splits used by simt_gemm for a requested split count.
inline int simt_splits(int K, int splits) {
  if (splits < 1) splits = 1;
  int kchunk = cdiv(K, splits);
  kchunk = cdiv(kchunk, SG_BK) * SG_BK;
  int s = cdiv(K, kchunk);
  return s < 1 ? 1 : s;
}

// Geometry of one conv layer (per-sample input / output, NHWC).
// max-pool argmax of a window whose ReLU'd input has max <= 0: the backward
// routes it no gradient (matches no tap); see maxpool_fwd_kernel
constexpr uint8_t kPoolDead = 0xFF;

struct ConvGeom {
  int n;           // batch
  int c, h, w;     // input (c = stored channels)
  int co, oh, ow;  // output
  int k, s;
};

// ---------------------------------------------------------------- operand functors
// forward: A = im2col(x) [m=(n,p,q)][kk=(i,j,c)], B = W [kk][o]
// im2col of a valid convolution is separable: x offset = row(m) + col(kk) with
// row = receptive-field origin of output pixel m and col = (tap, channel) offset.
template <class T>
struct FwdA {
  static constexpr bool M_FAST = false, SEPARABLE = true;
  const T* x;
  ConvGeom g;
  FastDiv d_ow, d_oh, d_c, d_k;
  __device__ size_t row(int m) const {
    uint32_t t, q, p, n;
    d_ow.divmod((uint32_t)m, t, q);
    d_oh.divmod(t, n, p);
    return (((size_t)n * g.h + p * g.s) * g.w + q * g.s) * g.c;
  }
  __device__ size_t col(int kk) const {
    uint32_t tap, c, i, j;
    d_c.divmod((uint32_t)kk, tap, c);
    d_k.divmod(tap, i, j);
    return ((size_t)i * g.w + j) * g.c + c;
  }
  __device__ float ld(size_t off) const { return ldf(x, off); }
  __device__ float operator()(int m, int kk) const { return ld(row(m) + col(kk)); }
};
template <class T>
FwdA<T> make_fwd_a(const T* x, const ConvGeom& g) {
  return FwdA<T>{x, g, FastDiv(g.ow), FastDiv(g.oh), FastDiv(g.c), FastDiv(g.k)};
}
struct FwdB {  // W [o][kk] fp32 master
  static constexpr bool N_FAST = false, SEPARABLE = false;
  const float* w;
  int K;
  __device__ float operator()(int kk, int o) const { return w[(size_t)o * K + kk]; }
};
template <class T>
struct FwdEpi {
  T* y;
  const float* bias;
  int co;
  bool relu;
  __device__ void operator()(int m, int o, int, float v) const {
    v += bias[o];
    if (relu) v = v > 0.f ? v : 0.f;
    stf(y, (size_t)m * co + o, v);
  }
};

// dgrad: A = gather(dY) [m=(n,h,w)][kk=(i,j,o)], B = W^T [kk][c]
template <class T>
struct DgradA {
  static constexpr bool M_FAST = false, SEPARABLE = false;
  const T* dy;
  ConvGeom g;
  FastDiv d_w, d_h, d_co, d_k;
  __device__ float operator()(int m, int kk) const {
    uint32_t t, wx, hy, n, tap, o, i, j;
    d_w.divmod((uint32_t)m, t, wx);
    d_h.divmod(t, n, hy);
    d_co.divmod((uint32_t)kk, tap, o);
    d_k.divmod(tap, i, j);
    int hp = (int)hy - (int)i, wq = (int)wx - (int)j;
    if (hp < 0 || wq < 0) return 0.f;
    if (hp % g.s || wq % g.s) return 0.f;
    hp /= g.s;
    wq /= g.s;
    if (hp >= g.oh || wq >= g.ow) return 0.f;
    return ldf(dy, (((size_t)n * g.oh + hp) * g.ow + wq) * g.co + o);
  }
};
template <class T>
DgradA<T> make_dgrad_a(const T* dy, const ConvGeom& g) {
  return DgradA<T>{dy, g, FastDiv(g.w), FastDiv(g.h), FastDiv(g.co), FastDiv(g.k)};
}
struct DgradB {  // W[o][i][j][c] read as [kk=(i,j,o)][c]
  static constexpr bool N_FAST = true, SEPARABLE = false;
  const float* w;
  ConvGeom g;
  __device__ float operator()(int kk, int c) const {
    int o = kk % g.co, tap = kk / g.co;
    return w[((size_t)o * g.k * g.k + tap) * g.c + c];
  }
};
template <class T>
struct DgradEpi {
  T* dx;
  const T* mask;  // activation whose (> 0) pattern gates the gradient (ReLU backward), or null
  int c;
  __device__ void operator()(int m, int ch, int, float v) const {
    size_t off = (size_t)m * c + ch;
    if (mask && !(ldf(mask, off) > 0.f)) v = 0.f;
    stf(dx, off, v);
  }
};

// wgrad: D[o][kk] = sum_m dY[m][o] * im2col(x)[m][kk]; A = dY^T, B = im2col(x)
template <class T>
struct WgradA {
  static constexpr bool M_FAST = true, SEPARABLE = false;
  const T* dy;
  int co;
  __device__ float operator()(int o, int m) const { return ldf(dy, (size_t)m * co + o); }
};
template <class T>
struct WgradB {  // B(k = output pixel m, n = (tap, channel)) = im2col(m, n): separable
  static constexpr bool N_FAST = true, SEPARABLE = true;
  FwdA<T> im2col;
  __device__ size_t row(int m) const { return im2col.row(m); }
  __device__ size_t col(int kk) const { return im2col.col(kk); }
  __device__ float ld(size_t off) const { return im2col.ld(off); }
  __device__ float operator()(int m, int kk) const { return im2col(m, kk); }
};
struct PartialEpi {  // part[split][rows][cols]
  float* part;
  int rows, cols;
  static constexpr bool VEC4 = true;
  __device__ void operator()(int r, int c, int split, float v) const {
    part[((size_t)split * rows + r) * cols + c] = v;
  }
  __device__ void store4(int r, int c, int split, const float* v, int cnt) const {
    const size_t off = ((size_t)split * rows + r) * cols + c;
    if (cnt == 4 && (off & 3) == 0) {
      *(float4*)(part + off) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
      for (int j = 0; j < cnt; ++j) part[off + j] = v[j];
    }
  }
};

// dense forward: y[b][o] = sum_i x[b][i] W[o][i]  (A = x, B = W^T), split-K partials
template <class T>
struct DenseXA {
  static constexpr bool M_FAST = false, SEPARABLE = false;
  const T* x;
  int in;
  __device__ float operator()(int b, int i) const { return ldf(x, (size_t)b * in + i); }
};
struct DenseWB {
  static constexpr bool N_FAST = false, SEPARABLE = false;
  const float* w;
  int in;
  __device__ float operator()(int i, int o) const { return w[(size_t)o * in + i]; }
};
// dense dX: dx[b][i] = sum_o g[b][o] W[o][i]
struct DenseGA {
  static constexpr bool M_FAST = false, SEPARABLE = false;
  const float* g;
  int out;
  __device__ float operator()(int b, int o) const { return g[(size_t)b * out + o]; }
};
struct DenseWN {
  static constexpr bool N_FAST = true, SEPARABLE = false;
  const float* w;
  int in;
  __device__ float operator()(int o, int i) const { return w[(size_t)o * in + i]; }
};
// dense dW: dW[o][i] = sum_b g[b][o] x[b][i]
struct DenseGT {
  static constexpr bool M_FAST = true, SEPARABLE = false;
  const float* g;
  int out;
  __device__ float operator()(int o, int b) const { return g[(size_t)b * out + o]; }
};
template <class T>
struct DenseXN {
  static constexpr bool N_FAST = true, SEPARABLE = false;
  const T* x;
  int in;
  __device__ float operator()(int b, int i) const { return ldf(x, (size_t)b * in + i); }
};

// Class-blocked transposed conv weights (dgrad B operand): for stride s the
// taps split into s*s residue classes (rh, rw) = (i mod s, j mod s); class cls
// owns a contiguous [c][ti*tj*co] block, K index (a'*tj + b')*co + o with the
// class's taps flipped (a' = ti-1-a, b' = tj-1-b; i = rh + s*a, j = rw + s*b):
// each class is then a plain stride-1 "full" convolution of dY.
__host__ __device__ inline int dg_taps(int k, int s, int r) { return r < k ? (k - r + s - 1) / s : 0; }
__host__ __device__ inline size_t dg_class_base(int k, int s, int c, int co, int cls) {
  size_t base = 0;
  for (int q = 0; q < cls; ++q) base += (size_t)c * dg_taps(k, s, q / s) * dg_taps(k, s, q % s) * co;
  return base;
}
__host__ __device__ inline size_t dg_wt_index(int k, int s, int c, int co, int i, int j, int ch, int o) {
  const int rh = i % s, rw = j % s, a = i / s, b = j / s;
  const int ti = dg_taps(k, s, rh), tj = dg_taps(k, s, rw), kcls = ti * tj * co;
  return dg_class_base(k, s, c, co, rh * s + rw) + (size_t)ch * kcls + ((size_t)(ti - 1 - a) * tj + (tj - 1 - b)) * co + o;
}

// classical momentum, in fp32 without FMA contraction (nn.py:306-322):
//   v <- mu*v - lr*g ; w <- w + v
__device__ __forceinline__ void sgd_update(float& w, float& v, float g, float lr, float mu) {
  v = __fsub_rn(__fmul_rn(mu, v), __fmul_rn(lr, g));
  w = __fadd_rn(w, v);
}

// dense dW with the momentum update fused (K = batch, no split; each (o,i) owned once)
struct DenseSgdEpi {
  float* w;
  float* vel;
  float* gw;  // optional: store the raw gradient (introspection)
  bf16* wbf;  // optional bf16 mirror
  int in;
  float lr, mu;
  __device__ void operator()(int o, int i, int, float g) const {
    size_t off = (size_t)o * in + i;
    if (gw) gw[off] = g;
    if (!w) return;  // gradient only
    float wv = w[off], vv = vel[off];
    sgd_update(wv, vv, g, lr, mu);
    w[off] = wv;
    vel[off] = vv;
    if (wbf) wbf[off] = __float2bfloat16_rn(wv);
  }
  struct Pre {
    float4 w, v;
  };
  __device__ Pre prefetch4(int o, int i, int cnt) const {
    const size_t off = (size_t)o * in + i;
    Pre p;
    if (w && cnt == 4 && (off & 3) == 0) {
      p.w = *(const float4*)(w + off);
      p.v = *(const float4*)(vel + off);
    }
    return p;
  }
  __device__ void commit4(int o, int i, const float* g, int cnt, Pre p) const {
    const size_t off = (size_t)o * in + i;
    if (!w) {
      if (cnt == 4 && (off & 3) == 0) *(float4*)(gw + off) = make_float4(g[0], g[1], g[2], g[3]);
      else for (int j = 0; j < cnt; ++j) gw[off + j] = g[j];
      return;
    }
    if (cnt == 4 && (off & 3) == 0) {
      if (gw) *(float4*)(gw + off) = make_float4(g[0], g[1], g[2], g[3]);
      sgd_update(p.w.x, p.v.x, g[0], lr, mu);
      sgd_update(p.w.y, p.v.y, g[1], lr, mu);
      sgd_update(p.w.z, p.v.z, g[2], lr, mu);
      sgd_update(p.w.w, p.v.w, g[3], lr, mu);
      *(float4*)(w + off) = p.w;
      *(float4*)(vel + off) = p.v;
      if (wbf) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(p.w.x, p.w.y), hi = __floats2bfloat162_rn(p.w.z, p.w.w);
        uint2 u;
        u.x = *(const uint32_t*)&lo;
        u.y = *(const uint32_t*)&hi;
        *(uint2*)(wbf + off) = u;
      }
    } else {
      for (int j = 0; j < cnt; ++j) (*this)(o, i + j, 0, g[j]);
    }
  }
};

}  // namespace ce
