// Device kernels of the candidate training step (CUDA-core path).
//
// Layouts: activations NHWC (channels innermost, first-layer channels padded
// to a multiple of 8 with zeros); conv weights [o][kh][kw][c_pad]; dense
// weights [o][in] with `in` in (h, w, c_pad) flatten order. The reference
// flattens in (c, h, w) order (nn.py:197-199); the permutation is applied to
// the first dense layer's columns when parameters are loaded.
#pragma once
#include "common.cuh"

namespace ce {

// ---------------------------------------------------------------- generic SIMT GEMM
// D[m, n] = sum_k A(m, k) * B(k, n) over k in the split's range; E(m, n, split, v)
// consumes each result. 64x64 tile, BK=16, 256 threads, 4x4 outputs per thread.
constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

template <int TM, class AF, class BF, class EP>
__global__ void __launch_bounds__(256) simt_gemm_kernel(const AF A, const BF B, const EP E, int M, int N, int K,
                                                       int kchunk) {
  constexpr int BM = 16 * TM;  // TM rows per thread: 64-row tiles, or 32 for skinny M (batch rows)
  __shared__ float As[SG_BK][BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * SG_BN;
  const int kbeg = blockIdx.z * kchunk;
  const int kend = min(K, kbeg + kchunk);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[TM][4];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // Separable operands (im2col: element offset = row part(m) + column part(k)):
  // each thread's rows (A) / columns (B) are fixed across the K loop, so their
  // offset parts are computed once here.
  size_t a_row[TM];
  bool a_ok[TM];
  if constexpr (AF::SEPARABLE) {
#pragma unroll
    for (int j = 0; j < TM; ++j) {
      const int m = m0 + (threadIdx.x >> 4) + 16 * j;
      a_ok[j] = m < M;
      a_row[j] = a_ok[j] ? A.row(m) : 0;
    }
  }
  size_t b_col = 0;
  bool b_ok = false;
  if constexpr (BF::SEPARABLE) {
    const int n = n0 + (threadIdx.x & 63);
    b_ok = n < N;
    b_col = b_ok ? B.col(n) : 0;
  }
  for (int k0 = kbeg; k0 < kend; k0 += SG_BK) {
    if constexpr (AF::SEPARABLE) {  // thread loads column kk = tid % 16 of rows tid/16 + 16 j
      const int kk = threadIdx.x & 15, k = k0 + kk;
      const bool kok = k < kend;
      const size_t ko = kok ? A.col(k) : 0;
#pragma unroll
      for (int j = 0; j < TM; ++j) As[kk][(threadIdx.x >> 4) + 16 * j] = (kok && a_ok[j]) ? A.ld(a_row[j] + ko) : 0.f;
    } else
#pragma unroll
    for (int e = threadIdx.x; e < BM * SG_BK; e += 256) {
      int mm, kk;
      if (AF::M_FAST) {
        mm = e % BM;
        kk = e / BM;
      } else {
        kk = e % SG_BK;
        mm = e / SG_BK;
      }
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < kend) ? A(m, k) : 0.f;
    }
    if constexpr (BF::SEPARABLE) {  // thread loads column nn = tid % 64 of rows tid/64 + 4 j
      const int nn = threadIdx.x & 63;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int kk = (threadIdx.x >> 6) + 4 * j, k = k0 + kk;
        Bs[kk][nn] = (b_ok && k < kend) ? B.ld(B.row(k) + b_col) : 0.f;
      }
    } else
#pragma unroll
    for (int e = threadIdx.x; e < SG_BN * SG_BK; e += 256) {
      int nn, kk;
      if (BF::N_FAST) {
        nn = e % SG_BN;
        kk = e / SG_BN;
      } else {
        kk = e % SG_BK;
        nn = e / SG_BK;
      }
      const int n = n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (n < N && k < kend) ? B(k, n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[TM], b[4];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty * TM + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < N) E(m, n, blockIdx.z, acc[i][j]);
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
  if (M <= 32) {
    dim3 grid(cdiv(M, 32), cdiv(N, SG_BN), splits);
    simt_gemm_kernel<2><<<grid, 256, 0, st>>>(A, B, E, M, N, K, kchunk);
  } else {
    dim3 grid(cdiv(M, SG_BM), cdiv(N, SG_BN), splits);
    simt_gemm_kernel<4><<<grid, 256, 0, st>>>(A, B, E, M, N, K, kchunk);
  }
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
  __device__ void operator()(int r, int c, int split, float v) const {
    part[((size_t)split * rows + r) * cols + c] = v;
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
    float wv = w[off], vv = vel[off];
    sgd_update(wv, vv, g, lr, mu);
    w[off] = wv;
    vel[off] = vv;
    if (wbf) wbf[off] = __float2bfloat16_rn(wv);
  }
};

}  // namespace ce
