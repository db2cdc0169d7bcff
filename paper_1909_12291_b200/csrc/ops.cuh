// Element-wise / reduction kernels of the training step: batch gather and
// normalisation, max-pool forward/backward, column sums, fused SGD updates,
// dense split-K reduction, softmax cross-entropy, prediction head and the
// host-layout <-> device-layout parameter permutations.
#pragma once
#include <algorithm>
#include "kernels.cuh"

namespace ce {

inline int grid_for(size_t n, int threads = 256) {
  size_t g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

// 8 consecutive elements <-> float[8] (16-byte bf16 / 2x16-byte fp32 vectors), defined below
template <class T>
__device__ __forceinline__ void load8(const T* p, float (&v)[8]);
template <class T>
__device__ __forceinline__ void store8(T* p, const float (&v)[8]);

// ---------------------------------------------------------------- input
// x[b][y][x][cp] = cp < C ? pix[idx[b]][cp][y][x] / 255 : 0      (data.py:65-66)
// idx source: perm[epoch*n_perm + bi*B + b] with (epoch, bi) from the device
// step counter (graph-replayable), or a plain base index (predict).
// One thread per 4 consecutive pixels: one 4-byte load per channel plane and
// 4 x (Cp/8) 16-byte stores; the correctly rounded v/255 (true division, as
// numpy's astype(f32)/f32(255)) comes from a 256-entry shared table.
constexpr int kGatherPx = 4;
inline dim3 gather_grid(int HW, int B) { return dim3((unsigned)((HW + kGatherPx * 256 - 1) / (kGatherPx * 256)), B); }

template <class T>
__global__ void __launch_bounds__(256) gather_u8_kernel(const uint8_t* __restrict__ pix,
                                                        const uint8_t* __restrict__ labels,
                                                        const int32_t* __restrict__ perm,
                                                        const int* __restrict__ step_ctr, int n_perm,
                                                        int steps_per_epoch, int base, int B, int C, int Cp, int HW,
                                                        T* __restrict__ x, int32_t* __restrict__ y) {
  __shared__ float lut[256];
  lut[threadIdx.x] = __fdiv_rn((float)threadIdx.x, 255.0f);  // blockDim.x == 256
  const int b = blockIdx.y;
  int src;
  if (perm && step_ctr) {
    const int step = *step_ctr;
    const int epoch = step / steps_per_epoch, bi = step - epoch * steps_per_epoch;
    src = perm[(size_t)epoch * n_perm + (size_t)bi * B + b];
  } else if (perm) {  // plain index list (kernel-level ABI)
    src = perm[base + b];
  } else {
    src = base + b;
  }
  __syncthreads();
  const uint8_t* img = pix + (size_t)src * C * HW;
  T* xb = x + (size_t)b * HW * Cp;
  if ((HW & 3) == 0 && (reinterpret_cast<uintptr_t>(pix) & 3) == 0) {
    const int HW4 = HW >> 2;
    for (int p4 = blockIdx.x * blockDim.x + threadIdx.x; p4 < HW4; p4 += gridDim.x * blockDim.x) {
      for (int c0 = 0; c0 < Cp; c0 += 8) {
        float v[kGatherPx][8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + u;
          if (c < C) {
            const uint32_t q = __ldg(reinterpret_cast<const uint32_t*>(img + (size_t)c * HW) + p4);
#pragma unroll
            for (int k = 0; k < kGatherPx; ++k) v[k][u] = lut[(q >> (8 * k)) & 0xff];
          } else {
#pragma unroll
            for (int k = 0; k < kGatherPx; ++k) v[k][u] = 0.f;
          }
        }
#pragma unroll
        for (int k = 0; k < kGatherPx; ++k) store8(xb + ((size_t)p4 * kGatherPx + k) * Cp + c0, v[k]);
      }
    }
  } else {
    for (int px = blockIdx.x * blockDim.x + threadIdx.x; px < HW; px += gridDim.x * blockDim.x) {
      for (int c0 = 0; c0 < Cp; c0 += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + u;
          v[u] = c < C ? lut[img[(size_t)c * HW + px]] : 0.f;
        }
        store8(xb + (size_t)px * Cp + c0, v);
      }
    }
  }
  if (y && labels && blockIdx.x == 0 && threadIdx.x == 0) y[b] = labels[src];
}

// fp32 NCHW (host batch) -> T NHWC padded
template <class T>
__global__ void nchw_to_nhwc_kernel(const float* __restrict__ in, int B, int C, int Cp, int HW, T* __restrict__ x) {
  size_t total = (size_t)B * HW;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    size_t b = e / HW, px = e % HW;
    for (int c = 0; c < Cp; ++c) stf(x + e * Cp, c, c < C ? in[(b * C + c) * HW + px] : 0.f);
  }
}

// T NHWC (Cp) -> fp32 NCHW (C)
template <class T>
__global__ void nhwc_to_nchw_kernel(const T* __restrict__ x, int B, int C, int Cp, int HW, float* __restrict__ out) {
  size_t total = (size_t)B * C * HW;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    size_t px = e % HW, t = e / HW;
    size_t c = t % C, b = t / C;
    out[e] = ldf(x, (b * HW + px) * Cp + c);
  }
}

// ---------------------------------------------------------------- max pool
// ties -> first window element in row-major order (nn.py:119-150). One thread
// per (pixel, 8-channel group): 16-byte loads, 32-bit index math.
template <class T>
__device__ __forceinline__ void load8(const T* p, float (&v)[8]);
template <class T>
__device__ __forceinline__ void store8(T* p, const float (&v)[8]);

// Window size K and stride S are template parameters (search space: K in {2,3},
// S in {1,2,3}) so every tap load is issued before the first compare.
// relu_flag: the pool input is a ReLU output, so the gradient of a window
// whose max is not > 0 is zero (mask(x > 0) at the argmax position); the
// forward stores argmax 0xFF for such windows, which never matches a tap in
// the backward, and the mask tensor is not read there at all.

template <class T, int K, int S>
__global__ void __launch_bounds__(256) maxpool_fwd_kernel(const T* __restrict__ x, ConvGeom g, T* __restrict__ y,
                                                          uint8_t* __restrict__ arg, bool relu_flag) {
  const int cg = g.c / 8;
  const int total = g.n * g.oh * g.ow * cg;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int c0 = (e % cg) * 8;
    int t = e / cg;
    const int q = t % g.ow;
    t /= g.ow;
    const int p = t % g.oh, n = t / g.oh;
    const T* base = x + (((size_t)n * g.h + p * S) * g.w + q * S) * g.c + c0;
    float v[K * K][8];
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j) load8(base + ((size_t)i * g.w + j) * g.c, v[i * K + j]);
    float best[8];
    uint8_t bi[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      best[u] = v[0][u];
      bi[u] = 0;
#pragma unroll
      for (int tap = 1; tap < K * K; ++tap)
        if (v[tap][u] > best[u]) {
          best[u] = v[tap][u];
          bi[u] = (uint8_t)tap;
        }
      if (relu_flag && !(best[u] > 0.f)) bi[u] = kPoolDead;
    }
    const size_t o = (size_t)e * 8;
    store8(y + o, best);
    if (arg) *(uint2*)(arg + o) = *(const uint2*)bi;
  }
}

// gather form: dx[n,h,w,c] = sum over windows (p,q) whose argmax hits (h,w),
// accumulated in window order; optional ReLU mask of the pool input (the
// kernel-level ABI; the network path folds the mask into the argmax).
template <class T, class TG, int K, int S>
__global__ void __launch_bounds__(256) maxpool_bwd_kernel(const TG* __restrict__ dy, const uint8_t* __restrict__ arg,
                                                          ConvGeom g, const T* __restrict__ mask, TG* __restrict__ dx) {
  constexpr int W = (K + S - 1) / S;  // windows covering a pixel along one axis
  const int cg = g.c / 8;
  const int total = g.n * g.h * g.w * cg;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int c0 = (e % cg) * 8;
    int t = e / cg;
    const int wx = t % g.w;
    t /= g.w;
    const int hy = t % g.h, n = t / g.h;
    // highest window index covering hy / wx, then walk down W candidates
    const int p_top = min(hy / S, g.oh - 1), q_top = min(wx / S, g.ow - 1);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint2 a2[W][W];
    float v[W][W][8];
    bool ok[W][W];
#pragma unroll
    for (int di = 0; di < W; ++di)
#pragma unroll
      for (int dj = 0; dj < W; ++dj) {
        const int p = p_top - (W - 1 - di), q = q_top - (W - 1 - dj);
        ok[di][dj] = p >= 0 && q >= 0 && hy - p * S < K && wx - q * S < K;
        if (ok[di][dj]) {
          const size_t o = (((size_t)n * g.oh + p) * g.ow + q) * g.c + c0;
          a2[di][dj] = *(const uint2*)(arg + o);
          load8(dy + o, v[di][dj]);
        }
      }
#pragma unroll
    for (int di = 0; di < W; ++di)
#pragma unroll
      for (int dj = 0; dj < W; ++dj) {
        if (!ok[di][dj]) continue;
        const int p = p_top - (W - 1 - di), q = q_top - (W - 1 - dj);
        const uint8_t hit = (uint8_t)((hy - p * S) * K + (wx - q * S));
        const uint8_t* a = (const uint8_t*)&a2[di][dj];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (a[u] == hit) acc[u] += v[di][dj][u];
      }
    const size_t off = (size_t)e * 8;
    if (mask) {
      float m[8];
      load8(mask + off, m);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (!(m[u] > 0.f)) acc[u] = 0.f;
    }
    store8(dx + off, acc);
  }
}

// Strip forms: a thread walks kPoolStrip consecutive rows of one (pixel column,
// 8-channel group) and keeps the window rows it still needs in registers, so
// overlapping windows (S < K) load each input row once per thread instead of K
// times. Same tie rule (first max in row-major window order) and the same
// accumulation order (p, then q ascending) as the per-element kernels above.
constexpr int kPoolStrip = 8;
constexpr size_t kPoolStripMinWork = (size_t)148 * 2048 * 8;  // >= 8 strip rows per resident thread

template <class T, int K, int S>
__global__ void __launch_bounds__(256, K == 2 ? 4 : 2) maxpool_fwd_strip_kernel(const T* __restrict__ x, ConvGeom g, T* __restrict__ y,
                                                                uint8_t* __restrict__ arg, bool relu_flag) {
  const int cg = g.c / 8, strips = (g.oh + kPoolStrip - 1) / kPoolStrip;
  const int total = g.n * strips * g.ow * cg;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int c0 = (e % cg) * 8;
    int t = e / cg;
    const int q = t % g.ow;
    t /= g.ow;
    const int sp = t % strips, n = t / strips;
    const int p0 = sp * kPoolStrip, p1 = min(g.oh, p0 + kPoolStrip);
    const T* col = x + ((size_t)n * g.h * g.w + (size_t)q * S) * g.c + c0;  // (row 0, col q*S)
    float v[K][K][8];  // window rows i = 0..K-1 of the current output row
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j) load8(col + ((size_t)(p0 * S + i) * g.w + j) * g.c, v[i][j]);
    for (int p = p0; p < p1; ++p) {
      if (p > p0) {
        if constexpr (S < K) {
#pragma unroll
          for (int i = 0; i < K - S; ++i)
#pragma unroll
            for (int j = 0; j < K; ++j)
#pragma unroll
              for (int u = 0; u < 8; ++u) v[i][j][u] = v[i + S][j][u];
#pragma unroll
          for (int i = K - S; i < K; ++i)
#pragma unroll
            for (int j = 0; j < K; ++j) load8(col + ((size_t)(p * S + i) * g.w + j) * g.c, v[i][j]);
        } else {
#pragma unroll
          for (int i = 0; i < K; ++i)
#pragma unroll
            for (int j = 0; j < K; ++j) load8(col + ((size_t)(p * S + i) * g.w + j) * g.c, v[i][j]);
        }
      }
      float best[8];
      uint8_t bi[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        best[u] = v[0][0][u];
        bi[u] = 0;
#pragma unroll
        for (int tap = 1; tap < K * K; ++tap)
          if (v[tap / K][tap % K][u] > best[u]) {
            best[u] = v[tap / K][tap % K][u];
            bi[u] = (uint8_t)tap;
          }
        if (relu_flag && !(best[u] > 0.f)) bi[u] = kPoolDead;
      }
      const size_t o = (((size_t)n * g.oh + p) * g.ow + q) * g.c + c0;
      store8(y + o, best);
      if (arg) *(uint2*)(arg + o) = *(const uint2*)bi;
    }
  }
}

// stride-1 backward: input row r receives from window rows p in [r-K+1, r]; the
// thread keeps those K rows (dy + argmax of its K window columns) in a ring
template <class T, class TG, int K>
__global__ void __launch_bounds__(256, K == 2 ? 4 : 2) maxpool_bwd_s1_strip_kernel(const TG* __restrict__ dy,
                                                                   const uint8_t* __restrict__ arg, ConvGeom g,
                                                                   const T* __restrict__ mask, TG* __restrict__ dx) {
  const int cg = g.c / 8, strips = (g.h + kPoolStrip - 1) / kPoolStrip;
  const int total = g.n * strips * g.w * cg;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int c0 = (e % cg) * 8;
    int t = e / cg;
    const int xw = t % g.w;
    t /= g.w;
    const int sp = t % strips, n = t / strips;
    const int r0 = sp * kPoolStrip, r1 = min(g.h, r0 + kPoolStrip);
    // window columns q = xw - K + 1 + jj (jj = 0..K-1, ascending q)
    float d[K][K][8];      // [ring row][jj][channel]
    uint2 a[K][K];
    bool ok[K][K];
    auto load_row = [&](int slot, int p) {
#pragma unroll
      for (int jj = 0; jj < K; ++jj) {
        const int qq = xw - K + 1 + jj;
        ok[slot][jj] = p >= 0 && p < g.oh && qq >= 0 && qq < g.ow;
        if (ok[slot][jj]) {
          const size_t o = (((size_t)n * g.oh + p) * g.ow + qq) * g.c + c0;
          a[slot][jj] = *(const uint2*)(arg + o);
          load8(dy + o, d[slot][jj]);
        }
      }
    };
    // ring slot i holds window row p = r - K + 1 + i for the current input row r
#pragma unroll
    for (int i = 0; i < K; ++i) load_row(i, r0 - K + 1 + i);
    for (int r = r0; r < r1; ++r) {
      if (r > r0) {
#pragma unroll
        for (int i = 0; i < K - 1; ++i)
#pragma unroll
          for (int jj = 0; jj < K; ++jj) {
            ok[i][jj] = ok[i + 1][jj];
            a[i][jj] = a[i + 1][jj];
#pragma unroll
            for (int u = 0; u < 8; ++u) d[i][jj][u] = d[i + 1][jj][u];
          }
        load_row(K - 1, r);
      }
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < K; ++i)  // p ascending
#pragma unroll
        for (int jj = 0; jj < K; ++jj) {  // q ascending
          if (!ok[i][jj]) continue;
          // tap of (r, xw) inside window (p, q): (r - p) * K + (xw - q)
          const uint8_t hit = (uint8_t)((K - 1 - i) * K + (K - 1 - jj));
          const uint8_t* av = (const uint8_t*)&a[i][jj];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (av[u] == hit) acc[u] += d[i][jj][u];
        }
      const size_t off = (((size_t)n * g.h + r) * g.w + xw) * g.c + c0;
      if (mask) {
        float m[8];
        load8(mask + off, m);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (!(m[u] > 0.f)) acc[u] = 0.f;
      }
      store8(dx + off, acc);
    }
  }
}

template <class T>
int launch_maxpool_fwd(const T* x, const ConvGeom& g, T* y, uint8_t* arg, bool relu_flag, cudaStream_t st) {
  // strips only pay for overlapping windows on maps large enough to keep every SM busy
  const size_t outs = (size_t)g.n * g.oh * g.ow * (g.c / 8);
  if (g.s < g.k && outs >= kPoolStripMinWork) {
    const int strips = (g.oh + kPoolStrip - 1) / kPoolStrip;
    const int sgrid = grid_for((size_t)g.n * strips * g.ow * (g.c / 8));
    if (g.k == 2) { maxpool_fwd_strip_kernel<T, 2, 1><<<sgrid, 256, 0, st>>>(x, g, y, arg, relu_flag); return CE_OK; }
    if (g.s == 1) { maxpool_fwd_strip_kernel<T, 3, 1><<<sgrid, 256, 0, st>>>(x, g, y, arg, relu_flag); return CE_OK; }
    maxpool_fwd_strip_kernel<T, 3, 2><<<sgrid, 256, 0, st>>>(x, g, y, arg, relu_flag);
    return CE_OK;
  }
  const int grid = grid_for(outs);
#define CE_POOL_F(KK, SS) \
  if (g.k == KK && g.s == SS) { maxpool_fwd_kernel<T, KK, SS><<<grid, 256, 0, st>>>(x, g, y, arg, relu_flag); return CE_OK; }
  CE_POOL_F(2, 1) CE_POOL_F(2, 2) CE_POOL_F(2, 3) CE_POOL_F(3, 1) CE_POOL_F(3, 2) CE_POOL_F(3, 3)
#undef CE_POOL_F
  return fail(CE_EINVAL, "max pool size %d stride %d not supported (size 2..3, stride 1..3)", g.k, g.s);
}

template <class T, class TG>
int launch_maxpool_bwd(const TG* dy, const uint8_t* arg, const ConvGeom& g, const T* mask, TG* dx, cudaStream_t st) {
  if (g.s == 1 && (size_t)g.n * g.h * g.w * (g.c / 8) >= kPoolStripMinWork) {
    const int strips = (g.h + kPoolStrip - 1) / kPoolStrip;
    const int sgrid = grid_for((size_t)g.n * strips * g.w * (g.c / 8));
    if (g.k == 2) { maxpool_bwd_s1_strip_kernel<T, TG, 2><<<sgrid, 256, 0, st>>>(dy, arg, g, mask, dx); return CE_OK; }
    if (g.k == 3) { maxpool_bwd_s1_strip_kernel<T, TG, 3><<<sgrid, 256, 0, st>>>(dy, arg, g, mask, dx); return CE_OK; }
  }
  const int grid = grid_for((size_t)g.n * g.h * g.w * (g.c / 8));
#define CE_POOL_B(KK, SS) \
  if (g.k == KK && g.s == SS) { maxpool_bwd_kernel<T, TG, KK, SS><<<grid, 256, 0, st>>>(dy, arg, g, mask, dx); return CE_OK; }
  CE_POOL_B(2, 1) CE_POOL_B(2, 2) CE_POOL_B(2, 3) CE_POOL_B(3, 1) CE_POOL_B(3, 2) CE_POOL_B(3, 3)
#undef CE_POOL_B
  return fail(CE_EINVAL, "max pool size %d stride %d not supported (size 2..3, stride 1..3)", g.k, g.s);
}

// ---------------------------------------------------------------- reductions
// Column sums of a row-major [M][N] matrix (bias gradients):
// part[block][o] = sum over the block's rows of dy[m][o]. Each thread owns 8
// consecutive columns (one 16-byte bf16 load / two float4), a block covers
// 256/(N/8) rows per iteration, and the block's row-groups are reduced in
// shared memory in a fixed order (deterministic).
template <class T>
__device__ __forceinline__ void load8(const T* p, float (&v)[8]);
template <>
__device__ __forceinline__ void load8<bf16>(const bf16* p, float (&v)[8]) {
  uint4 u = *(const uint4*)p;
  const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&v)[8]) {
  float4 a = *(const float4*)p, b = *(const float4*)(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <class T>
__device__ __forceinline__ void store8(T* p, const float (&v)[8]);
template <>
__device__ __forceinline__ void store8<bf16>(bf16* p, const float (&v)[8]) {
  uint4 u;
  __nv_bfloat162* h = (__nv_bfloat162*)&u;
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *(uint4*)p = u;
}
template <>
__device__ __forceinline__ void store8<float>(float* p, const float (&v)[8]) {
  *(float4*)p = make_float4(v[0], v[1], v[2], v[3]);
  *(float4*)(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}

template <class T>
__global__ void __launch_bounds__(256) colsum8_kernel(const T* __restrict__ dy, int M, int N, int rows_per_block,
                                                      float* __restrict__ part) {
  __shared__ float red[256][9];
  const int groups = N / 8;                 // column groups (N % 8 == 0)
  const int rgroups = 256 / groups;         // rows processed per iteration
  const int cg = threadIdx.x % groups, rg = threadIdx.x / groups;
  const int m0 = blockIdx.x * rows_per_block, m1 = min(M, m0 + rows_per_block);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (rg < rgroups) {
    for (int m = m0 + rg; m < m1; m += rgroups) {
      float v[8];
      load8(dy + (size_t)m * N + cg * 8, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += v[i];
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) red[threadIdx.x][i] = acc[i];
  __syncthreads();
  if (threadIdx.x < groups) {
    float tot[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < rgroups; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) tot[i] += red[r * groups + threadIdx.x][i];
#pragma unroll
    for (int i = 0; i < 8; ++i) part[(size_t)blockIdx.x * N + threadIdx.x * 8 + i] = tot[i];
  }
}

// generic (any N) fallback for dense biases with N % 8 != 0
template <class T>
__global__ void colsum_partial_kernel(const T* __restrict__ dy, int M, int N, int mchunk, float* __restrict__ part) {
  const int split = blockIdx.y;
  const int m0 = split * mchunk, m1 = min(M, m0 + mchunk);
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < N; o += gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int m = m0; m < m1; ++m) acc += ldf(dy, (size_t)m * N + o);
    part[(size_t)split * N + o] = acc;
  }
}

constexpr int kColsumMaxSplits = 256;

// launches the column sum; returns the number of partial rows written
template <class T>
inline int colsum(const T* dy, int M, int N, float* part, cudaStream_t st) {
  if (N % 8 == 0 && N <= 2048) {
    int rows = std::max(256, cdiv(M, kColsumMaxSplits));
    int blocks = cdiv(M, rows);
    colsum8_kernel<T><<<blocks, 256, 0, st>>>(dy, M, N, rows, part);
    return blocks;
  }
  int splits = std::max(1, std::min(64, M / 64));
  colsum_partial_kernel<T><<<dim3(cdiv(N, 128), splits), 128, 0, st>>>(dy, M, N, cdiv(M, splits), part);
  return splits;
}

// conv weights: g = sum_split part[split][o][kk]; momentum update of W (fp32 master)
// plus bf16 mirrors W[o][kk] and Wt[c][tap][o] (dgrad operand of the tensor path)
__global__ void conv_sgd_kernel(const float* __restrict__ part, int splits, int co, int K, int cp, int k, int s,
                                float* __restrict__ w, float* __restrict__ vel, float* __restrict__ gw,
                                bf16* __restrict__ wbf, bf16* __restrict__ wtbf, float lr, float mu) {
  size_t total = (size_t)co * K;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    float g = 0.f;
    for (int s = 0; s < splits; ++s) g += part[(size_t)s * total + e];
    if (gw) gw[e] = g;
    if (!w) continue;  // reduction only (kernel-level wgrad)
    float wv = w[e], vv = vel[e];
    sgd_update(wv, vv, g, lr, mu);
    w[e] = wv;
    vel[e] = vv;
    if (wbf) wbf[e] = __float2bfloat16_rn(wv);
    if (wtbf) {
      int o = e / K, kk = e % K;
      int c = kk % cp, tap = kk / cp;
      wtbf[dg_wt_index(k, s, cp, co, tap / k, tap % k, c, o)] = __float2bfloat16_rn(wv);
    }
  }
}

// Fixed-order warp sum of part[s][stride * s + off] over s in [0, splits):
// lane l adds s = l, l+32, ... then a fixed xor tree (deterministic).
__device__ __forceinline__ float warp_sum_splits(const float* __restrict__ part, int splits, size_t stride,
                                                 size_t off) {
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int s = lane; s < splits; s += 32) acc += part[(size_t)s * stride + off];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// Tiled conv weight update: tile = 32 output channels x 64 reduction columns
// (kk = (i, j, c)). Each thread owns 2 rows x 4 columns: split partials, W, V
// and the bf16 mirror stream as float4 / 8-byte vectors along kk; the
// dgrad-operand transpose Wt ([class][c][tap][o], o innermost) is staged in
// shared memory and written as 16-byte rows of 8 output channels. Blocks of
// the first column tile also reduce and apply the bias update (fixed split
// order, deterministic). With w == null only the gradient is produced.
constexpr int CS_TO = 32, CS_TK = 64;
__device__ __forceinline__ float4 f4add(float4 a, const float4& b) {
  a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
  return a;
}
__global__ void __launch_bounds__(256) conv_sgd_tiled_kernel(
    const float* __restrict__ part, int splits, int co, int K, int cp, int k, int s, float* __restrict__ w,
    float* __restrict__ vel, float* __restrict__ gw, bf16* __restrict__ wbf, bf16* __restrict__ wtbf,
    const float* __restrict__ bpart, int bsplits, float* __restrict__ b, float* __restrict__ vb,
    float* __restrict__ gb, float lr, float mu) {
  __shared__ __align__(16) bf16 tile[CS_TK][CS_TO + 8];
  const int kq = threadIdx.x & 15, orow = threadIdx.x >> 4;
  const int kk0 = blockIdx.x * CS_TK + kq * 4, o_base = blockIdx.y * CS_TO;
  const size_t total = (size_t)co * K;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o = o_base + orow + 16 * h;
    if (o >= co || kk0 >= K) continue;
    const size_t e = (size_t)o * K + kk0;
    float4 g = *(const float4*)(part + e);
    for (int sp = 1; sp < splits; ++sp) g = f4add(g, *(const float4*)(part + (size_t)sp * total + e));
    if (gw) *(float4*)(gw + e) = g;
    if (!w) continue;
    float4 wv = *(const float4*)(w + e), vv = *(const float4*)(vel + e);
    sgd_update(wv.x, vv.x, g.x, lr, mu);
    sgd_update(wv.y, vv.y, g.y, lr, mu);
    sgd_update(wv.z, vv.z, g.z, lr, mu);
    sgd_update(wv.w, vv.w, g.w, lr, mu);
    *(float4*)(w + e) = wv;
    *(float4*)(vel + e) = vv;
    const __nv_bfloat162 lo = __floats2bfloat162_rn(wv.x, wv.y), hi = __floats2bfloat162_rn(wv.z, wv.w);
    if (wbf) {
      uint2 u;
      u.x = *(const uint32_t*)&lo;
      u.y = *(const uint32_t*)&hi;
      *(uint2*)(wbf + e) = u;
    }
    const int ol = orow + 16 * h;
    tile[kq * 4 + 0][ol] = lo.x;
    tile[kq * 4 + 1][ol] = lo.y;
    tile[kq * 4 + 2][ol] = hi.x;
    tile[kq * 4 + 3][ol] = hi.y;
  }
  if (w && wtbf) {
    __syncthreads();
    // 64 columns x 4 chunks of 8 output channels: one 16-byte store each
    const int kl = threadIdx.x >> 2, oc = (threadIdx.x & 3) * 8;
    const int kk = blockIdx.x * CS_TK + kl, o = o_base + oc;
    if (kk < K && o < co) {
      const int c = kk % cp, tap = kk / cp;
      const size_t dst = dg_wt_index(k, s, cp, co, tap / k, tap % k, c, o);
      *(uint4*)(wtbf + dst) = *(const uint4*)&tile[kl][oc];
    }
  }
  if (blockIdx.x == 0 && bpart) {  // bias of this tile's 32 channels: 8 warps x 4, warp-parallel over splits
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int oo = warp; oo < CS_TO; oo += 8) {
      const int o = o_base + oo;
      if (o >= co) break;
      const float g = warp_sum_splits(bpart, bsplits, co, o);
      if (lane == 0) {
        if (gb) gb[o] = g;
        if (b) {
          float bv = b[o], v = vb[o];
          sgd_update(bv, v, g, lr, mu);
          b[o] = bv;
          vb[o] = v;
        }
      }
    }
  }
}
// Many splits over a small layer: one warp per weight element, lanes take
// strided splits and a fixed xor tree combines them (warp_sum_splits, deterministic);
// block 0 also reduces and applies the bias update.
__global__ void __launch_bounds__(256) conv_sgd_warp_kernel(
    const float* __restrict__ part, int splits, int co, int K, int cp, int k, int s, float* __restrict__ w,
    float* __restrict__ vel, float* __restrict__ gw, bf16* __restrict__ wbf, bf16* __restrict__ wtbf,
    const float* __restrict__ bpart, int bsplits, float* __restrict__ b, float* __restrict__ vb,
    float* __restrict__ gb, float lr, float mu) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t total = (size_t)co * K;
  const unsigned eblocks = (unsigned)((total + 7) / 8);
  if (blockIdx.x >= eblocks) {  // trailing blocks: one warp per bias channel
    const int o = (int)(blockIdx.x - eblocks) * 8 + warp;
    if (!bpart || o >= co) return;
    const float g = warp_sum_splits(bpart, bsplits, co, o);
    if (lane == 0) {
      if (gb) gb[o] = g;
      if (b) {
        float bv = b[o], v = vb[o];
        sgd_update(bv, v, g, lr, mu);
        b[o] = bv;
        vb[o] = v;
      }
    }
    return;
  }
  const size_t e = (size_t)blockIdx.x * 8 + warp;
  if (e < total) {
    const float g = warp_sum_splits(part, splits, total, e);
    if (lane == 0) {
      if (gw) gw[e] = g;
      if (w) {
        float wv = w[e], vv = vel[e];
        sgd_update(wv, vv, g, lr, mu);
        w[e] = wv;
        vel[e] = vv;
        if (wbf) wbf[e] = __float2bfloat16_rn(wv);
        if (wtbf) {
          const int o = (int)(e / K), kk = (int)(e % K), c = kk % cp, tap = kk / cp;
          wtbf[dg_wt_index(k, s, cp, co, tap / k, tap % k, c, o)] = __float2bfloat16_rn(wv);
        }
      }
    }
  }
}
// Many splits over a mid-sized layer: one thread per float4 of weights, splits
// summed in order (loads coalesced across lanes); trailing blocks reduce the bias
// with one warp per channel. The dgrad transpose (if any) is written per element.
__global__ void __launch_bounds__(256) conv_sgd_vec_kernel(
    const float* __restrict__ part, int splits, int co, int K, int cp, int k, int s, float* __restrict__ w,
    float* __restrict__ vel, float* __restrict__ gw, bf16* __restrict__ wbf, bf16* __restrict__ wtbf,
    const float* __restrict__ bpart, int bsplits, float* __restrict__ b, float* __restrict__ vb,
    float* __restrict__ gb, float lr, float mu, unsigned eblocks) {
  const size_t total = (size_t)co * K;
  if (blockIdx.x >= eblocks) {  // bias: one warp per channel
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int o = (int)(blockIdx.x - eblocks) * 8 + warp;
    if (!bpart || o >= co) return;
    const float g = warp_sum_splits(bpart, bsplits, co, o);
    if (lane == 0) {
      if (gb) gb[o] = g;
      if (b) {
        float bv = b[o], v = vb[o];
        sgd_update(bv, v, g, lr, mu);
        b[o] = bv;
        vb[o] = v;
      }
    }
    return;
  }
  const size_t e = ((size_t)blockIdx.x * 256 + threadIdx.x) * 4;  // K % 4 == 0
  if (e >= total) return;
  float4 g = *(const float4*)(part + e);
#pragma unroll 4
  for (int sp = 1; sp < splits; ++sp) g = f4add(g, *(const float4*)(part + (size_t)sp * total + e));
  if (gw) *(float4*)(gw + e) = g;
  if (!w) return;
  float4 wv = *(const float4*)(w + e), vv = *(const float4*)(vel + e);
  sgd_update(wv.x, vv.x, g.x, lr, mu);
  sgd_update(wv.y, vv.y, g.y, lr, mu);
  sgd_update(wv.z, vv.z, g.z, lr, mu);
  sgd_update(wv.w, vv.w, g.w, lr, mu);
  *(float4*)(w + e) = wv;
  *(float4*)(vel + e) = vv;
  const __nv_bfloat162 lo = __floats2bfloat162_rn(wv.x, wv.y), hi = __floats2bfloat162_rn(wv.z, wv.w);
  if (wbf) {
    uint2 u;
    u.x = *(const uint32_t*)&lo;
    u.y = *(const uint32_t*)&hi;
    *(uint2*)(wbf + e) = u;
  }
  if (wtbf) {
    const bf16 v4[4] = {lo.x, lo.y, hi.x, hi.y};
    for (int j = 0; j < 4; ++j) {
      const size_t ej = e + j;
      const int o = (int)(ej / K), kk = (int)(ej % K), c = kk % cp, tap = kk / cp;
      wtbf[dg_wt_index(k, s, cp, co, tap / k, tap % k, c, o)] = v4[j];
    }
  }
}

inline void launch_conv_sgd(const float* part, int splits, int co, int K, int cp, int k, int s, float* w, float* vel,
                            float* gw, bf16* wbf, bf16* wtbf, const float* bpart, int bsplits, float* b, float* vb,
                            float* gb, float lr, float mu, cudaStream_t st) {
  const size_t total = (size_t)co * K;
  if (splits > 16 && total <= 16384) {  // many splits over a tiny layer: one warp per element
    const unsigned blocks = (unsigned)((total + 7) / 8 + (co + 7) / 8);
    conv_sgd_warp_kernel<<<blocks, 256, 0, st>>>(part, splits, co, K, cp, k, s, w, vel, gw, wbf, wtbf, bpart, bsplits,
                                                 b, vb, gb, lr, mu);
    return;
  }
  if (splits > 16) {  // many splits, more elements: a thread per float4, splits in order
    const unsigned eblocks = (unsigned)((total / 4 + 255) / 256);
    conv_sgd_vec_kernel<<<eblocks + (unsigned)((co + 7) / 8), 256, 0, st>>>(
        part, splits, co, K, cp, k, s, w, vel, gw, wbf, wtbf, bpart, bsplits, b, vb, gb, lr, mu, eblocks);
    return;
  }
  dim3 grid((K + CS_TK - 1) / CS_TK, (co + CS_TO - 1) / CS_TO);
  conv_sgd_tiled_kernel<<<grid, 256, 0, st>>>(part, splits, co, K, cp, k, s, w, vel, gw, wbf, wtbf, bpart, bsplits, b,
                                              vb, gb, lr, mu);
}


// bias: g = sum_split part[split][o]; one warp per output channel
__global__ void bias_sgd_kernel(const float* __restrict__ part, int splits, int n, float* __restrict__ b,
                                float* __restrict__ vel, float* __restrict__ gb, float lr, float mu) {
  const int o = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (o >= n) return;
  const float g = warp_sum_splits(part, splits, n, o);
  if ((threadIdx.x & 31) != 0) return;
  if (gb) gb[o] = g;
  if (!b) return;
  float bv = b[o], vv = vel[o];
  sgd_update(bv, vv, g, lr, mu);
  b[o] = bv;
  vel[o] = vv;
}
inline void launch_bias_sgd(const float* part, int splits, int n, float* b, float* vel, float* gb, float lr, float mu,
                            cudaStream_t st) {
  bias_sgd_kernel<<<cdiv(n, 8), 256, 0, st>>>(part, splits, n, b, vel, gb, lr, mu);
}

// dense forward reduce: y[b][o] = bias[o] + sum_split part[split][b][o]
__global__ void dense_reduce_kernel(const float* __restrict__ part, int splits, int B, int out,
                                    const float* __restrict__ bias, float* __restrict__ y) {
  const size_t total = (size_t)B * out;
  if (splits >= 16) {  // one warp per output element
    const size_t e = blockIdx.x * (size_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (e >= total) return;
    const float acc = warp_sum_splits(part, splits, total, e);
    if ((threadIdx.x & 31) == 0) y[e] = acc + (bias ? bias[e % out] : 0.f);
    return;
  }
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += part[(size_t)s * total + e];
    y[e] = acc + (bias ? bias[e % out] : 0.f);
  }
}
inline void launch_dense_reduce(const float* part, int splits, int B, int out, const float* bias, float* y,
                                cudaStream_t st) {
  const size_t total = (size_t)B * out;
  if (splits >= 16)
    dense_reduce_kernel<<<(unsigned)((total + 7) / 8), 256, 0, st>>>(part, splits, B, out, bias, y);
  else
    dense_reduce_kernel<<<grid_for(total), 256, 0, st>>>(part, splits, B, out, bias, y);
}

// ---------------------------------------------------------------- loss
// softmax cross-entropy (nn.py:287-303), one block, B <= 1024:
// loss = -mean(logp[label]); grad = (softmax - onehot) / B.
// Writes losses[*step] and advances the step counter (end of the step).
// Without a step counter the loss goes to losses[0] (kernel-level ABI); a label
// outside [0, K) makes the loss NaN.
template <class TL>
__global__ void xent_kernel(const float* __restrict__ logits, const TL* __restrict__ y, int B, int K,
                            float* __restrict__ grad, float* __restrict__ losses, int* __restrict__ step_ctr,
                            int* __restrict__ nonfinite) {
  __shared__ double red[1024];
  const int b = threadIdx.x;
  double lp = 0.0;
  if (b < B) {
    const float* z = logits + (size_t)b * K;
    float mx = z[0];
    for (int k = 1; k < K; ++k) mx = fmaxf(mx, z[k]);
    float se = 0.f;
    for (int k = 0; k < K; ++k) se += expf(z[k] - mx);
    float lse = logf(se);
    const long long lab = (long long)y[b];
    if (lab < 0 || lab >= K) lp = __longlong_as_double(0x7ff8000000000000ll);
    for (int k = 0; k < K; ++k) {
      float logp = (z[k] - mx) - lse;
      float gk = expf(logp);
      if (k == lab) {
        gk -= 1.0f;
        lp = (double)logp;
      }
      grad[(size_t)b * K + k] = gk / (float)B;
    }
  }
  red[threadIdx.x] = lp;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int step = step_ctr ? *step_ctr : 0;
    const float loss = (float)(-red[0] / B);
    losses[step] = loss;
    if (nonfinite && !isfinite(loss)) *nonfinite = 1;  // host stops replaying (evaluator.py:168-170)
    if (step_ctr) *step_ctr = step + 1;
  }
}

// predict head (evaluator.py:179-185): p = softmax(logits); score = p[:,1]; pred = argmax
__global__ void predict_head_kernel(const float* __restrict__ logits, int B, int K, int base,
                                    double* __restrict__ scores, int64_t* __restrict__ preds) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const float* z = logits + (size_t)b * K;
  float mx = z[0];
  int am = 0;
  for (int k = 1; k < K; ++k)
    if (z[k] > mx) {
      mx = z[k];
      am = k;
    }
  float se = 0.f;
  for (int k = 0; k < K; ++k) se += expf(z[k] - mx);
  scores[base + b] = (double)(expf(z[1] - mx) / se);
  preds[base + b] = am;
}

// ---------------------------------------------------------------- parameter layouts
// conv: host (o, c, i, j) <-> device [o][i][j][cp]
__global__ void conv_w_to_dev_kernel(const float* __restrict__ hw, int co, int c, int cp, int k, float* __restrict__ w) {
  size_t total = (size_t)co * k * k * cp;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    int ch = e % cp;
    size_t t = e / cp;
    int j = t % k;
    t /= k;
    int i = t % k;
    int o = t / k;
    w[e] = ch < c ? hw[(((size_t)o * c + ch) * k + i) * k + j] : 0.f;
  }
}
__global__ void conv_w_to_host_kernel(const float* __restrict__ w, int co, int c, int cp, int k, float* __restrict__ hw) {
  size_t total = (size_t)co * c * k * k;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    int j = e % k;
    size_t t = e / k;
    int i = t % k;
    t /= k;
    int ch = t % c;
    int o = t / c;
    hw[e] = w[(((size_t)o * k + i) * k + j) * cp + ch];
  }
}
// dense after features: host column (c, h, w) <-> device column (h, w, cp)
__global__ void dense_w_to_dev_kernel(const float* __restrict__ hw, size_t rows, int c, int cp, int hwsz,
                                      float* __restrict__ w) {
  size_t in_dev = (size_t)hwsz * cp, in_host = (size_t)hwsz * c;
  size_t total = rows * in_dev;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    size_t r = e / in_dev, col = e % in_dev;
    int ch = col % cp;
    size_t px = col / cp;
    w[e] = ch < c ? hw[r * in_host + (size_t)ch * hwsz + px] : 0.f;
  }
}
__global__ void dense_w_to_host_kernel(const float* __restrict__ w, size_t rows, int c, int cp, int hwsz,
                                       float* __restrict__ hw) {
  size_t in_dev = (size_t)hwsz * cp, in_host = (size_t)hwsz * c;
  size_t total = rows * in_host;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    size_t r = e / in_host, col = e % in_host;
    int ch = col / hwsz;
    size_t px = col % hwsz;
    hw[e] = w[r * in_dev + px * cp + ch];
  }
}
// [rows][cols] fp32 -> [rows][cols_pad] bf16 with zero padding
__global__ void f32_to_bf16_pad_kernel(const float* __restrict__ a, size_t rows, int cols, int cols_pad,
                                       bf16* __restrict__ b) {
  size_t total = rows * cols_pad;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    size_t r = e / cols_pad;
    int c = e % cols_pad;
    b[e] = c < cols ? __float2bfloat16_rn(a[r * cols + c]) : __float2bfloat16_rn(0.f);
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ a, size_t n, bf16* __restrict__ b) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    b[e] = __float2bfloat16_rn(a[e]);
}
__global__ void conv_wt_kernel(const float* __restrict__ w, int co, int k, int s, int cp, bf16* __restrict__ wt) {
  const int taps = k * k;
  size_t total = (size_t)co * taps * cp;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    int c = e % cp;
    size_t t = e / cp;
    int tap = t % taps;
    int o = t / taps;
    wt[dg_wt_index(k, s, cp, co, tap / k, tap % k, c, o)] = __float2bfloat16_rn(w[e]);
  }
}

// bf16 [o][tap][c] -> class-blocked transpose (dgrad B operand)
__global__ void transpose_w_bf16_kernel(const bf16* __restrict__ w, int co, int k, int s, int cp,
                                        bf16* __restrict__ wt) {
  const int taps = k * k;
  size_t total = (size_t)co * taps * cp;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    int c = e % cp;
    size_t t = e / cp;
    int tap = t % taps;
    int o = t / taps;
    wt[dg_wt_index(k, s, cp, co, tap / k, tap % k, c, o)] = w[e];
  }
}


}  // namespace ce
