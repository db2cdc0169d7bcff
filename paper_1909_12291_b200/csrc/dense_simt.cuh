// Small-batch dense backward on CUDA cores (nn.py:233-240 + sgd_step 306-322).
//
// For B <= 64 the dense dW pass is a streaming read-modify-write of W and its
// velocity (16 B/param + the bf16 mirror) with only B FMAs per parameter, so
// it is HBM-bound even on FFMA. These kernels keep it at the HBM roofline:
// each thread owns 8 output rows x 4 consecutive input columns (float4 rows of
// W / V, fully coalesced), the X tile is staged in shared memory and the G
// values are warp-uniform broadcasts, and the W / V loads of the update are
// issued before the FMA loop so their latency overlaps the arithmetic.
// The same tile shape serves dX = G W (reduction over the output units).
#pragma once
#include <cstdlib>
#include "kernels.cuh"

namespace ce {

constexpr int DS_TI = 256;  // input columns per block: 64 threads x float4
constexpr int DS_TR = 32;   // rows per block: 4 thread-rows x 8
constexpr int DS_KC = 32;   // reduction chunk staged per iteration

template <int R>
__device__ __forceinline__ void fma_rx4(float (&acc)[R][4], const float* g, const float4& x) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    acc[r][0] = fmaf(g[r], x.x, acc[r][0]);
    acc[r][1] = fmaf(g[r], x.y, acc[r][1]);
    acc[r][2] = fmaf(g[r], x.z, acc[r][2]);
    acc[r][3] = fmaf(g[r], x.w, acc[r][3]);
  }
}
__device__ __forceinline__ void fma8x4(float (&acc)[8][4], const float* g8, const float4& x) { fma_rx4<8>(acc, g8, x); }

// 4 consecutive elements as float (vectorised when aligned)
__device__ __forceinline__ float4 ld4f(const float* p) { return *(const float4*)p; }
__device__ __forceinline__ float4 ld4f(const bf16* p) {
  const uint2 u = *(const uint2*)p;
  const float2 a = __bfloat1622float2(*(const __nv_bfloat162*)&u.x), b = __bfloat1622float2(*(const __nv_bfloat162*)&u.y);
  return make_float4(a.x, a.y, b.x, b.y);
}

// dW[o][i] = sum_b g[b][o] x[b][i]; fused momentum SGD of w / vel (skipped when
// w is null: gradient only), optional raw gradient gw and bf16 mirror wb [o][wb_ld].
// R rows per thread: block tile (4R) x 256; grid (cdiv(in, 256), cdiv(out, 4R)), 256 threads.
template <class TX, int R>
__global__ void __launch_bounds__(256, R == 4 ? 3 : 2)
    dense_dw_sgd_simt_kernel(const TX* __restrict__ x, int x_ld, const float* __restrict__ g, int B, int in, int out,
                             float* __restrict__ w, float* __restrict__ vel, float* __restrict__ gw,
                             bf16* __restrict__ wb, int wb_ld, float lr, float mu) {
  constexpr int TR = 4 * R;
  __shared__ __align__(16) float Xs[DS_KC][DS_TI];
  __shared__ __align__(16) float Gs[DS_KC][TR];
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int ib = blockIdx.x * DS_TI, ob = blockIdx.y * TR;
  const int i0 = ib + tx * 4, o0 = ob + ty * R;
  const bool vec = ((in & 3) == 0) && (i0 + 3 < in);
  const bool xvec = (x_ld & 3) == 0;
  float4 pw[R], pv[R];
  if (w) {  // the update's operands, in flight during the FMA loop
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int o = o0 + r;
      if (o < out && vec) {
        pw[r] = __ldcs((const float4*)(w + (size_t)o * in + i0));
        pv[r] = __ldcs((const float4*)(vel + (size_t)o * in + i0));
      }
    }
  }
  float acc[R][4];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.f;
  for (int b0 = 0; b0 < B; b0 += DS_KC) {
    const int bc = min(DS_KC, B - b0);
    if (xvec) {
      for (int e = threadIdx.x; e < bc * (DS_TI / 4); e += 256) {
        const int bb = e / (DS_TI / 4), q = e % (DS_TI / 4), i = ib + q * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i + 3 < x_ld) v = ld4f(x + (size_t)(b0 + bb) * x_ld + i);
        *(float4*)&Xs[bb][q * 4] = v;
      }
    } else {
      for (int e = threadIdx.x; e < bc * DS_TI; e += 256) {
        const int bb = e / DS_TI, ii = e % DS_TI, i = ib + ii;
        Xs[bb][ii] = i < in ? ldf(x, (size_t)(b0 + bb) * x_ld + i) : 0.f;
      }
    }
    for (int e = threadIdx.x; e < bc * TR; e += 256) {
      const int bb = e / TR, oo = e % TR, o = ob + oo;
      Gs[bb][oo] = o < out ? g[(size_t)(b0 + bb) * out + o] : 0.f;
    }
    __syncthreads();
    for (int bb = 0; bb < bc; ++bb) {
      const float4 xv = *(const float4*)&Xs[bb][tx * 4];
      float gr[R];
#pragma unroll
      for (int h = 0; h < R / 4; ++h) {
        const float4 gv = *(const float4*)&Gs[bb][ty * R + 4 * h];
        gr[4 * h] = gv.x; gr[4 * h + 1] = gv.y; gr[4 * h + 2] = gv.z; gr[4 * h + 3] = gv.w;
      }
      fma_rx4<R>(acc, gr, xv);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int o = o0 + r;
    if (o >= out || i0 >= in) continue;
    const size_t off = (size_t)o * in + i0;
    if (vec) {
      if (gw) __stcs((float4*)(gw + off), make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]));
      if (!w) continue;
      sgd_update(pw[r].x, pv[r].x, acc[r][0], lr, mu);
      sgd_update(pw[r].y, pv[r].y, acc[r][1], lr, mu);
      sgd_update(pw[r].z, pv[r].z, acc[r][2], lr, mu);
      sgd_update(pw[r].w, pv[r].w, acc[r][3], lr, mu);
      __stcs((float4*)(w + off), pw[r]);
      __stcs((float4*)(vel + off), pv[r]);
      if (wb) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(pw[r].x, pw[r].y), hi = __floats2bfloat162_rn(pw[r].z, pw[r].w);
        uint2 u;
        u.x = *(const uint32_t*)&lo;
        u.y = *(const uint32_t*)&hi;
        *(uint2*)(wb + (size_t)o * wb_ld + i0) = u;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (i0 + j >= in) break;
        if (gw) gw[off + j] = acc[r][j];
        if (!w) continue;
        float wv = w[off + j], vv = vel[off + j];
        sgd_update(wv, vv, acc[r][j], lr, mu);
        w[off + j] = wv;
        vel[off + j] = vv;
        if (wb) wb[(size_t)o * wb_ld + i0 + j] = __float2bfloat16_rn(wv);
      }
    }
  }
}

// Strip variant of the dW + SGD pass for wide layers: a CTA owns a 64-column
// strip of W, stages x[:, strip] in shared memory ONCE, and walks its range of
// rows in 64-row chunks (g staged per chunk). The per-tile kernel above refills
// the same x strip for every 16-row tile, which costs as much L2->SM traffic as
// W itself. Thread (cq = tid % 16, rg = tid / 16) owns 4 rows x 4 columns per
// chunk; accumulation order (b ascending) is the tile kernel's, so the results
// are bit-identical. grid (in / 64, row splits); in % 4 == 0, x_ld % 4 == 0.
constexpr int DSS_TI = 64, DSS_TR = 64, DSS_MAXB = 64;
template <class TX>
__global__ void __launch_bounds__(256)
    dense_dw_sgd_strip_kernel(const TX* __restrict__ x, int x_ld, const float* __restrict__ g, int B, int in,
                              int out, int rows_per_split, float* __restrict__ w, float* __restrict__ vel,
                              float* __restrict__ gw, bf16* __restrict__ wb, int wb_ld, float lr, float mu) {
  extern __shared__ __align__(16) float dss_smem[];
  float* Xs = dss_smem;               // [B][64]
  float* Gs = dss_smem + B * DSS_TI;  // [B][64]
  const int cq = threadIdx.x & 15, rg = threadIdx.x >> 4;
  const int ib = blockIdx.x * DSS_TI, i0 = ib + cq * 4;
  const bool colok = i0 < in;  // in % 4 == 0: a quad is all in or all out
  for (int e = threadIdx.x; e < B * (DSS_TI / 4); e += 256) {
    const int bb = e / (DSS_TI / 4), q = e % (DSS_TI / 4), i = ib + q * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < in) v = ld4f(x + (size_t)bb * x_ld + i);
    *(float4*)&Xs[bb * DSS_TI + q * 4] = v;
  }
  const int o_begin = blockIdx.y * rows_per_split, o_end = min(out, o_begin + rows_per_split);
  for (int oc = o_begin; oc < o_end; oc += DSS_TR) {
    const int o0 = oc + rg * 4;
    float4 pw[4], pv[4];
    if (w && colok) {  // the update's operands, in flight during the staging and FMA loop
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (o0 + r < o_end) {
          pw[r] = __ldcs((const float4*)(w + (size_t)(o0 + r) * in + i0));
          pv[r] = __ldcs((const float4*)(vel + (size_t)(o0 + r) * in + i0));
        }
    }
    __syncthreads();  // previous chunk's Gs reads done (first pass: Xs staged)
    for (int e = threadIdx.x; e < B * DSS_TR; e += 256) {
      const int bb = e / DSS_TR, oo = e % DSS_TR, o = oc + oo;
      Gs[bb * DSS_TR + oo] = o < o_end ? g[(size_t)bb * out + o] : 0.f;
    }
    __syncthreads();
    float acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.f;
#pragma unroll 4
    for (int bb = 0; bb < B; ++bb) {
      const float4 xv = *(const float4*)&Xs[bb * DSS_TI + cq * 4];
      const float4 gv = *(const float4*)&Gs[bb * DSS_TR + rg * 4];
      const float gr[4] = {gv.x, gv.y, gv.z, gv.w};
      fma_rx4<4>(acc, gr, xv);
    }
    if (!colok) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int o = o0 + r;
      if (o >= o_end) break;
      const size_t off = (size_t)o * in + i0;
      if (gw) __stcs((float4*)(gw + off), make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]));
      if (!w) continue;
      sgd_update(pw[r].x, pv[r].x, acc[r][0], lr, mu);
      sgd_update(pw[r].y, pv[r].y, acc[r][1], lr, mu);
      sgd_update(pw[r].z, pv[r].z, acc[r][2], lr, mu);
      sgd_update(pw[r].w, pv[r].w, acc[r][3], lr, mu);
      __stcs((float4*)(w + off), pw[r]);
      __stcs((float4*)(vel + off), pv[r]);
      if (wb) {
        const __nv_bfloat162 lo = __floats2bfloat162_rn(pw[r].x, pw[r].y),
                             hi = __floats2bfloat162_rn(pw[r].z, pw[r].w);
        uint2 u;
        u.x = *(const uint32_t*)&lo;
        u.y = *(const uint32_t*)&hi;
        *(uint2*)(wb + (size_t)o * wb_ld + i0) = u;
      }
    }
  }
}

inline bool dense_dw_strip_disabled() {  // CE_DENSE_DW_STRIP=0: per-tile kernel (comparison)
  static const bool off = [] {
    const char* e = getenv("CE_DENSE_DW_STRIP");
    return e && e[0] == '0';
  }();
  return off;
}

// dX[b][i] = sum_o g[b][o] w[o][i] (pre-update weights), gated by (mask > 0).
// grid (cdiv(B, 32), cdiv(in, 256)): blocks sharing a W tile run back to back.
template <class TO, class TM>
__global__ void __launch_bounds__(256, 2)
    dense_dx_simt_kernel(const float* __restrict__ g, const float* __restrict__ w, int B, int in, int out,
                         const TM* __restrict__ mask, TO* __restrict__ dx) {
  __shared__ __align__(16) float Ws[DS_KC][DS_TI];
  __shared__ __align__(16) float Gs[DS_KC][DS_TR];
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int bb0 = blockIdx.x * DS_TR, ib = blockIdx.y * DS_TI;
  const int i0 = ib + tx * 4, b0 = bb0 + ty * 8;
  const bool vec_in = (in & 3) == 0;
  float acc[8][4];
#pragma unroll
  for (int r = 0; r < 8; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.f;
  for (int oc = 0; oc < out; oc += DS_KC) {
    const int n = min(DS_KC, out - oc);
    if (vec_in) {
      for (int e = threadIdx.x; e < n * (DS_TI / 4); e += 256) {
        const int oo = e / (DS_TI / 4), q = e % (DS_TI / 4), i = ib + q * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < in) v = *(const float4*)(w + (size_t)(oc + oo) * in + i);
        *(float4*)&Ws[oo][q * 4] = v;
      }
    } else {
      for (int e = threadIdx.x; e < n * DS_TI; e += 256) {
        const int oo = e / DS_TI, ii = e % DS_TI, i = ib + ii;
        Ws[oo][ii] = i < in ? w[(size_t)(oc + oo) * in + i] : 0.f;
      }
    }
    for (int e = threadIdx.x; e < n * DS_TR; e += 256) {
      const int oo = e / DS_TR, bl = e % DS_TR, b = bb0 + bl;
      Gs[oo][bl] = b < B ? g[(size_t)b * out + oc + oo] : 0.f;
    }
    __syncthreads();
    for (int oo = 0; oo < n; ++oo) {
      const float4 wv = *(const float4*)&Ws[oo][tx * 4];
      const float4 ga = *(const float4*)&Gs[oo][ty * 8], gb = *(const float4*)&Gs[oo][ty * 8 + 4];
      const float g8[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
      fma8x4(acc, g8, wv);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int b = b0 + r;
    if (b >= B) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + j;
      if (i >= in) break;
      const size_t off = (size_t)b * in + i;
      float v = acc[r][j];
      if (mask && !(ldf(mask, off) > 0.f)) v = 0.f;
      stf(dx, off, v);
    }
  }
}

// Same dX tile with the next 32-output chunk of W / G fetched into registers while
// the current one is consumed (double-buffered shared memory, one barrier per
// chunk); used when in % 4 == 0 (float4 rows of W).
constexpr int DXP_SMEM = 2 * (DS_KC * DS_TI + DS_KC * DS_TR) * 4;
template <class TO, class TM>
__global__ void __launch_bounds__(256, 2)
    dense_dx_simt_pipe_kernel(const float* __restrict__ g, const float* __restrict__ w, int B, int in, int out,
                              const TM* __restrict__ mask, TO* __restrict__ dx) {
  extern __shared__ __align__(16) float dxs[];
  float* const gs0 = dxs + 2 * DS_KC * DS_TI;
  const int tid = threadIdx.x, tx = tid & 63, ty = tid >> 6;
  const int bb0 = blockIdx.x * DS_TR, ib = blockIdx.y * DS_TI;
  const int i0 = ib + tx * 4, b0 = bb0 + ty * 8;
  float4 rw[8];
  float rg[4];
  auto fetch = [&](int oc) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // e = tid + 256 j -> (oo = e / 64, q = e % 64)
      const int e = tid + 256 * j, oo = e >> 6, q = e & 63, i = ib + q * 4;
      rw[j] = (oc + oo < out && i < in) ? *(const float4*)(w + (size_t)(oc + oo) * in + i)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // e = tid + 256 j -> (oo = e / 32, bl = e % 32)
      const int e = tid + 256 * j, oo = e >> 5, bl = e & 31, b = bb0 + bl;
      rg[j] = (oc + oo < out && b < B) ? g[(size_t)b * out + oc + oo] : 0.f;
    }
  };
  auto stash = [&](int buf) {
    float* W = dxs + buf * (DS_KC * DS_TI);
    float* G = gs0 + buf * (DS_KC * DS_TR);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = tid + 256 * j;
      *(float4*)(W + (e >> 6) * DS_TI + (e & 63) * 4) = rw[j];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int e = tid + 256 * j;
      G[(e >> 5) * DS_TR + (e & 31)] = rg[j];
    }
  };
  float acc[8][4];
#pragma unroll
  for (int r = 0; r < 8; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.f;
  fetch(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (int oc = 0; oc < out; oc += DS_KC) {
    const bool more = oc + DS_KC < out;
    if (more) fetch(oc + DS_KC);
    const float* W = dxs + buf * (DS_KC * DS_TI);
    const float* G = gs0 + buf * (DS_KC * DS_TR);
    const int n = min(DS_KC, out - oc);
#pragma unroll 4
    for (int oo = 0; oo < n; ++oo) {
      const float4 wv = *(const float4*)(W + oo * DS_TI + tx * 4);
      const float4 ga = *(const float4*)(G + oo * DS_TR + ty * 8), gb = *(const float4*)(G + oo * DS_TR + ty * 8 + 4);
      const float g8[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
      fma8x4(acc, g8, wv);
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int b = b0 + r;
    if (b >= B) continue;
    const size_t off = (size_t)b * in + i0;
    if (i0 + 3 < in) {
      float v[4] = {acc[r][0], acc[r][1], acc[r][2], acc[r][3]};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (mask && !(ldf(mask, off + j) > 0.f)) v[j] = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) stf(dx, off + j, v[j]);
    } else {
      for (int j = 0; j < 4 && i0 + j < in; ++j) {
        float v = acc[r][j];
        if (mask && !(ldf(mask, off + j) > 0.f)) v = 0.f;
        stf(dx, off + j, v);
      }
    }
  }
}

// Split-K dense forward on CUDA cores (fp32 check mode, small batch):
// part[split][b][o] = sum over the split's k-range of x[b][k] W[o][k].
// Block = 64R outputs x 32 rows, 256 threads: warp w takes rows 8 (w % 4) .. +7
// and output half w / 4; lane -> R outputs (o = half * 32R + lane + 32 j). Each
// W value read from shared memory (per-lane rows: 4 wavefronts per float4)
// feeds 8 rows of FMAs -- at 4 rows per thread the W reads alone saturate
// shared memory. W is staged [o][k] with a 36-float stride (conflict-free fill
// from float4 rows and conflict-free per-lane reads), x is staged [k][b] and
// read as warp-uniform float4 broadcasts; the next K chunk is fetched into
// registers while the current one is consumed (one barrier per chunk).
constexpr int DF_TB = 32, DF_KC = 32, DF_WS = DF_KC + 4, DF_XS = DF_TB + 4;
template <int R>
constexpr int df_smem() { return 2 * (64 * R * DF_WS + DF_KC * DF_XS) * 4; }
// R outputs per lane: block tile 64R outputs (R chosen per layer to limit padding)
template <class TX, int R>
__global__ void __launch_bounds__(256, 2) dense_fwd_simt_kernel(const TX* __restrict__ x, const float* __restrict__ w,
                                                                int B, int in, int out, int kchunk,
                                                                float* __restrict__ part) {
  constexpr int DF_TO = 64 * R;
  extern __shared__ __align__(16) float dsm[];
  // buffer b: W at dsm + b * DF_TO * DF_WS, x at xs0 + b * DF_KC * DF_XS
  float* const xs0 = dsm + 2 * DF_TO * DF_WS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rgp = warp & 3, oh = warp >> 2;
  const int ob = blockIdx.x * DF_TO, bb = blockIdx.y * DF_TB;
  const int k0 = blockIdx.z * kchunk, k1 = min(in, k0 + kchunk);
  const bool kvec = (in & 3) == 0;
  // fetch mapping: W: 2R float4 per thread (row = tid/8 + 32 i, kq = tid % 8); x: 1 float4 (b = tid/8)
  const int frow = tid >> 3, fkq = tid & 7;
  float4 rw[2 * R], rx;
  auto fetch = [&](int kc) {
    const int k = kc + fkq * 4;
#pragma unroll
    for (int i = 0; i < 2 * R; ++i) {
      const int o = ob + frow + 32 * i;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (o < out) {
        const float* src = w + (size_t)o * in;
        if (kvec && k + 3 < k1) {
          v = *(const float4*)(src + k);
        } else {
          v.x = k < k1 ? src[k] : 0.f;
          v.y = k + 1 < k1 ? src[k + 1] : 0.f;
          v.z = k + 2 < k1 ? src[k + 2] : 0.f;
          v.w = k + 3 < k1 ? src[k + 3] : 0.f;
        }
      }
      rw[i] = v;
    }
    const int b = bb + frow;
    rx = make_float4(0.f, 0.f, 0.f, 0.f);
    if (b < B) {
      const TX* src = x + (size_t)b * in;
      rx.x = k < k1 ? ldf(src, k) : 0.f;
      rx.y = k + 1 < k1 ? ldf(src, k + 1) : 0.f;
      rx.z = k + 2 < k1 ? ldf(src, k + 2) : 0.f;
      rx.w = k + 3 < k1 ? ldf(src, k + 3) : 0.f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 2 * R; ++i)
      *(float4*)(dsm + buf * (DF_TO * DF_WS) + (frow + 32 * i) * DF_WS + fkq * 4) = rw[i];
    float* d = xs0 + buf * (DF_KC * DF_XS) + (fkq * 4) * DF_XS + frow;
    d[0] = rx.x; d[DF_XS] = rx.y; d[2 * DF_XS] = rx.z; d[3 * DF_XS] = rx.w;
  };
  float acc[R][8];
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[j][r] = 0.f;
  if (k0 < k1) {
    fetch(k0);
    stash(0);
  }
  __syncthreads();
  int buf = 0;
  for (int kc = k0; kc < k1; kc += DF_KC) {
    const bool more = kc + DF_KC < k1;
    if (more) fetch(kc + DF_KC);
    const float* W = dsm + buf * (DF_TO * DF_WS) + (oh * 32 * R + lane) * DF_WS;
    const float* X = xs0 + buf * (DF_KC * DF_XS) + rgp * 8;
#pragma unroll 2
    for (int kk = 0; kk < DF_KC; kk += 4) {
      float4 wq[R];
#pragma unroll
      for (int j = 0; j < R; ++j) wq[j] = *(const float4*)(W + 32 * j * DF_WS + kk);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4 xa = *(const float4*)(X + (kk + u) * DF_XS), xb = *(const float4*)(X + (kk + u) * DF_XS + 4);
        const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const float wv = u == 0 ? wq[j].x : u == 1 ? wq[j].y : u == 2 ? wq[j].z : wq[j].w;
#pragma unroll
          for (int r = 0; r < 8; ++r) acc[j][r] = fmaf(xv[r], wv, acc[j][r]);
        }
      }
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  float* dst = part + (size_t)blockIdx.z * B * out;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int b = bb + rgp * 8 + r;
    if (b >= B) break;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int o = ob + oh * 32 * R + lane + 32 * j;
      if (o < out) dst[(size_t)b * out + o] = acc[j][r];
    }
  }
}

// CE_DENSE_FWD_GEMM=1 keeps the generic SIMT GEMM for the fp32 dense forward (comparison)
inline bool dense_fwd_simt_enabled() {
  static const bool off = [] {
    const char* e = getenv("CE_DENSE_FWD_GEMM");
    return e && e[0] == '1';
  }();
  return !off;
}

// outputs per lane minimising padded outputs (ties -> larger tiles)
inline int dense_fwd_simt_r(int out) {
  int best = 4;
  long long best_pad = -1;
  for (int r : {4, 3, 2}) {
    const long long pad = (long long)((out + 64 * r - 1) / (64 * r)) * 64 * r;
    if (best_pad < 0 || pad < best_pad) best_pad = pad, best = r;
  }
  return best;
}

inline int dense_fwd_simt_splits(int B, int in, int out, int num_sms) {
  const int to = 64 * dense_fwd_simt_r(out);
  const long long blocks = (long long)((out + to - 1) / to) * ((B + DF_TB - 1) / DF_TB);
  long long s = (2LL * num_sms + blocks - 1) / blocks;
  const long long cap = (in + 255) / 256;
  if (s > cap) s = cap;
  if (s > 256) s = 256;
  return s < 1 ? 1 : (int)s;
}

template <class TX, int R>
inline int dense_fwd_simt_r_launch(const TX* x, const float* w, int B, int in, int out, int splits, float* part,
                                   cudaStream_t st) {
  cudaFuncSetAttribute(dense_fwd_simt_kernel<TX, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, df_smem<R>());
  const int kchunk = ((in + splits - 1) / splits + DF_KC - 1) / DF_KC * DF_KC;
  const int s = (in + kchunk - 1) / kchunk;
  dim3 grid((out + 64 * R - 1) / (64 * R), (B + DF_TB - 1) / DF_TB, s);
  dense_fwd_simt_kernel<TX, R><<<grid, 256, df_smem<R>(), st>>>(x, w, B, in, out, kchunk, part);
  return s;
}

template <class TX>
inline int dense_fwd_simt(const TX* x, const float* w, int B, int in, int out, int splits, float* part,
                          cudaStream_t st) {
  switch (dense_fwd_simt_r(out)) {
    case 2: return dense_fwd_simt_r_launch<TX, 2>(x, w, B, in, out, splits, part, st);
    case 3: return dense_fwd_simt_r_launch<TX, 3>(x, w, B, in, out, splits, part, st);
    default: return dense_fwd_simt_r_launch<TX, 4>(x, w, B, in, out, splits, part, st);
  }
}

// ------------------------------------------------------------------ streaming-W FFMA (fp32 check mode)
// Wide fp32 layers at small batch (C2 #15: 262144 -> 523 at B = 32) are bound by the
// FMA pipe, not HBM: 2 FMAs per weight per row. These kernels give every weight to
// exactly one thread, straight from HBM into registers (prefetched one chunk ahead),
// and keep the small operand (x or the output gradient) in shared memory, read as
// warp-uniform float4 broadcasts: 8 FMAs per shared-memory load.
constexpr int DW_KC = 16;     // k per chunk
constexpr int DW_THREADS = 64;

// part[split][b][o] = sum over the split's k-range of x[b][k] w[o][k]; thread -> outputs
// o = base + tid + 64 j (j < 2), all BR rows of a row block
template <int BR>
__global__ void __launch_bounds__(DW_THREADS) dense_fwd_stream_kernel(const float* __restrict__ x,
                                                                      const float* __restrict__ w, int B, int in,
                                                                      int out, int kchunk, float* __restrict__ part) {
  constexpr int R = 2, XS = DW_KC + 4;
  __shared__ __align__(16) float xs[2][BR][XS];
  const int tid = threadIdx.x;
  const int ob = blockIdx.x * (DW_THREADS * R), bb = blockIdx.y * BR;
  const int k0 = blockIdx.z * kchunk, k1 = min(in, k0 + kchunk);
  float4 wc[R][DW_KC / 4], wn[R][DW_KC / 4];
  float acc[R][BR];
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int b = 0; b < BR; ++b) acc[j][b] = 0.f;
  auto fetch_w = [&](int kc, float4 (&dst)[R][DW_KC / 4]) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int o = ob + tid + DW_THREADS * j;
#pragma unroll
      for (int q = 0; q < DW_KC / 4; ++q) {
        const int k = kc + 4 * q;
        dst[j][q] = (o < out && k < k1) ? __ldcs((const float4*)(w + (size_t)o * in + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
  auto fetch_x = [&](int kc, int buf) {  // BR rows x 16 k: 4*BR float4, DW_THREADS threads
    for (int e = tid; e < BR * (DW_KC / 4); e += DW_THREADS) {
      const int r = e / (DW_KC / 4), q = e % (DW_KC / 4), k = kc + 4 * q, b = bb + r;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (b < B && k < k1) v = *(const float4*)(x + (size_t)b * in + k);
      *(float4*)&xs[buf][r][4 * q] = v;
    }
  };
  int buf = 0;
  if (k0 < k1) {
    fetch_w(k0, wc);
    fetch_x(k0, 0);
  }
  __syncthreads();
  for (int kc = k0; kc < k1; kc += DW_KC) {
    const bool more = kc + DW_KC < k1;
    if (more) fetch_w(kc + DW_KC, wn);
#pragma unroll
    for (int q = 0; q < DW_KC / 4; ++q) {
#pragma unroll
      for (int b = 0; b < BR; ++b) {
        const float4 xv = *(const float4*)&xs[buf][b][4 * q];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          float a = acc[j][b];
          a = fmaf(xv.x, wc[j][q].x, a);
          a = fmaf(xv.y, wc[j][q].y, a);
          a = fmaf(xv.z, wc[j][q].z, a);
          a = fmaf(xv.w, wc[j][q].w, a);
          acc[j][b] = a;
        }
      }
    }
    if (more) fetch_x(kc + DW_KC, buf ^ 1);
    __syncthreads();
    buf ^= 1;
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int q = 0; q < DW_KC / 4; ++q) wc[j][q] = wn[j][q];
  }
  float* dst = part + (size_t)blockIdx.z * B * out;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int o = ob + tid + DW_THREADS * j;
    if (o >= out) continue;
#pragma unroll
    for (int b = 0; b < BR; ++b)
      if (bb + b < B) dst[(size_t)(bb + b) * out + o] = acc[j][b];
  }
}

// dx[b][i] = sum_o g[b][o] w[o][i] (pre-update weights), gated by (mask > 0): thread -> inputs
// i, i+1 (float2 of every weight row, coalesced across the warp), all BR rows
template <int BR, class TM>
__global__ void __launch_bounds__(DW_THREADS) dense_dx_stream_kernel(const float* __restrict__ g,
                                                                     const float* __restrict__ w, int B, int in,
                                                                     int out, const TM* __restrict__ mask,
                                                                     float* __restrict__ dx) {
  constexpr int GS = DW_KC + 4;
  __shared__ __align__(16) float gs[2][BR][GS];
  const int tid = threadIdx.x;
  const int i = blockIdx.x * (2 * DW_THREADS) + 2 * tid, bb = blockIdx.y * BR;
  const bool ok = i + 1 < in;  // in % 2 == 0 (caller)
  float2 wc[DW_KC], wn[DW_KC];
  float acc[2][BR];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int b = 0; b < BR; ++b) acc[u][b] = 0.f;
  auto fetch_w = [&](int oc, float2 (&dst)[DW_KC]) {
#pragma unroll
    for (int q = 0; q < DW_KC; ++q) {
      const int o = oc + q;
      dst[q] = (ok && o < out) ? __ldcs((const float2*)(w + (size_t)o * in + i)) : make_float2(0.f, 0.f);
    }
  };
  auto fetch_g = [&](int oc, int buf) {
    for (int e = tid; e < BR * DW_KC; e += DW_THREADS) {
      const int r = e / DW_KC, q = e % DW_KC, o = oc + q, b = bb + r;
      gs[buf][r][q] = (b < B && o < out) ? g[(size_t)b * out + o] : 0.f;
    }
  };
  int buf = 0;
  fetch_w(0, wc);
  fetch_g(0, 0);
  __syncthreads();
  for (int oc = 0; oc < out; oc += DW_KC) {
    const bool more = oc + DW_KC < out;
    if (more) fetch_w(oc + DW_KC, wn);
#pragma unroll
    for (int q = 0; q < DW_KC / 4; ++q) {
#pragma unroll
      for (int b = 0; b < BR; ++b) {
        const float4 gv = *(const float4*)&gs[buf][b][4 * q];
        float a0 = acc[0][b], a1 = acc[1][b];
        a0 = fmaf(gv.x, wc[4 * q].x, a0);
        a1 = fmaf(gv.x, wc[4 * q].y, a1);
        a0 = fmaf(gv.y, wc[4 * q + 1].x, a0);
        a1 = fmaf(gv.y, wc[4 * q + 1].y, a1);
        a0 = fmaf(gv.z, wc[4 * q + 2].x, a0);
        a1 = fmaf(gv.z, wc[4 * q + 2].y, a1);
        a0 = fmaf(gv.w, wc[4 * q + 3].x, a0);
        a1 = fmaf(gv.w, wc[4 * q + 3].y, a1);
        acc[0][b] = a0;
        acc[1][b] = a1;
      }
    }
    if (more) fetch_g(oc + DW_KC, buf ^ 1);
    __syncthreads();
    buf ^= 1;
#pragma unroll
    for (int q = 0; q < DW_KC; ++q) wc[q] = wn[q];
  }
  if (!ok) return;
#pragma unroll
  for (int b = 0; b < BR; ++b) {
    if (bb + b >= B) break;
    const size_t off = (size_t)(bb + b) * in + i;
    float v0 = acc[0][b], v1 = acc[1][b];
    if (mask) {
      if (!(ldf(mask, off) > 0.f)) v0 = 0.f;
      if (!(ldf(mask, off + 1) > 0.f)) v1 = 0.f;
    }
    *(float2*)(dx + off) = make_float2(v0, v1);
  }
}

// fp32 layers that take the streaming kernels: wide (>= 1 M weights), B <= 64, rows of
// 16 B (in % 4 == 0). Opt-in (CE_DENSE_STREAM=1): on C2 #15 (262144 -> 523, B = 32) they
// measured slower than the tiled kernels (forward 413 vs 335 us, backward 812 vs 703 us):
// the per-lane weight rows scatter every warp load over 32 DRAM rows.
inline bool dense_stream_enabled(int B, int in, long long params) {
  static const bool on = [] {
    const char* e = getenv("CE_DENSE_STREAM");
    return e && e[0] == '1';
  }();
  return on && B <= 64 && (in & 3) == 0 && params >= (1ll << 20);
}
inline int dense_fwd_stream_splits(int B, int in, int out, int num_sms) {
  const long long blocks = (long long)((out + 2 * DW_THREADS - 1) / (2 * DW_THREADS)) * ((B + 31) / 32);
  long long s = (6LL * num_sms + blocks - 1) / blocks;  // ~6 resident 64-thread CTAs per SM
  const long long cap = (in + 255) / 256;
  if (s > cap) s = cap;
  if (s > 512) s = 512;
  return s < 1 ? 1 : (int)s;
}
// returns the split count written to part
inline int dense_fwd_stream(const float* x, const float* w, int B, int in, int out, int splits, float* part,
                            cudaStream_t st) {
  const int kchunk = ((in + splits - 1) / splits + DW_KC - 1) / DW_KC * DW_KC;
  const int s = (in + kchunk - 1) / kchunk;
  if (B <= 16) {
    dim3 grid((out + 2 * DW_THREADS - 1) / (2 * DW_THREADS), (B + 15) / 16, s);
    dense_fwd_stream_kernel<16><<<grid, DW_THREADS, 0, st>>>(x, w, B, in, out, kchunk, part);
  } else {
    dim3 grid((out + 2 * DW_THREADS - 1) / (2 * DW_THREADS), (B + 31) / 32, s);
    dense_fwd_stream_kernel<32><<<grid, DW_THREADS, 0, st>>>(x, w, B, in, out, kchunk, part);
  }
  return s;
}
template <class TM>
inline void dense_dx_stream(const float* g, const float* w, int B, int in, int out, const TM* mask, float* dx,
                            cudaStream_t st) {
  if (B <= 16) {
    dim3 grid((in + 2 * DW_THREADS - 1) / (2 * DW_THREADS), (B + 15) / 16);
    dense_dx_stream_kernel<16, TM><<<grid, DW_THREADS, 0, st>>>(g, w, B, in, out, mask, dx);
  } else {
    dim3 grid((in + 2 * DW_THREADS - 1) / (2 * DW_THREADS), (B + 31) / 32);
    dense_dx_stream_kernel<32, TM><<<grid, DW_THREADS, 0, st>>>(g, w, B, in, out, mask, dx);
  }
}

// fp32 check mode: these kernels up to B = 64, the generic SIMT GEMM above.
constexpr int kDenseSimtMaxBatch = 64;
// bf16: measured on B200 (C2 heads, 51-137 M params): the FFMA dW+SGD pass
// beats the tcgen05 one up to B = 32 (191 vs 273 us at B = 16) and loses at
// B = 64 (289 vs 247 us), where 64 FMAs/param start to cost.
constexpr int kDenseDwSimtMaxBatchBf16 = 32;

// bf16 runtime: dense dW + SGD on CUDA cores for small batches unless
// CE_DENSE_DW_TC=1 forces the tcgen05 pass (kept for comparison).
inline bool dense_dw_simt_enabled(int B) {
  static const bool force_tc = [] {
    const char* e = getenv("CE_DENSE_DW_TC");
    return e && e[0] == '1';
  }();
  static const int maxb = [] {  // CE_DENSE_DW_SIMT_MAXB=N moves the crossover (measurement)
    const char* e = getenv("CE_DENSE_DW_SIMT_MAXB");
    return e ? atoi(e) : kDenseDwSimtMaxBatchBf16;
  }();
  return !force_tc && B <= maxb;
}

inline int dense_dw_rows() {  // rows per thread (CE_DENSE_DW_ROWS = 4 | 8)
  static const int r = [] {
    const char* e = getenv("CE_DENSE_DW_ROWS");
    return (e && e[0] == '8') ? 8 : 4;
  }();
  return r;
}

template <class TX>
inline void dense_dw_sgd_simt(const TX* x, int x_ld, const float* g, int B, int in, int out, float* w, float* vel,
                              float* gw, bf16* wb, int wb_ld, float lr, float mu, cudaStream_t st) {
  if (!dense_dw_strip_disabled() && (in & 3) == 0 && (x_ld & 3) == 0 && B <= DSS_MAXB) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int strips = cdiv(in, DSS_TI), chunks = cdiv(out, DSS_TR);
    const int splits = std::max(1, std::min(chunks, cdiv(6 * sms, strips)));  // >= ~6 CTAs per SM
    const int rows = cdiv(chunks, splits) * DSS_TR;
    const int smem = 2 * B * DSS_TI * (int)sizeof(float);
    dense_dw_sgd_strip_kernel<TX><<<dim3(strips, cdiv(out, rows)), 256, smem, st>>>(
        x, x_ld, g, B, in, out, rows, w, vel, gw, wb, wb_ld, lr, mu);
    return;
  }
  if (dense_dw_rows() == 8) {
    dim3 grid(cdiv(in, DS_TI), cdiv(out, 32));
    dense_dw_sgd_simt_kernel<TX, 8><<<grid, 256, 0, st>>>(x, x_ld, g, B, in, out, w, vel, gw, wb, wb_ld, lr, mu);
  } else {
    dim3 grid(cdiv(in, DS_TI), cdiv(out, 16));
    dense_dw_sgd_simt_kernel<TX, 4><<<grid, 256, 0, st>>>(x, x_ld, g, B, in, out, w, vel, gw, wb, wb_ld, lr, mu);
  }
}

template <class TO, class TM>
inline void dense_dx_simt(const float* g, const float* w, int B, int in, int out, const TM* mask, TO* dx,
                          cudaStream_t st) {
  dim3 grid(cdiv(B, DS_TR), cdiv(in, DS_TI));
  if ((in & 3) == 0) {
    // per device (a process may drive several GPUs): set on every launch, it is cheap
    cudaFuncSetAttribute(dense_dx_simt_pipe_kernel<TO, TM>, cudaFuncAttributeMaxDynamicSharedMemorySize, DXP_SMEM);
    dense_dx_simt_pipe_kernel<TO, TM><<<grid, 256, DXP_SMEM, st>>>(g, w, B, in, out, mask, dx);
    return;
  }
  dense_dx_simt_kernel<TO, TM><<<grid, 256, 0, st>>>(g, w, B, in, out, mask, dx);
}

}  // namespace ce
