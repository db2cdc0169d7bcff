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
  return !force_tc && B <= kDenseDwSimtMaxBatchBf16;
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
  dense_dx_simt_kernel<TO, TM><<<grid, 256, 0, st>>>(g, w, B, in, out, mask, dx);
}

}  // namespace ce
