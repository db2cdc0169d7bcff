// Fused classifier head: the final Dense(in -> classes) layer of every genome
// (genome.py:330-335 appends Dense(., 2)) together with the loss.
//
// As separate passes the head costs 3 launches forward (split-K GEMM, reduce,
// softmax-xent) and 5 backward (bf16 copy of dL/dlogits, dX, dW + SGD, bias
// column sum, bias SGD) for a layer with a handful of output rows: the work is
// a single stream over x (and W), so each direction becomes one kernel.
//   forward  logits = x W^T + b (nn.py:225-231) and, when training, the
//            softmax cross-entropy (nn.py:287-303): CTAs own input chunks (W
//            staged in shared memory, a warp per batch row), write partials,
//            and the last CTA to finish (device ticket, fixed summation order)
//            adds the bias, writes the logits and runs the loss exactly as
//            xent_kernel does (loss into losses[step], step counter, non-finite flag).
//   backward dX = g W (pre-update weights, nn.py:240) and dW = g^T x (nn.py:238)
//            from one read of x, with the momentum update of W / V fused
//            (nn.py:306-322); block 0 reduces and applies the bias update.
#pragma once
#include "ops.cuh"
#include "dense_simt.cuh"

namespace ce {

constexpr int kHeadMaxOut = 4;
// CE_DISABLE_HEAD=1 runs the final layer through the generic dense passes (comparison)
inline bool head_disabled() {
  static const bool off = [] {
    const char* e = getenv("CE_DISABLE_HEAD");
    return e && e[0] == '1';
  }();
  return off;
}
constexpr int kHeadMaxBatch = 256;
constexpr int kHeadFwdChunk = 2048;  // input columns per forward CTA
constexpr int kHeadRowsPerCta = 32;  // batch rows per forward CTA

template <class TX, int OUT>
__global__ void __launch_bounds__(256) head_fwd_kernel(const TX* __restrict__ x, int x_ld, const float* __restrict__ w,
                                                       const float* __restrict__ bias, int B, int in, int chunk,
                                                       float* __restrict__ partial, unsigned* __restrict__ ticket,
                                                       float* __restrict__ logits, const int32_t* __restrict__ labels,
                                                       float* __restrict__ grad, float* __restrict__ losses,
                                                       int* __restrict__ step_ctr, int* __restrict__ nonfinite) {
  __shared__ __align__(16) float Ws[OUT][kHeadFwdChunk];
  __shared__ double red[256];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = blockIdx.x * chunk, i1 = min(in, i0 + chunk), n = i1 - i0;
  // blockIdx.y: group of kHeadRowsPerCta batch rows (more CTAs when in is small)
  const int b_lo = blockIdx.y * kHeadRowsPerCta, b_hi = min(B, b_lo + kHeadRowsPerCta);
  for (int e = threadIdx.x; e < OUT * n; e += blockDim.x) {
    const int o = e / n, i = e % n;
    Ws[o][i] = w[(size_t)o * in + i0 + i];
  }
  __syncthreads();
  const bool vec = ((x_ld & 7) == 0) && ((i0 & 7) == 0);  // 8 consecutive columns per lane
  // two rows per warp pass (b, b + 8): 8 x-vector loads in flight per lane
  for (int b = b_lo + warp; b < b_hi; b += 16) {
    const bool two = b + 8 < b_hi;
    float acc[2][OUT];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int o = 0; o < OUT; ++o) acc[r][o] = 0.f;
    const TX* xr0 = x + (size_t)b * x_ld + i0;
    const TX* xr1 = x + (size_t)(two ? b + 8 : b) * x_ld + i0;
    if (vec) {
      const int n8 = n & ~7;
      for (int i = lane * 8; i < n8; i += 4 * 256) {
        float xv[2][4][8];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (i + q * 256 < n8) {
            load8(xr0 + i + q * 256, xv[0][q]);
            if (two) load8(xr1 + i + q * 256, xv[1][q]);
          }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (i + q * 256 >= n8) break;
          const int iq = i + q * 256;
#pragma unroll
          for (int o = 0; o < OUT; ++o) {
            const float4 wa = *(const float4*)&Ws[o][iq], wb = *(const float4*)&Ws[o][iq + 4];
            const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[0][o] = fmaf(xv[0][q][u], wv[u], acc[0][o]);
            if (two) {
#pragma unroll
              for (int u = 0; u < 8; ++u) acc[1][o] = fmaf(xv[1][q][u], wv[u], acc[1][o]);
            }
          }
        }
      }
      for (int i = n8 + lane; i < n; i += 32) {
        const float x0 = ldf(xr0, i), x1 = ldf(xr1, i);
#pragma unroll
        for (int o = 0; o < OUT; ++o) {
          acc[0][o] = fmaf(x0, Ws[o][i], acc[0][o]);
          acc[1][o] = fmaf(x1, Ws[o][i], acc[1][o]);
        }
      }
    } else {
      for (int i = lane; i < n; i += 32) {
        const float x0 = ldf(xr0, i), x1 = ldf(xr1, i);
#pragma unroll
        for (int o = 0; o < OUT; ++o) {
          acc[0][o] = fmaf(x0, Ws[o][i], acc[0][o]);
          acc[1][o] = fmaf(x1, Ws[o][i], acc[1][o]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (r == 1 && !two) break;
      const int br = b + 8 * r;
#pragma unroll
      for (int o = 0; o < OUT; ++o) {
        float v = acc[r][o];
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
        if (lane == 0) partial[(size_t)(br * OUT + o) * gridDim.x + blockIdx.x] = v;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int G = (int)gridDim.x, E = B * OUT;
  // [logit][cta] partials, lanes over consecutive CTAs; 8 logits per warp at once
  // (8 independent loads per lane per step), each summed in CTA order then by a
  // fixed xor tree (deterministic)
  for (int e0 = warp * 8; e0 < E; e0 += 64) {
    float s[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] = 0.f;
    for (int c = lane; c < G; c += 32) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (e0 + j < E) s[j] += __ldcg(partial + (size_t)(e0 + j) * G + c);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], m);
      if (lane == 0 && e0 + j < E) logits[e0 + j] = s[j] + bias[(e0 + j) % OUT];
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;  // ready for the next launch / graph replay
  if (!labels) return;
  __syncthreads();
  // softmax cross-entropy: same arithmetic as xent_kernel (nn.py:287-303)
  double lp = 0.0;
  const int b = threadIdx.x;
  if (b < B) {
    const float* z = logits + (size_t)b * OUT;
    float mx = z[0];
    for (int k = 1; k < OUT; ++k) mx = fmaxf(mx, z[k]);
    float se = 0.f;
    for (int k = 0; k < OUT; ++k) se += expf(z[k] - mx);
    const float lse = logf(se);
    const long long lab = (long long)labels[b];
    if (lab < 0 || lab >= OUT) lp = __longlong_as_double(0x7ff8000000000000ll);
    for (int k = 0; k < OUT; ++k) {
      const float logp = (z[k] - mx) - lse;
      float gk = expf(logp);
      if (k == lab) {
        gk -= 1.0f;
        lp = (double)logp;
      }
      grad[(size_t)b * OUT + k] = gk / (float)B;
    }
  }
  red[threadIdx.x] = lp;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int step = *step_ctr;
    const float loss = (float)(-red[0] / B);
    losses[step] = loss;
    if (nonfinite && !isfinite(loss)) *nonfinite = 1;
    *step_ctr = step + 1;
  }
}

__device__ __forceinline__ void st4(float* p, const float (&v)[4]) { *(float4*)p = make_float4(v[0], v[1], v[2], v[3]); }
__device__ __forceinline__ void st4(bf16* p, const float (&v)[4]) {
  const __nv_bfloat162 lo = __floats2bfloat162_rn(v[0], v[1]), hi = __floats2bfloat162_rn(v[2], v[3]);
  uint2 u;
  u.x = *(const uint32_t*)&lo;
  u.y = *(const uint32_t*)&hi;
  *(uint2*)p = u;
}

// one thread per 4 consecutive input columns; grid cdiv(in, 1024)
template <class TX, class TD, int OUT>
__global__ void __launch_bounds__(256) head_bwd_kernel(const TX* __restrict__ x, int x_ld, const float* __restrict__ g,
                                                       int B, int in, float* __restrict__ w, float* __restrict__ vel,
                                                       float* __restrict__ gw, TD* __restrict__ dx,
                                                       const TD* __restrict__ mask, float* __restrict__ b,
                                                       float* __restrict__ vb, float* __restrict__ gb, float lr,
                                                       float mu) {
  __shared__ float Gs[kHeadMaxBatch][OUT];
  for (int e = threadIdx.x; e < B * OUT; e += blockDim.x) Gs[e / OUT][e % OUT] = g[e];
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < OUT) {  // bias: sum over the batch in order
    const int o = threadIdx.x;
    float s = 0.f;
    for (int r = 0; r < B; ++r) s += Gs[r][o];
    if (gb) gb[o] = s;
    float bv = b[o], v = vb[o];
    sgd_update(bv, v, s, lr, mu);
    b[o] = bv;
    vb[o] = v;
  }
  const int i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i0 >= in) return;
  const int nj = min(4, in - i0);
  const bool wvec = ((in & 3) == 0) && nj == 4;
  const bool xvec = ((x_ld & 3) == 0) && nj == 4;
  const bool mask_x = mask && (const void*)mask == (const void*)x && x_ld == in;
  float wv[OUT][4], vv[OUT][4], acc[OUT][4];
#pragma unroll
  for (int o = 0; o < OUT; ++o) {
    const size_t off = (size_t)o * in + i0;
    if (wvec) {
      const float4 a = *(const float4*)(w + off), c = *(const float4*)(vel + off);
      wv[o][0] = a.x; wv[o][1] = a.y; wv[o][2] = a.z; wv[o][3] = a.w;
      vv[o][0] = c.x; vv[o][1] = c.y; vv[o][2] = c.z; vv[o][3] = c.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        wv[o][j] = j < nj ? w[off + j] : 0.f;
        vv[o][j] = j < nj ? vel[off + j] : 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[o][j] = 0.f;
  }
#pragma unroll 4
  for (int r = 0; r < B; ++r) {
    float xv[4];
    if (xvec) {
      const float4 t = ld4f(x + (size_t)r * x_ld + i0);
      xv[0] = t.x; xv[1] = t.y; xv[2] = t.z; xv[3] = t.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) xv[j] = j < nj ? ldf(x, (size_t)r * x_ld + i0 + j) : 0.f;
    }
    float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int o = 0; o < OUT; ++o) {
      const float gr = Gs[r][o];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[o][j] = fmaf(gr, xv[j], acc[o][j]);
        d[j] = fmaf(gr, wv[o][j], d[j]);
      }
    }
    if (dx) {
      const size_t off = (size_t)r * in + i0;
      if (mask_x && xvec) {  // the ReLU mask is this layer's input: reuse xv, one vector store
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (!(xv[j] > 0.f)) d[j] = 0.f;
        st4(dx + off, d);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j >= nj) break;
          float v = d[j];
          if (mask && !(ldf(mask, off + j) > 0.f)) v = 0.f;
          stf(dx, off + j, v);
        }
      }
    }
  }
#pragma unroll
  for (int o = 0; o < OUT; ++o) {
    const size_t off = (size_t)o * in + i0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= nj) break;
      if (gw) gw[off + j] = acc[o][j];
      sgd_update(wv[o][j], vv[o][j], acc[o][j], lr, mu);
    }
    if (wvec) {
      *(float4*)(w + off) = make_float4(wv[o][0], wv[o][1], wv[o][2], wv[o][3]);
      *(float4*)(vel + off) = make_float4(vv[o][0], vv[o][1], vv[o][2], vv[o][3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < nj) {
          w[off + j] = wv[o][j];
          vel[off + j] = vv[o][j];
        }
    }
  }
}

// Narrow inputs (in <= kHeadBwdSmallIn): the one-thread-per-4-columns kernel above has
// a single CTA whose threads walk all B rows serially (latency-bound, ~37 us for the
// FIXED 64 -> 2 head at B = 64). Here a CTA owns 64 columns and its 16 row groups
// split the batch: thread (cq, rg) takes columns 4cq..4cq+3 of rows rg, rg+16, ...;
// dX of those (row, column) pairs is complete in-thread, the dW partials of the 16
// row groups are added in a fixed order in shared memory (deterministic), then the
// momentum update runs as in head_bwd_kernel.
constexpr int kHeadBwdSmallIn = 4096;
template <class TX, class TD, int OUT>
__global__ void __launch_bounds__(256) head_bwd_small_kernel(const TX* __restrict__ x, int x_ld,
                                                             const float* __restrict__ g, int B, int in,
                                                             float* __restrict__ w, float* __restrict__ vel,
                                                             float* __restrict__ gw, TD* __restrict__ dx,
                                                             const TD* __restrict__ mask, float* __restrict__ b,
                                                             float* __restrict__ vb, float* __restrict__ gb, float lr,
                                                             float mu) {
  __shared__ float Gs[kHeadMaxBatch][OUT];
  __shared__ float red[16][OUT][64];
  for (int e = threadIdx.x; e < B * OUT; e += blockDim.x) Gs[e / OUT][e % OUT] = g[e];
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < OUT) {  // bias: sum over the batch in order
    const int o = threadIdx.x;
    float s = 0.f;
    for (int r = 0; r < B; ++r) s += Gs[r][o];
    if (gb) gb[o] = s;
    float bv = b[o], v = vb[o];
    sgd_update(bv, v, s, lr, mu);
    b[o] = bv;
    vb[o] = v;
  }
  const int cq = threadIdx.x & 15, rg = threadIdx.x >> 4;
  const int i0 = blockIdx.x * 64 + cq * 4;
  const int nj = i0 < in ? min(4, in - i0) : 0;
  float wv[OUT][4], acc[OUT][4];
#pragma unroll
  for (int o = 0; o < OUT; ++o)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      wv[o][j] = j < nj ? w[(size_t)o * in + i0 + j] : 0.f;
      acc[o][j] = 0.f;
    }
  for (int r = rg; r < B; r += 16) {
    float xv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) xv[j] = j < nj ? ldf(x, (size_t)r * x_ld + i0 + j) : 0.f;
    float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int o = 0; o < OUT; ++o) {
      const float gr = Gs[r][o];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[o][j] = fmaf(gr, xv[j], acc[o][j]);
        d[j] = fmaf(gr, wv[o][j], d[j]);
      }
    }
    if (dx) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= nj) break;
        const size_t off = (size_t)r * in + i0 + j;
        float v = d[j];
        if (mask && !(ldf(mask, off) > 0.f)) v = 0.f;
        stf(dx, off, v);
      }
    }
  }
#pragma unroll
  for (int o = 0; o < OUT; ++o)
#pragma unroll
    for (int j = 0; j < 4; ++j) red[rg][o][cq * 4 + j] = acc[o][j];
  __syncthreads();
  if (rg != 0 || nj == 0) return;
#pragma unroll
  for (int o = 0; o < OUT; ++o) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= nj) break;
      float s = 0.f;
      for (int q = 0; q < 16; ++q) s += red[q][o][cq * 4 + j];  // row groups in order
      const size_t off = (size_t)o * in + i0 + j;
      if (gw) gw[off] = s;
      float wq = wv[o][j], vq = vel[off];
      sgd_update(wq, vq, s, lr, mu);
      w[off] = wq;
      vel[off] = vq;
    }
  }
}

// column chunks of the forward; rows are split over cdiv(B, kHeadRowsPerCta) CTAs
inline int head_fwd_grid(int in, int num_sms, int B = kHeadRowsPerCta) {
  const int rows = (B + kHeadRowsPerCta - 1) / kHeadRowsPerCta;
  int grid = (in + 255) / 256;  // >= 256 columns per CTA
  const int cap = (2 * num_sms + rows - 1) / rows;
  if (grid > cap) grid = cap;
  const int chunk = ((in + grid - 1) / grid + 7) / 8 * 8;
  if (chunk > kHeadFwdChunk) grid = (in + kHeadFwdChunk - 1) / kHeadFwdChunk;
  return grid < 1 ? 1 : grid;
}

template <class TX>
inline int launch_head_fwd(const TX* x, int x_ld, const float* w, const float* bias, int B, int in, int out,
                           float* partial, unsigned* ticket, float* logits, const int32_t* labels, float* grad,
                           float* losses, int* step_ctr, int* nonfinite, int num_sms, cudaStream_t st) {
  const int gx = head_fwd_grid(in, num_sms, B);
  const dim3 grid(gx, (B + kHeadRowsPerCta - 1) / kHeadRowsPerCta);
  const int chunk = ((in + gx - 1) / gx + 7) / 8 * 8;
  if (chunk > kHeadFwdChunk) return fail(CE_EINVAL, "head forward: chunk %d too large", chunk);
#define CE_HEAD_F(O)                                                                                               \
  if (out == O) {                                                                                                  \
    head_fwd_kernel<TX, O><<<grid, 256, 0, st>>>(x, x_ld, w, bias, B, in, chunk, partial, ticket, logits, labels, \
                                                 grad, losses, step_ctr, nonfinite);                              \
    return CE_OK;                                                                                                  \
  }
  CE_HEAD_F(1) CE_HEAD_F(2) CE_HEAD_F(3) CE_HEAD_F(4)
#undef CE_HEAD_F
  return fail(CE_EINVAL, "head forward: %d outputs", out);
}

template <class TX, class TD>
inline int launch_head_bwd(const TX* x, int x_ld, const float* g, int B, int in, int out, float* w, float* vel,
                           float* gw, TD* dx, const TD* mask, float* b, float* vb, float* gb, float lr, float mu,
                           cudaStream_t st) {
  const int grid = (in + 1023) / 1024;
  const bool small = in <= kHeadBwdSmallIn;
#define CE_HEAD_B(O)                                                                                                \
  if (out == O) {                                                                                                   \
    if (small)                                                                                                      \
      head_bwd_small_kernel<TX, TD, O><<<(in + 63) / 64, 256, 0, st>>>(x, x_ld, g, B, in, w, vel, gw, dx, mask, b, \
                                                                       vb, gb, lr, mu);                             \
    else                                                                                                            \
      head_bwd_kernel<TX, TD, O><<<grid, 256, 0, st>>>(x, x_ld, g, B, in, w, vel, gw, dx, mask, b, vb, gb, lr, mu); \
    return CE_OK;                                                                                                   \
  }
  CE_HEAD_B(1) CE_HEAD_B(2) CE_HEAD_B(3) CE_HEAD_B(4)
#undef CE_HEAD_B
  return fail(CE_EINVAL, "head backward: %d outputs", out);
}

}  // namespace ce
