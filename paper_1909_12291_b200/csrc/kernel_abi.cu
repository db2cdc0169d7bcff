// Kernel-level C ABI (include/menndl_sm100.h, "kernel level"): single conv /
// pool passes on caller-owned device tensors and a caller stream. Used by the
// bf16-exact parity tests (T1) and by the conv microbenchmarks; the candidate
// runtime (net.cu) calls the same kernels directly.
#include "ops.cuh"
#include "conv_tc.cuh"
#include "dense_tc.cuh"
#include "dense_simt.cuh"
#include "init.cuh"

using namespace ce;

namespace {

int check_desc(const ce_conv_desc* d, bool conv) {
  if (!d) return fail(CE_EINVAL, "null descriptor");
  if (d->n < 1 || d->c < 1 || d->h < 1 || d->w < 1 || d->kernel < 1 || d->stride < 1)
    return fail(CE_EINVAL, "bad conv/pool descriptor");
  if (d->h < d->kernel || d->w < d->kernel) return fail(CE_EINVAL, "window %d exceeds input %dx%d", d->kernel, d->h, d->w);
  if (d->c % 8) return fail(CE_EINVAL, "stored channels must be a multiple of 8 (got %d)", d->c);
  if (conv && (d->c_out % 8 || d->c_out < 8))
    return fail(CE_EINVAL, "conv channels must be multiples of 8 (got %d -> %d)", d->c, d->c_out);
  if (d->precision != CE_PREC_BF16 && d->precision != CE_PREC_FP32) return fail(CE_EINVAL, "bad precision");
  return CE_OK;
}

ConvGeom geom(const ce_conv_desc* d, bool conv) {
  ConvGeom g;
  g.n = d->n;
  g.c = d->c;
  g.h = d->h;
  g.w = d->w;
  g.k = d->kernel;
  g.s = d->stride;
  g.oh = (d->h - d->kernel) / d->stride + 1;
  g.ow = (d->w - d->kernel) / d->stride + 1;
  g.co = conv ? d->c_out : d->c;
  return g;
}

int sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

__global__ void sgd_momentum_kernel(float* __restrict__ w, float* __restrict__ vel, const float* __restrict__ g,
                                    size_t count, float lr, float mu) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x) {
    float wv = w[e], vv = vel[e];
    sgd_update(wv, vv, g[e], lr, mu);
    w[e] = wv;
    vel[e] = vv;
  }
}

int check_dense(const ce_dense_desc* d) {
  if (!d) return fail(CE_EINVAL, "null descriptor");
  if (d->n < 1 || d->in < 1 || d->out < 1) return fail(CE_EINVAL, "bad dense descriptor (n=%d in=%d out=%d)", d->n, d->in, d->out);
  if (d->precision != CE_PREC_BF16 && d->precision != CE_PREC_FP32) return fail(CE_EINVAL, "bad precision");
  if (d->precision == CE_PREC_BF16 && d->n > 256) return fail(CE_EINVAL, "bf16 dense supports n <= 256 (got %d)", d->n);
  return CE_OK;
}

int pad8(int v) { return (v + 7) / 8 * 8; }

// split-K partial count of the dense forward for this descriptor
int dense_fwd_part_splits(const ce_dense_desc* d) {
  if (d->precision == CE_PREC_BF16) return dense_fwd_splits(d->out, d->in, sms());
  return simt_splits(d->in, pick_splits(simt_tiles(d->n, d->out), d->in, 256, sms(), 8, 256));
}

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

size_t wgrad_ws(const ConvGeom& g, bool tc) {
  const int K = g.k * g.k * g.c, Mo = g.n * g.oh * g.ow;
  int splits = tc ? conv_wgrad_splits(g, g.n, sms()) : simt_splits(Mo, 8);
  return (size_t)splits * g.co * K * 4 + (size_t)(kColsumMaxSplits + 64) * g.co * 4 + 256;
}

}  // namespace

extern "C" {

size_t ce_conv_workspace_bytes(const ce_conv_desc* d) {
  if (check_desc(d, true)) return 0;
  ConvGeom g = geom(d, true);
  const bool tc = d->precision == CE_PREC_BF16 && conv_tc_enabled();
  size_t dg = (size_t)g.co * g.k * g.k * g.c * 2 + 256;
  size_t wg = wgrad_ws(g, tc);
  return dg > wg ? dg : wg;
}

int ce_conv_fwd(const ce_conv_desc* d, const void* x, const void* w, const float* bias, int relu, int pool_k,
                int pool_s, void* y, uint8_t* arg, void* stream) {
  if (int s = check_desc(d, true)) return s;
  ConvGeom g = geom(d, true);
  cudaStream_t st = (cudaStream_t)stream;
  const int M = g.n * g.oh * g.ow, K = g.k * g.k * g.c;
  if (pool_k > 0) {  // max-pool epilogue: y / arg are the pooled map and its argmax
    if (d->precision != CE_PREC_BF16 || !conv_tc_enabled())
      return fail(CE_EINVAL, "the max-pool epilogue runs on the bf16 tensor-core path only");
    if (!arg || !pool_fusable(pool_k, pool_s) || g.oh < pool_k || g.ow < pool_k)
      return fail(CE_EINVAL, "max-pool epilogue: window %d stride %d not fusable (needs 2 or 3, stride >= window)",
                  pool_k, pool_s);
    return conv_fwd_tc_pool(g, (const bf16*)x, (const bf16*)w, bias, relu, pool_k, pool_s, (bf16*)y, arg, sms(), st);
  }
  if (d->precision == CE_PREC_BF16) {
    if (conv_tc_enabled()) return conv_fwd_tc(g, (const bf16*)x, (const bf16*)w, bias, relu, (bf16*)y, sms(), st);
    return fail(CE_EINVAL, "bf16 kernel-level conv requires the tensor-core path");
  }
  simt_gemm(make_fwd_a((const float*)x, g), FwdB{(const float*)w, K}, FwdEpi<float>{(float*)y, bias, g.co, relu != 0},
            M, g.co, K, 1, st);
  CE_CHECK_LAUNCH();
  return CE_OK;
}

int ce_conv_dgrad(const ce_conv_desc* d, const void* dy, const void* w, const void* mask, void* dx, void* workspace,
                  size_t ws_bytes, void* stream) {
  if (int s = check_desc(d, true)) return s;
  ConvGeom g = geom(d, true);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t wn = (size_t)g.co * g.k * g.k * g.c;
  if (d->precision == CE_PREC_BF16) {
    if (!conv_tc_enabled()) return fail(CE_EINVAL, "bf16 kernel-level conv requires the tensor-core path");
    if (!workspace || ws_bytes < wn * 2) return fail(CE_EINVAL, "dgrad workspace too small");
    bf16* wt = (bf16*)workspace;
    // [o][tap][c] bf16 -> [c][tap][o]
    const bf16* wb = (const bf16*)w;
    transpose_w_bf16_kernel<<<grid_for(wn), 256, 0, st>>>(wb, g.co, g.k, g.s, g.c, wt);
    CE_CHECK_LAUNCH();
    return conv_dgrad_tc(g, (const bf16*)dy, wt, (const bf16*)mask, (bf16*)dx, sms(), st);
  }
  simt_gemm(make_dgrad_a((const float*)dy, g), DgradB{(const float*)w, g},
            DgradEpi<float>{(float*)dx, (const float*)mask, g.c}, g.n * g.h * g.w, g.c, g.k * g.k * g.co, 1, st);
  CE_CHECK_LAUNCH();
  return CE_OK;
}

int ce_conv_wgrad(const ce_conv_desc* d, const void* x, const void* dy, float* dw, float* db, void* workspace,
                  size_t ws_bytes, void* stream) {
  if (int s = check_desc(d, true)) return s;
  ConvGeom g = geom(d, true);
  cudaStream_t st = (cudaStream_t)stream;
  const int K = g.k * g.k * g.c, Mo = g.n * g.oh * g.ow;
  const bool tc = d->precision == CE_PREC_BF16;
  if (tc && !conv_tc_enabled()) return fail(CE_EINVAL, "bf16 kernel-level conv requires the tensor-core path");
  if (!workspace || ws_bytes < wgrad_ws(g, tc)) return fail(CE_EINVAL, "wgrad workspace too small");
  float* part = (float*)workspace;
  int splits;
  if (tc) {
    if (int s = conv_wgrad_tc(g, (const bf16*)x, (const bf16*)dy, part, &splits, sms(), st)) return s;
  } else {
    splits = simt_splits(Mo, 8);
    simt_gemm(WgradA<float>{(const float*)dy, g.co}, WgradB<float>{make_fwd_a((const float*)x, g)},
              PartialEpi{part, g.co, K}, g.co, K, Mo, splits, st);
  }
  CE_CHECK_LAUNCH();
  float* bpart = part + (size_t)splits * g.co * K;
  const int bsplits = tc ? colsum((const bf16*)dy, Mo, g.co, bpart, st) : colsum((const float*)dy, Mo, g.co, bpart, st);
  launch_conv_sgd(part, splits, g.co, K, g.c, g.k, g.s, nullptr, nullptr, dw, nullptr, nullptr, bpart, bsplits, nullptr,
                  nullptr, db, 0.f, 0.f, st);
  CE_CHECK_LAUNCH();
  return CE_OK;
}

int ce_maxpool_fwd(const ce_conv_desc* d, const void* x, void* y, uint8_t* arg, void* stream) {
  if (int s = check_desc(d, false)) return s;
  ConvGeom g = geom(d, false);
  size_t total = (size_t)g.n * g.oh * g.ow * g.c;
  cudaStream_t st = (cudaStream_t)stream;
  (void)total;
  int e = d->precision == CE_PREC_BF16 ? launch_maxpool_fwd<bf16>((const bf16*)x, g, (bf16*)y, arg, false, st)
                                       : launch_maxpool_fwd<float>((const float*)x, g, (float*)y, arg, false, st);
  if (e) return e;
  CE_CHECK_LAUNCH();
  return CE_OK;
}

int ce_maxpool_bwd(const ce_conv_desc* d, const void* dy, const uint8_t* arg, const void* mask, void* dx,
                   void* stream) {
  if (int s = check_desc(d, false)) return s;
  ConvGeom g = geom(d, false);
  size_t total = (size_t)g.n * g.h * g.w * g.c;
  cudaStream_t st = (cudaStream_t)stream;
  (void)total;
  int e = d->precision == CE_PREC_BF16
              ? launch_maxpool_bwd<bf16, bf16>((const bf16*)dy, arg, g, (const bf16*)mask, (bf16*)dx, st)
              : launch_maxpool_bwd<float, float>((const float*)dy, arg, g, (const float*)mask, (float*)dx, st);
  if (e) return e;
  CE_CHECK_LAUNCH();
  return CE_OK;
}


int ce_gather_u8_normalize(const uint8_t* pixels, int c, int h, int w, const int32_t* idx, int n, int c_store,
                           int precision, void* out, void* stream) {
  if (!pixels || !idx || !out || n < 1 || c < 1 || h < 1 || w < 1 || c_store < c)
    return fail(CE_EINVAL, "bad gather arguments (n=%d c=%d c_store=%d)", n, c, c_store);
  cudaStream_t st = (cudaStream_t)stream;
  const int HW = h * w;
  dim3 grid = gather_grid(HW, n);
  if (precision == CE_PREC_BF16)
    gather_u8_kernel<bf16><<<grid, 256, 0, st>>>(pixels, nullptr, idx, nullptr, 0, 0, 0, n, c, c_store, HW, (bf16*)out,
                                                 nullptr);
  else if (precision == CE_PREC_FP32)
    gather_u8_kernel<float><<<grid, 256, 0, st>>>(pixels, nullptr, idx, nullptr, 0, 0, 0, n, c, c_store, HW,
                                                  (float*)out, nullptr);
  else
    return fail(CE_EINVAL, "bad precision");
  CE_CHECK_LAUNCH();
  return CE_OK;
}

size_t ce_dense_workspace_bytes(const ce_dense_desc* d) {
  if (check_dense(d)) return 0;
  const size_t fwd = (size_t)dense_fwd_part_splits(d) * d->n * d->out * 4;
  const size_t gbf = d->precision == CE_PREC_BF16 ? align256((size_t)d->n * pad8(d->out) * 2) : 0;
  const size_t bwd = gbf + (size_t)(kColsumMaxSplits + 64) * d->out * 4;
  return (fwd > bwd ? fwd : bwd) + 256;
}

int ce_dense_fwd(const ce_dense_desc* d, const void* x, const float* w, const void* w16, const float* b, float* y,
                 void* workspace, size_t ws_bytes, void* stream) {
  if (int s = check_dense(d)) return s;
  if (!x || !y) return fail(CE_EINVAL, "null dense operand");
  if (!workspace || ws_bytes < ce_dense_workspace_bytes(d)) return fail(CE_EINVAL, "dense workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  float* part = (float*)workspace;
  int splits;
  if (d->precision == CE_PREC_BF16) {
    if (!w16) return fail(CE_EINVAL, "bf16 dense needs the bf16 weight mirror");
    const int in_pad = pad8(d->in);
    if (int s = dense_fwd_tc((const bf16*)x, in_pad, (const bf16*)w16, d->in, in_pad, d->out, d->n, part, &splits,
                             sms(), st))
      return s;
  } else {
    if (!w) return fail(CE_EINVAL, "null dense weights");
    splits = dense_fwd_part_splits(d);
    simt_gemm(DenseXA<float>{(const float*)x, d->in}, DenseWB{w, d->in}, PartialEpi{part, d->n, d->out}, d->n, d->out,
              d->in, splits, st);
  }
  CE_CHECK_LAUNCH();
  launch_dense_reduce(part, splits, d->n, d->out, b, y, st);
  CE_CHECK_LAUNCH();
  return CE_OK;
}

int ce_dense_bwd(const ce_dense_desc* d, const void* x, const float* dy, float* w, void* w16, float* b, void* dx,
                 const void* mask, float* dw, float* db, const ce_sgd_args* sgd, void* workspace, size_t ws_bytes,
                 void* stream) {
  if (int s = check_dense(d)) return s;
  if (!x || !dy) return fail(CE_EINVAL, "null dense operand");
  if (!workspace || ws_bytes < ce_dense_workspace_bytes(d)) return fail(CE_EINVAL, "dense workspace too small");
  if (sgd) {
    if (!(sgd->lr > 0.f)) return fail(CE_EINVAL, "lr must be positive, got %g", (double)sgd->lr);
    if (!(sgd->momentum >= 0.f && sgd->momentum < 1.f))
      return fail(CE_EINVAL, "momentum must lie in [0, 1), got %g", (double)sgd->momentum);
    if (!w || !b || !sgd->vel_w || !sgd->vel_b) return fail(CE_EINVAL, "fused SGD needs w, b and both velocities");
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int n = d->n, in = d->in, out = d->out;
  const float lr = sgd ? sgd->lr : 0.f, mu = sgd ? sgd->momentum : 0.f;
  float* bpart;
  if (d->precision == CE_PREC_BF16) {
    if (!w16) return fail(CE_EINVAL, "bf16 dense needs the bf16 weight mirror");
    const int in_pad = pad8(in), out_pad = pad8(out);
    bf16* gbf = (bf16*)workspace;
    bpart = (float*)((char*)workspace + align256((size_t)n * out_pad * 2));
    f32_to_bf16_pad_kernel<<<grid_for((size_t)n * out_pad), 256, 0, st>>>(dy, n, out, out_pad, gbf);
    CE_CHECK_LAUNCH();
    if (dx) {
      if (int s = dense_dx_tc((const bf16*)w16, gbf, in, in_pad, out, out_pad, n, (const bf16*)mask, (bf16*)dx, sms(),
                              st))
        return s;
    }
    if ((sgd || dw) && dense_dw_simt_enabled(n)) {
      dense_dw_sgd_simt((const bf16*)x, in_pad, dy, n, in, out, sgd ? w : nullptr, sgd ? sgd->vel_w : nullptr, dw,
                        sgd ? (bf16*)w16 : nullptr, in_pad, lr, mu, st);
    } else if (sgd || dw) {
      if (int s = dense_dw_sgd_tc((const bf16*)x, in_pad, gbf, in, in_pad, out, out_pad, n, sgd ? w : nullptr,
                                  sgd ? sgd->vel_w : nullptr, dw, sgd ? (bf16*)w16 : nullptr, lr, mu, sms(), st))
        return s;
    }
  } else {
    if (!w && dx) return fail(CE_EINVAL, "null dense weights");
    bpart = (float*)workspace;
    const bool small = n <= kDenseSimtMaxBatch;
    if (dx && small)
      dense_dx_simt(dy, w, n, in, out, (const float*)mask, (float*)dx, st);
    else if (dx)
      simt_gemm(DenseGA{dy, out}, DenseWN{w, in}, DenseDxEpi<float, float>{(float*)dx, (const float*)mask, in}, n, in,
                out, 1, st);
    if ((sgd || dw) && small) {
      dense_dw_sgd_simt((const float*)x, in, dy, n, in, out, sgd ? w : nullptr, sgd ? sgd->vel_w : nullptr, dw,
                        (bf16*)nullptr, 0, lr, mu, st);
    } else if (sgd || dw) {
      DenseSgdEpi se{sgd ? w : nullptr, sgd ? sgd->vel_w : nullptr, dw, nullptr, in, lr, mu};
      simt_gemm(DenseGT{dy, out}, DenseXN<float>{(const float*)x, in}, se, out, in, n, 1, st);
    }
  }
  CE_CHECK_LAUNCH();
  if (sgd || db) {
    const int bs = colsum(dy, n, out, bpart, st);
    launch_bias_sgd(bpart, bs, out, sgd ? b : nullptr, sgd ? sgd->vel_b : nullptr, db, lr, mu, st);
    CE_CHECK_LAUNCH();
  }
  return CE_OK;
}

int ce_softmax_xent(const float* logits, const int64_t* labels, int n, int k, float* loss, float* grad,
                    void* stream) {
  if (!logits || !labels || !loss || !grad) return fail(CE_EINVAL, "null xent operand");
  if (n < 1 || n > 1024 || k < 1) return fail(CE_EINVAL, "xent supports 1 <= n <= 1024 rows (got n=%d k=%d)", n, k);
  xent_kernel<int64_t><<<1, 1024, 0, (cudaStream_t)stream>>>(logits, labels, n, k, grad, loss, nullptr, nullptr);
  CE_CHECK_LAUNCH();
  return CE_OK;
}

int ce_sgd_momentum(float* w, float* vel, const float* g, size_t count, float lr, float momentum, void* stream) {
  if (!(lr > 0.f)) return fail(CE_EINVAL, "lr must be positive, got %g", (double)lr);
  if (!(momentum >= 0.f && momentum < 1.f)) return fail(CE_EINVAL, "momentum must lie in [0, 1), got %g", (double)momentum);
  if (count == 0) return CE_OK;
  if (!w || !vel || !g) return fail(CE_EINVAL, "null sgd operand");
  sgd_momentum_kernel<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>(w, vel, g, count, lr, momentum);
  CE_CHECK_LAUNCH();
  return CE_OK;
}

}  // extern "C"

// ReLU of the operator API (nn.py:170-183): y = x > 0 ? x : 0 and the u8 mask (x > 0);
// backward dx = dy * mask. T = bf16 or float; 8 elements per thread when aligned.
template <class T>
__global__ void __launch_bounds__(256) relu_fwd_kernel(const T* __restrict__ x, size_t count, T* __restrict__ y,
                                                       uint8_t* __restrict__ mask) {
  const size_t n8 = count / 8;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n8; e += (size_t)gridDim.x * blockDim.x) {
    float v[8];
    load8(x + e * 8, v);
    uint8_t m[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      m[u] = v[u] > 0.f;
      v[u] = m[u] ? v[u] : 0.f;
    }
    store8(y + e * 8, v);
    if (mask) *(uint2*)(mask + e * 8) = *(const uint2*)m;
  }
  for (size_t e = n8 * 8 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count;
       e += (size_t)gridDim.x * blockDim.x) {
    const float v = ldf(x, e);
    const bool pos = v > 0.f;
    stf(y, e, pos ? v : 0.f);
    if (mask) mask[e] = pos;
  }
}

template <class T>
__global__ void __launch_bounds__(256) relu_bwd_kernel(const T* __restrict__ dy, const uint8_t* __restrict__ mask,
                                                       size_t count, T* __restrict__ dx) {
  const size_t n8 = count / 8;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n8; e += (size_t)gridDim.x * blockDim.x) {
    float v[8];
    load8(dy + e * 8, v);
    const uint2 m2 = *(const uint2*)(mask + e * 8);
    const uint8_t* m = (const uint8_t*)&m2;
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = m[u] ? v[u] : 0.f;
    store8(dx + e * 8, v);
  }
  for (size_t e = n8 * 8 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count;
       e += (size_t)gridDim.x * blockDim.x)
    stf(dx, e, mask[e] ? ldf(dy, e) : 0.f);
}

extern "C" {

int ce_relu_fwd(const void* x, size_t count, int precision, void* y, uint8_t* mask, void* stream) {
  if (count == 0) return CE_OK;
  if (!x || !y) return fail(CE_EINVAL, "null relu operand");
  if (((uintptr_t)x | (uintptr_t)y | (uintptr_t)mask) & 15) return fail(CE_EINVAL, "relu operands must be 16-byte aligned");
  const size_t g = grid_for((count + 7) / 8);
  if (precision == CE_PREC_BF16)
    relu_fwd_kernel<bf16><<<g, 256, 0, (cudaStream_t)stream>>>((const bf16*)x, count, (bf16*)y, mask);
  else if (precision == CE_PREC_FP32)
    relu_fwd_kernel<float><<<g, 256, 0, (cudaStream_t)stream>>>((const float*)x, count, (float*)y, mask);
  else
    return fail(CE_EINVAL, "bad precision %d", precision);
  CE_CHECK_LAUNCH();
  return CE_OK;
}

int ce_relu_bwd(const void* dy, const uint8_t* mask, size_t count, int precision, void* dx, void* stream) {
  if (count == 0) return CE_OK;
  if (!dy || !mask || !dx) return fail(CE_EINVAL, "null relu operand");
  if (((uintptr_t)dy | (uintptr_t)dx | (uintptr_t)mask) & 15) return fail(CE_EINVAL, "relu operands must be 16-byte aligned");
  const size_t g = grid_for((count + 7) / 8);
  if (precision == CE_PREC_BF16)
    relu_bwd_kernel<bf16><<<g, 256, 0, (cudaStream_t)stream>>>((const bf16*)dy, mask, count, (bf16*)dx);
  else if (precision == CE_PREC_FP32)
    relu_bwd_kernel<float><<<g, 256, 0, (cudaStream_t)stream>>>((const float*)dy, mask, count, (float*)dx);
  else
    return fail(CE_EINVAL, "bad precision %d", precision);
  CE_CHECK_LAUNCH();
  return CE_OK;
}

int ce_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, uint64_t skip,
                     double low, double high, float* out, size_t count, void* stream) {
  if (count == 0) return CE_OK;
  if (!out) return fail(CE_EINVAL, "null output");
  InitLayout L{};
  L.kind = 0;
  const size_t nchunks = (count + kInitChunk - 1) / kInitChunk;
  kaiming_uniform_kernel<<<grid_for(nchunks, 128), 128, 0, (cudaStream_t)stream>>>(
      state_hi, state_lo, inc_hi, inc_lo, (unsigned long long)skip, count, low, high - low, L, out);
  CE_CHECK_LAUNCH();
  return CE_OK;
}

int ce_permute_flatten_weights(const float* src, size_t rows, int c, int c_store, int hw, int direction, float* dst,
                               void* stream) {
  if (!src || !dst || c < 1 || c_store < c || hw < 1) return fail(CE_EINVAL, "bad permute arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (direction == 0)
    dense_w_to_dev_kernel<<<grid_for(rows * hw * c_store), 256, 0, st>>>(src, rows, c, c_store, hw, dst);
  else if (direction == 1)
    dense_w_to_host_kernel<<<grid_for(rows * hw * c), 256, 0, st>>>(src, rows, c, c_store, hw, dst);
  else
    return fail(CE_EINVAL, "direction must be 0 or 1");
  CE_CHECK_LAUNCH();
  return CE_OK;
}

}  // extern "C"

#ifdef CE_TC_TRACE
extern "C" int ce_debug_fake_load(int on) {
  return cudaMemcpyToSymbol(ce::g_tc_fake_load, &on, sizeof(int)) == cudaSuccess ? CE_OK : CE_ECUDA;
}
// debug builds only (tools/tc_trace.py): copy and reset the tc_engine event trace
extern "C" int ce_debug_trace(unsigned long long* out, unsigned int* counts) {
  if (cudaMemcpyFromSymbol(out, ce::g_tc_trace, sizeof(ce::g_tc_trace)) != cudaSuccess) return CE_ECUDA;
  if (cudaMemcpyFromSymbol(counts, ce::g_tc_trace_n, sizeof(ce::g_tc_trace_n)) != cudaSuccess) return CE_ECUDA;
  static const unsigned int zero[4][3] = {};
  return cudaMemcpyToSymbol(ce::g_tc_trace_n, zero, sizeof(zero)) == cudaSuccess ? CE_OK : CE_ECUDA;
}
#endif
