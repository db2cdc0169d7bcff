// Kernel-level C ABI (include/menndl_sm100.h, "kernel level"): single conv /
// pool passes on caller-owned device tensors and a caller stream. Used by the
// bf16-exact parity tests (T1) and by the conv microbenchmarks; the candidate
// runtime (net.cu) calls the same kernels directly.
#include "ops.cuh"
#include "conv_tc.cuh"

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

int ce_conv_fwd(const ce_conv_desc* d, const void* x, const void* w, const float* bias, int relu, void* y,
                void* stream) {
  if (int s = check_desc(d, true)) return s;
  ConvGeom g = geom(d, true);
  cudaStream_t st = (cudaStream_t)stream;
  const int M = g.n * g.oh * g.ow, K = g.k * g.k * g.c;
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
  conv_sgd_kernel<<<grid_for((size_t)g.co * K), 256, 0, st>>>(part, splits, g.co, K, g.c, g.k, g.s, nullptr, nullptr,
                                                               dw, nullptr, nullptr, 0.f, 0.f);
  launch_bias_sgd(bpart, bsplits, g.co, nullptr, nullptr, db, 0.f, 0.f, st);
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

}  // extern "C"
