// Dense (fully connected) layers on the tcgen05 engine (bf16 mode).
//
// Reference: Dense.forward / Dense.backward (nn.py:225-240) and the momentum
// update (nn.py:306-322). Layouts: fp32 master W [out][in] (+ momentum V),
// bf16 mirror Wb [out][in_pad] (in_pad = round_up(in, 8), zero pad), inputs
// x bf16 [B][x_stride], output-gradient copy gb bf16 [B][out_pad] (zero pad).
//
//   fwd : D[o][b] = sum_i Wb[o][i] x[b][i]      A = Wb (TMA, SW128), B = x (TMA, SW128); split-K
//         epilogue: fp32 partials part[split][b][o] -> dense_reduce_kernel adds the splits + bias
//   dX  : D[i][b] = sum_o Wb[o][i] gb[b][o]     A = Wb^T (MN-major gather), B = gb (K-major)
//         epilogue: x ReLU mask of the input activation; bf16 (features) or fp32 (dense input)
//   dW  : D[i][o] = sum_b x[b][i] gb[b][o]      A = x^T, B = gb^T (both MN-major)
//         epilogue: momentum SGD on W/V (fp32, no FMA contraction) + bf16 mirror, in place;
//         every (o, i) is owned by one thread and dX has already consumed the old Wb.
#pragma once
#include "conv_tc.cuh"

namespace ce {

struct DenseFwdLoader {
  static constexpr int A_MN_MAJOR = 0, B_MN_MAJOR = 0;
  static constexpr bool A_TMA_SW128 = true, B_TMA_SW128 = true, PURE_TMA = true;
  CUtensorMap amap, bmap;
  int BN;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int, const uint8_t*,
                       uint64_t* full) const {
    mbar_expect_tx(full, (uint32_t)(TC_BM + BN) * 128u);
    tma_load_2d(sA, &amap, kb * TC_BK, c.m0, full);
    tma_load_2d(sB, &bmap, kb * TC_BK, c.n0, full);
  }
};

struct DenseFwdEpi {
  float* part;  // [split][B][out]
  int out, B;
  __device__ void store(const TileCoord& c, int row, int col, const float (&v)[16]) const {
    const int o = c.m0 + row;
    if (o >= out) return;
    float* base = part + (size_t)c.split * B * out + o;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int b = c.n0 + col + i;
      if (b < B) base[(size_t)b * out] = v[i];
    }
  }
  __device__ void finish(int, int) const {}
};

template <bool TMA>
struct DenseDxLoader {
  static constexpr int A_MN_MAJOR = 1, B_MN_MAJOR = 0;
  static constexpr bool A_TMA_SW128 = TMA, B_TMA_SW128 = TMA, PURE_TMA = TMA;
  CUtensorMap amap;  // Wb [out rows (K)][in_pad (MN)], 64x64 MN-major boxes
  CUtensorMap bmap;  // gb [B rows][out_pad (K)], K-major boxes
  const bf16* wb;  // [out][in_pad]
  const bf16* gb;  // [B][out_pad]
  int in, in_pad, out, out_pad, B, BN;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int ptid, const uint8_t*,
                       uint64_t* full) const {
    if (TMA) {
      mbar_expect_tx(full, (uint32_t)(TC_BM + BN) * 128u);
      tma_load_2d(sA, &amap, c.m0, kb * TC_BK, full);
      tma_load_2d(sA + 8192, &amap, c.m0 + 64, kb * TC_BK, full);
      tma_load_2d(sB, &bmap, kb * TC_BK, c.n0, full);
      return;
    }
    {  // A: 16 groups of 8 input features x 64 output units
      const int grp = ptid & 15;
      const int i0 = c.m0 + grp * 8;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kr = (ptid >> 4) + 16 * e;
        const int o = kb * TC_BK + kr;
        const bool ok = i0 < in && o < out;
        cp_async16(sA + mnmajor_off(TC_BM, grp, kr), ok ? (const void*)(wb + (size_t)o * in_pad + i0) : (const void*)wb,
                   ok ? 16u : 0u);
      }
    }
    for (int ch = ptid; ch < BN * 8; ch += TC_PRODUCERS) {  // B: batch rows x 8 chunks of output units
      const int r = ch % BN, kc = ch / BN;
      const int o0 = kb * TC_BK + kc * 8;
      const bool ok = r < B && o0 < out_pad;
      cp_async16(sB + kmajor_off(BN, r, kc), ok ? (const void*)(gb + (size_t)r * out_pad + o0) : (const void*)gb,
                 ok ? 16u : 0u);
    }
  }
};

template <class TO, class TM>
struct DenseDxEpiTc {
  TO* dx;        // [B][in]
  const TM* mask;
  int in, B;
  __device__ void store(const TileCoord& c, int row, int col, const float (&v)[16]) const {
    const int i = c.m0 + row;
    const int b0 = c.n0 + col;
    if (i >= in || b0 >= B) return;
    const int n = B - b0 < 16 ? B - b0 : 16;
    float mk[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) mk[u] = (mask && u < n) ? ldf(mask, (size_t)(b0 + u) * in + i) : 1.f;
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (u < n) stf(dx, (size_t)(b0 + u) * in + i, mk[u] > 0.f ? v[u] : 0.f);
  }
  __device__ void finish(int, int) const {}
};

struct DenseDwLoader {
  static constexpr int A_MN_MAJOR = 1, B_MN_MAJOR = 1;
  static constexpr bool A_TMA_SW128 = false, B_TMA_SW128 = false, PURE_TMA = false;
  const bf16* x;   // [B][x_stride]
  const bf16* gb;  // [B][out_pad]
  int in, x_stride, out_pad, B, BN;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int ptid, const uint8_t*,
                       uint64_t*) const {
    {
      const int grp = ptid & 15;
      const int i0 = c.m0 + grp * 8;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kr = (ptid >> 4) + 16 * e;
        const int b = kb * TC_BK + kr;
        const bool ok = i0 < in && b < B;
        cp_async16(sA + mnmajor_off(TC_BM, grp, kr), ok ? (const void*)(x + (size_t)b * x_stride + i0) : (const void*)x,
                   ok ? 16u : 0u);
      }
    }
    const int groups = BN / 8;
    for (int ch = ptid; ch < groups * TC_BK; ch += TC_PRODUCERS) {
      const int grp = ch % groups, kr = ch / groups;
      const int o0 = c.n0 + grp * 8, b = kb * TC_BK + kr;
      const bool ok = o0 < out_pad && b < B;
      cp_async16(sB + mnmajor_off(BN, grp, kr), ok ? (const void*)(gb + (size_t)b * out_pad + o0) : (const void*)gb,
                 ok ? 16u : 0u);
    }
  }
};

struct DenseDwSgdEpi {
  static constexpr int EPI_WARPS = 16;  // memory-bound epilogue: more warps = more loads in flight
  float* w;      // [out][in] fp32 master
  float* vel;
  float* gw;     // optional raw gradient
  bf16* wb;      // [out][in_pad]
  int in, in_pad, out;
  float lr, mu;
  __device__ void store(const TileCoord& c, int row, int col, const float (&v)[16]) const {
    const int o0 = c.n0 + col;
    const int i = c.m0 + row;
    if (i >= in || o0 >= out) return;
    const int n = out - o0 < 16 ? out - o0 : 16;
    if (!w) {  // gradient only (kernel-level ce_dense_bwd without SGD)
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (u < n) gw[(size_t)(o0 + u) * in + i] = v[u];
      return;
    }
    float wv[16], vv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (u < n) {
        const size_t off = (size_t)(o0 + u) * in + i;
        wv[u] = __ldcs(w + off);
        vv[u] = __ldcs(vel + off);
      }
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (u < n) {
        const size_t off = (size_t)(o0 + u) * in + i;
        if (gw) gw[off] = v[u];
        sgd_update(wv[u], vv[u], v[u], lr, mu);
        __stcs(w + off, wv[u]);
        __stcs(vel + off, vv[u]);
        if (wb) wb[(size_t)(o0 + u) * in_pad + i] = __float2bfloat16_rn(wv[u]);
      }
    }
  }

  __device__ void finish(int, int) const {}
};

// ------------------------------------------------------------------ launchers
inline int dense_fwd_splits(int out, int in, int num_sms) {
  const int m_tiles = (out + TC_BM - 1) / TC_BM;
  const int nkb = (in + TC_BK - 1) / TC_BK;
  int s = num_sms / m_tiles;
  if (s > nkb / 2) s = nkb / 2;
  if (s > 148) s = 148;
  return s < 1 ? 1 : s;
}

// returns the number of partial splits written to `part`
inline int dense_fwd_tc(const bf16* x, int x_stride, const bf16* wb, int in, int in_pad, int out, int B, float* part,
                        int* splits_out, int num_sms, cudaStream_t st) {
  return with_bn(B, [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    TcShape sh = tc_make_shape(out, B, in, BN, dense_fwd_splits(out, in, num_sms));
    *splits_out = sh.splits;
    DenseFwdLoader ld{};
    ld.BN = BN;
    if (!make_tmap_kmajor(&ld.amap, wb, out, in, TC_BM, in_pad) || !make_tmap_kmajor(&ld.bmap, x, B, in, BN, x_stride))
      return fail(CE_ECUDA, "dense_fwd_tc: tensor map encoding failed");
    DenseFwdEpi ep{part, out, B};
    cudaError_t e = tc_launch<BN>(ld, ep, sh, num_sms, st);
    return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "dense_fwd_tc: %s", cudaGetErrorString(e));
  });
}

template <class TO, class TM>
inline int dense_dx_tc(const bf16* wb, const bf16* gb, int in, int in_pad, int out, int out_pad, int B, const TM* mask,
                       TO* dx, int num_sms, cudaStream_t st) {
  return with_bn(B, [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    TcShape sh = tc_make_shape(in, B, out_pad, BN, 1);
    DenseDxEpiTc<TO, TM> ep{dx, mask, in, B};
    cudaError_t e;
    DenseDxLoader<true> ldt{};
    if (!tma_disabled() && make_tmap_mn64(&ldt.amap, wb, out, in_pad) &&
        make_tmap_kmajor(&ldt.bmap, gb, B, out_pad, BN, out_pad)) {
      ldt.wb = wb; ldt.gb = gb; ldt.in = in; ldt.in_pad = in_pad; ldt.out = out; ldt.out_pad = out_pad;
      ldt.B = B; ldt.BN = BN;
      e = tc_launch<BN>(ldt, ep, sh, num_sms, st);
    } else {
      DenseDxLoader<false> ld{};
      ld.wb = wb; ld.gb = gb; ld.in = in; ld.in_pad = in_pad; ld.out = out; ld.out_pad = out_pad;
      ld.B = B; ld.BN = BN;
      e = tc_launch<BN>(ld, ep, sh, num_sms, st);
    }
    return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "dense_dx_tc: %s", cudaGetErrorString(e));
  });
}

inline int dense_dw_sgd_tc(const bf16* x, int x_stride, const bf16* gb, int in, int in_pad, int out, int out_pad, int B,
                           float* w, float* vel, float* gw, bf16* wb, float lr, float mu, int num_sms,
                           cudaStream_t st) {
  return with_bn(out < 256 ? out : 256, [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    TcShape sh = tc_make_shape(in, out, B, BN, 1);
    DenseDwLoader ld{x, gb, in, x_stride, out_pad, B, BN};
    DenseDwSgdEpi ep{w, vel, gw, wb, in, in_pad, out, lr, mu};
    cudaError_t e = tc_launch<BN>(ld, ep, sh, num_sms, st);
    return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "dense_dw_tc: %s", cudaGetErrorString(e));
  });
}

}  // namespace ce
