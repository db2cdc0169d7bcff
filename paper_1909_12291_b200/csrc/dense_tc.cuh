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

// ------------------------------------------------------------------ fp32 check mode on tensor cores
// v -> three bf16 (hi, mid, lo) with v - (hi + mid + lo) below 2^-24 |v|
__device__ __forceinline__ void split3(float v, bf16& hi, bf16& mid, bf16& lo) {
  hi = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(hi);
  mid = __float2bfloat16_rn(r1);
  lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
}
// 4 consecutive fp32 values -> 8 bytes in each of the 3 planes at byte offset `off` of plane 0
__device__ __forceinline__ void store_split4(uint32_t plane0, uint32_t plane_bytes, uint32_t off, float4 v) {
  bf16 h[4], m[4], l[4];
  split3(v.x, h[0], m[0], l[0]);
  split3(v.y, h[1], m[1], l[1]);
  split3(v.z, h[2], m[2], l[2]);
  split3(v.w, h[3], m[3], l[3]);
  const uint2 uh = *(const uint2*)h, um = *(const uint2*)m, ul = *(const uint2*)l;
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(plane0 + off), "r"(uh.x), "r"(uh.y) : "memory");
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(plane0 + plane_bytes + off), "r"(um.x), "r"(um.y) : "memory");
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(plane0 + 2 * plane_bytes + off), "r"(ul.x), "r"(ul.y)
               : "memory");
}
// 4 fp32 from row `row` (row stride ld), columns k..k+3 (< kmax), zero-filled
__device__ __forceinline__ float4 ld4_guard(const float* base, size_t ld, int row, int rows, int k, int kmax) {
  if (row >= rows || k >= kmax) return make_float4(0.f, 0.f, 0.f, 0.f);
  const float* p = base + (size_t)row * ld + k;
  if (k + 3 < kmax && ((ld & 3) == 0)) return *(const float4*)p;
  return make_float4(p[0], k + 1 < kmax ? p[1] : 0.f, k + 2 < kmax ? p[2] : 0.f, k + 3 < kmax ? p[3] : 0.f);
}

// fp32 dense forward part[split][b][o] = sum_k x[b][k] W[o][k] (nn.py:225-231) on the
// tensor cores: A = W rows (outputs, K-major), B = x rows (batch, K-major), both split
// into bf16 planes by the producers (Split3 in tc_engine.cuh).
struct DenseSplitFwdLoader {
  static constexpr int A_MN_MAJOR = 0, B_MN_MAJOR = 0;
  static constexpr bool A_TMA_SW128 = false, B_TMA_SW128 = false, PURE_TMA = false, SYNC_FILL = true, SPLIT3 = true;
  const float* w;  // [out][in]
  const float* x;  // [B][x_ld]
  int in, out, B, x_ld, BN;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int ptid, const uint8_t*,
                       uint64_t*) const {
    const int kq = ptid & 15, k = kb * TC_BK + 4 * kq;
    const uint32_t off_k = kmajor_off(TC_BM, 0, kq >> 1) + (kq & 1) * 8;
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = ld4_guard(w, (size_t)in, c.m0 + (ptid >> 4) + 16 * i, out, k, in);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      store_split4(sA, TC_BM * TC_BK * 2, off_k + (uint32_t)((ptid >> 4) + 16 * i) * 16u, v[i]);
    const uint32_t offb_k = kmajor_off(BN, 0, kq >> 1) + (kq & 1) * 8;
    for (int r = ptid >> 4; r < BN; r += 16)
      store_split4(sB, BN * TC_BK * 2, offb_k + (uint32_t)r * 16u, ld4_guard(x, (size_t)x_ld, c.n0 + r, B, k, in));
  }
};

// fp32 dense dX[b][i] = sum_o g[b][o] W[o][i] (pre-update W, nn.py:240): A = W^T
// (MN-major: rows i contiguous in W's rows), B = g rows (K-major over o).
struct DenseSplitDxLoader {
  static constexpr int A_MN_MAJOR = 1, B_MN_MAJOR = 0;
  static constexpr bool A_TMA_SW128 = false, B_TMA_SW128 = false, PURE_TMA = false, SYNC_FILL = true, SPLIT3 = true;
  const float* w;  // [out][in]
  const float* g;  // [B][out]
  int in, out, B, BN;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int ptid, const uint8_t*,
                       uint64_t*) const {
    // A: 64 output rows (K) x 128 inputs (MN); thread -> row ptid/4, inputs (ptid%4)*32 .. +31
    const int kr = ptid >> 2, o = kb * TC_BK + kr, iq = (ptid & 3) * 32;
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = ld4_guard(w, (size_t)in, o, out, c.m0 + iq + 4 * j, in);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = iq + 4 * j;  // tile-local input index
      store_split4(sA, TC_BM * TC_BK * 2, mnmajor_off(TC_BM, i >> 3, kr) + (i & 4) * 2, v[j]);
    }
    const int kq = ptid & 15, k = kb * TC_BK + 4 * kq;
    const uint32_t offb_k = kmajor_off(BN, 0, kq >> 1) + (kq & 1) * 8;
    for (int r = ptid >> 4; r < BN; r += 16)
      store_split4(sB, BN * TC_BK * 2, offb_k + (uint32_t)r * 16u, ld4_guard(g, (size_t)out, c.n0 + r, B, k, out));
  }
};

// CE_DENSE_SPLIT3=1 sends fp32 check-mode dense layers (>= 1 M parameters, B <= 64:
// two accumulators x BN columns double-buffered must fit TMEM) to the split-plane
// tensor-core GEMMs. Off by default: the producers' synchronous fp32 loads and
// plane splits make it slower than the CUDA-core kernels on the C2 heads measured
// (C2 #15, 262144 -> 523 at B = 32: forward 472 vs 335 us, profiles/r02_notes.md).
constexpr long long kDenseSplitMinParams = 1ll << 20;
inline bool dense_split3_enabled(int B, long long params) {
  static const bool on = [] {
    const char* e = getenv("CE_DENSE_SPLIT3");
    return e && e[0] == '1';
  }();
  return on && B <= 64 && params >= kDenseSplitMinParams;
}

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

// fp32 dense forward on the tensor cores (split planes); returns the partial split count
// tensor-core accumulation is not round-to-nearest: the fp32-check-mode forward keeps
// every split's TMEM chain at <= kSplit3MaxKb K blocks and reduces the splits in IEEE fp32
constexpr int kSplit3MaxKb = 8;
inline int dense_fwd_split3_splits(int out, int in, int num_sms) {
  const int nkb = (in + TC_BK - 1) / TC_BK;
  return std::max(dense_fwd_splits(out, in, num_sms), (nkb + kSplit3MaxKb - 1) / kSplit3MaxKb);
}

inline int dense_fwd_split3(const float* x, int x_ld, const float* w, int in, int out, int B, float* part,
                            int* splits_out, int num_sms, cudaStream_t st) {
  return with_bn(B, [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    TcShape sh = tc_make_shape(out, B, in, BN, dense_fwd_split3_splits(out, in, num_sms));
    *splits_out = sh.splits;
    DenseSplitFwdLoader ld{w, x, in, out, B, x_ld, BN};
    DenseFwdEpi ep{part, out, B};
    cudaError_t e = tc_launch<BN>(ld, ep, sh, num_sms, st);
    return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "dense_fwd_split3: %s", cudaGetErrorString(e));
  });
}

template <class TM>
inline int dense_dx_split3(const float* g, const float* w, int B, int in, int out, const TM* mask, float* dx,
                           int num_sms, cudaStream_t st) {
  return with_bn(B, [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    TcShape sh = tc_make_shape(in, B, out, BN, 1);
    DenseSplitDxLoader ld{w, g, in, out, B, BN};
    DenseDxEpiTc<float, TM> ep{dx, mask, in, B};
    cudaError_t e = tc_launch<BN>(ld, ep, sh, num_sms, st);
    return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "dense_dx_split3: %s", cudaGetErrorString(e));
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
