// Packed first conv layer (tcgen05).
//
// The image layer stores 3 real channels padded to 8 (one 16-byte chunk per
// pixel), so its implicit GEMMs run K = k*k*8 where only k*k*3 columns carry
// data (k = 6: 288 vs 108). A conv whose input is channel-padded and that needs
// no dX (the first parameterised layer) instead runs two plain GEMMs over a
// packed im2col matrix with kPackedCpt = 4 columns per tap (the 3 real
// channels and one zero, so a 16-byte chunk is exactly two taps):
//     xcol[m][kk],  kk = (i*k + j)*4 + c  for kk < Kr = 4*k*k (c >= c_real: 0),
//                   xcol[m][Kr] = 1, zero up to Kp = pad8(Kr + 1),
// written once per forward (conv.forward, nn.py:82-94):
//   forward  y = xcol . Wp^T      M = pixels, N = C_out, K = Kp  (pure 2D TMA)
//   wgrad    D = xcol^T . dY      M = Kp, N = C_out, K = pixels  (2D TMA, split-K)
// Row Kr of D is sum_pixels dY = the bias gradient (nn.py:115), so the
// separate column-sum pass over dY disappears. Wp[o][kk] is the packed bf16
// mirror of the fp32 master W[o][i][j][c_pad] (column Kr held at zero: the
// bias is added in fp32 by the epilogue).
#pragma once
#include "conv_tc.cuh"
#include "dense_tc.cuh"

namespace ce {

// CE_DISABLE_PACKED=1 runs the first layer through the padded implicit GEMMs (comparison)
inline bool packed_disabled() {
  static const bool off = [] {
    const char* e = getenv("CE_DISABLE_PACKED");
    return e && e[0] == '1';
  }();
  return off;
}

constexpr int kPackedCpt = 4;  // packed columns per tap (c_real <= 4 <= stored channels)
inline int packed_kr(const ConvGeom& g, int c_real) { return g.k * g.k * kPackedCpt; }
inline int packed_kp(const ConvGeom& g, int c_real) { return (packed_kr(g, c_real) + 1 + 7) / 8 * 8; }
inline bool packable(const ConvGeom& g, int c_real) { return c_real <= kPackedCpt && g.c >= kPackedCpt; }

// one thread per (pixel, 8-column chunk): 8 gathered bf16 -> one 16-byte store.
// Column kk reads x at (receptive-field origin) + off[kk]; off is built once per
// block in shared memory (-1: the ones column, -2: zero padding); index math
// is 32-bit with magic-number division.
// POOL: rows in the window-major order of `pm` (conv_tc.cuh PoolMap); padding
// rows are all zero, the ones column included, so they add nothing to the
// packed wgrad (bias row) either.
constexpr int kPackedMaxKp = 1024;
template <class T, bool POOL = false>
__global__ void __launch_bounds__(256) im2col_packed_kernel(const T* __restrict__ x, ConvGeom g, int c_real,
                                                            int Kp, FastDiv d_chunks, FastDiv d_ow, FastDiv d_oh,
                                                            T* __restrict__ xcol, PoolMap pm, uint32_t rows) {
  __shared__ int off[kPackedMaxKp];
  const int Kr = g.k * g.k * kPackedCpt;
  for (int kk = threadIdx.x; kk < Kp; kk += blockDim.x) {
    if (kk < Kr) {
      const int tap = kk / kPackedCpt, c = kk - tap * kPackedCpt;
      const int i = tap / g.k, j = tap - i * g.k;
      off[kk] = c < c_real ? (i * g.w + j) * g.c + c : -2;
    } else {
      off[kk] = kk == Kr ? -1 : -2;
    }
  }
  __syncthreads();
  const uint32_t total = rows * (uint32_t)(Kp / 8);
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    uint32_t m, ch, t, q, p, n;
    d_chunks.divmod(e, m, ch);
    bool ok = true;
    if constexpr (POOL) {
      ok = pm.pixel((int)(m / TC_BM), (int)(m % TC_BM), n, p, q);
    } else {
      d_ow.divmod(m, t, q);
      d_oh.divmod(t, n, p);
    }
    float v[8];
    if (ok) {
      const T* base = x + (((size_t)n * g.h + p * g.s) * g.w + q * g.s) * g.c;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int o = off[ch * 8 + u];
        v[u] = o >= 0 ? ldf(base, (size_t)o) : (o == -1 ? 1.f : 0.f);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = 0.f;
    }
    store8(xcol + (size_t)m * Kp + ch * 8, v);  // bf16 values round-trip exactly
  }
}

// Wp[o][kk] = bf16(W[o][i][j][c]) for kk < Kr, 0 beyond (incl. the ones column)
template <class TW>
__global__ void pack_first_w_kernel(const float* __restrict__ w, int co, int k, int cp, int c_real, int Kp,
                                    TW* __restrict__ wp) {
  const int Kr = k * k * kPackedCpt;
  const size_t total = (size_t)co * Kp;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int o = (int)(e / Kp), kk = (int)(e % Kp);
    float v = 0.f;
    if (kk < Kr) {
      const int tap = kk / kPackedCpt, c = kk - tap * kPackedCpt;
      if (c < c_real) v = w[((size_t)o * k * k + tap) * cp + c];
    }
    stf(wp, e, v);
  }
}

inline int conv_fwd_packed(const ConvGeom& g, const bf16* xcol, int Kp, const bf16* wp, const float* bias, int relu,
                           bf16* y, int num_sms, cudaStream_t st) {
  const int M = g.n * g.oh * g.ow;
  return with_bn(pick_bn((M + TC_BM - 1) / TC_BM, g.co, num_sms), [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    TcShape sh = tc_make_shape(M, g.co, Kp, BN, 1);
    DenseFwdLoader ld{};
    ld.BN = BN;
    if (!make_tmap_kmajor(&ld.amap, xcol, M, Kp, TC_BM) || !make_tmap_kmajor(&ld.bmap, wp, g.co, Kp, BN))
      return fail(CE_ECUDA, "conv_fwd_packed: tensor map encoding failed");
    FwdTcEpi ep{y, bias, M, g.co, relu};
    cudaError_t e = tc_launch<BN>(ld, ep, sh, num_sms, st);
    return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_fwd_packed: %s", cudaGetErrorString(e));
  });
}

// Packed first conv + non-overlapping max-pool: xcol rows in PoolMap order
// (launch_im2col_packed with the map), pooled epilogue.
inline int conv_fwd_packed_pool(const ConvGeom& g, const bf16* xcol, int Kp, const bf16* wp, const float* bias,
                                int relu, const PoolMap& pm, bf16* y, uint8_t* arg, int num_sms, cudaStream_t st) {
  const int Mp = pool_rows(pm);
  return with_bn(pick_bn(Mp / TC_BM, g.co, num_sms), [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    return with_pool_kk(pm.ps, [&](auto kkc) {
      constexpr int KK = decltype(kkc)::value;
      TcShape sh = tc_make_shape(Mp, g.co, Kp, BN, 1);
      DenseFwdLoader ld{};
      ld.BN = BN;
      if (!make_tmap_kmajor(&ld.amap, xcol, Mp, Kp, TC_BM) || !make_tmap_kmajor(&ld.bmap, wp, g.co, Kp, BN))
        return fail(CE_ECUDA, "conv_fwd_packed_pool: tensor map encoding failed");
      FwdPoolEpi<KK> ep{y, arg, bias, g.co, relu, pm};
      cudaError_t e = tc_launch<BN>(ld, ep, sh, num_sms, st);
      return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_fwd_packed_pool: %s", cudaGetErrorString(e));
    });
  });
}

// Backward of the fused pool for the packed layer, in the same window-major row
// order as its xcol: dY[m][o] = dy_pooled[window][o] at the argmax tap, 0 at
// the other taps, at dead windows and on padding rows (nn.py:156-167; stride
// >= window, so every conv output has at most one window).
template <class T>
__global__ void __launch_bounds__(256) pool_expand_rows_kernel(const T* __restrict__ dyp, const uint8_t* __restrict__ arg,
                                                               PoolMap pm, int co, uint32_t rows, T* __restrict__ dy) {
  const int cg = co / 8;
  const uint32_t total = rows * (uint32_t)cg;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const uint32_t m = e / cg;
    const int c0 = (int)(e - m * cg) * 8;
    const int r = (int)(m % TC_BM), lane = r & 31;
    const int wl = lane / pm.KK, tap = lane - wl * pm.KK;
    const int window = (int)(m / TC_BM) * pm.WPT + (r >> 5) * pm.WPW + wl;
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (wl < pm.WPW && window < pm.windows) {
      const size_t o = (size_t)window * co + c0;
      float g[8];
      load8(dyp + o, g);
      const uint2 a2 = *(const uint2*)(arg + o);
      const uint8_t* a = (const uint8_t*)&a2;
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = a[u] == tap ? g[u] : 0.f;
    }
    store8(dy + (size_t)m * co + c0, v);
  }
}

template <class T>
inline void launch_pool_expand_rows(const T* dyp, const uint8_t* arg, const PoolMap& pm, int co, T* dy,
                                    cudaStream_t st) {
  const uint32_t rows = (uint32_t)pool_rows(pm);
  pool_expand_rows_kernel<T><<<grid_for((size_t)rows * (co / 8)), 256, 0, st>>>(dyp, arg, pm, co, rows, dy);
}

inline int conv_wgrad_packed_splits(int Kp, int Mo, int num_sms) {
  const int m_tiles = (Kp + TC_BM - 1) / TC_BM;
  const long long nkb = ((long long)Mo + TC_BK - 1) / TC_BK;
  long long want = num_sms / m_tiles;
  if (want > nkb / 4) want = nkb / 4;
  if (want > 128) want = 128;
  return want < 1 ? 1 : (int)want;
}

// ------------------------------------------------------------------ implicit packed operand
// The packed im2col row of an output pixel (kk = tap*4 + c, ones column at Kr,
// zero to Kp) is built by the producer warps straight from the channel-padded
// input into the stage's shared-memory tile: no im2col matrix in HBM (it would
// cost Kp*2 bytes per pixel twice, k^2-fold the input). With 4 columns per tap
// a 16-byte chunk is two taps = two 8-byte loads of (c0, c1, c2, 0) from the
// 8-channel input pixels.
//   fwd   (MN = false): A = xrow, K-major [128 pixels][64 kk] per k-block; B = Wp
//         by 2D TMA. Epilogue as conv_fwd_packed (bias/ReLU, or the pooled one).
//   wgrad (MN = true) : A = xrow^T, MN-major [128 kk][64 pixels]; B = dY [pixels][co]
//         by 64x64 TMA boxes (BN >= 64) or plain loads. Row Kr of D = sum dY = db.
// POOL: pixels in the window-major PoolMap order (padding rows all zero, the ones
// column included, so they add nothing to D).
template <bool MN, bool POOL, bool TMA_B>
struct PackedTcLoader {
  static constexpr int A_MN_MAJOR = MN, B_MN_MAJOR = MN;
  static constexpr bool A_TMA_SW128 = false, B_TMA_SW128 = TMA_B, PURE_TMA = false, SYNC_FILL = true;
  CUtensorMap bmap;  // fwd: Wp [co][Kp]; wgrad: dY [rows][co] (TMA_B)
  const bf16* x;     // channel-padded input [n][h][w][g.c], g.c >= 4, channels >= c_real zero
  const bf16* dy;    // wgrad without TMA_B
  ConvGeom g;
  int c_real, Kr, Kp, rows, BN;
  FastDiv d_ow, d_oh;
  PoolMap pm;
  __device__ void init(uint8_t* table, int tid, int nthreads) const {
    int* off = (int*)table;  // input offset of each tap relative to the receptive-field origin
    for (int t = tid; t < g.k * g.k; t += nthreads) {
      const int i = t / g.k, j = t - i * g.k;
      off[t] = (i * g.w + j) * g.c;
    }
  }
  // input offset of the receptive-field origin of GEMM row m, or -1 for a padding row
  __device__ __forceinline__ long long origin(int m) const {
    uint32_t n, p, q, t;
    if constexpr (POOL) {
      if (!pm.pixel(m / TC_BM, m % TC_BM, n, p, q)) return -1;
    } else {
      if (m >= rows) return -1;
      d_ow.divmod((uint32_t)m, t, q);
      d_oh.divmod(t, n, p);
    }
    return (((long long)n * g.h + p * g.s) * g.w + q * g.s) * g.c;
  }
  // xrow[kk0 .. kk0+7] of the row at `base` (kk0 % 8 == 0), as 8 packed bf16
  __device__ __forceinline__ uint4 chunk(long long base, int kk0, const int* off) const {
    if (base < 0 || kk0 > Kr) return make_uint4(0u, 0u, 0u, 0u);
    const uint32_t one = 0x3F80u;  // bf16(1.0) in the low half
    if (kk0 == Kr) return make_uint4(one, 0u, 0u, 0u);
    const int t0 = kk0 / kPackedCpt;  // < k*k here
    const uint2 a = *(const uint2*)(x + base + off[t0]);
    if (kk0 + 8 <= Kr) {
      const uint2 b = *(const uint2*)(x + base + off[t0 + 1]);
      return make_uint4(a.x, a.y, b.x, b.y);
    }
    return make_uint4(a.x, a.y, one, 0u);  // Kr % 8 == 4: last tap, then the ones column
  }
  // forward (!MN): the register-pipelined fill (tc_engine SyncPipe); wgrad keeps load()
  static constexpr bool PIPE = !MN;
  struct Regs {
    uint4 v[4];
  };
  __device__ void fetch(const TileCoord& c, int kb, int ptid, const uint8_t* table, Regs& rg) const {
    const int* off = (const int*)table;
    const int kcs = min(8, ((Kp - kb * TC_BK + 15) / 16) * 2);
    const int r = ptid & (TC_BM - 1), kc0 = ptid >> 7;
    const long long base = origin(c.m0 + r);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int kc = kc0 + 2 * e;
      rg.v[e] = kc < kcs ? chunk(base, kb * TC_BK + kc * 8, off) : make_uint4(0u, 0u, 0u, 0u);
    }
  }
  __device__ void put(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int ptid, const Regs& rg,
                      uint64_t* full) const {
    if (ptid == 0) {
      mbar_expect_tx(full, (uint32_t)BN * 128u);
      tma_load_2d(sB, &bmap, kb * TC_BK, c.n0, full);
    }
    const int kcs = min(8, ((Kp - kb * TC_BK + 15) / 16) * 2);
    const int r = ptid & (TC_BM - 1), kc0 = ptid >> 7;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int kc = kc0 + 2 * e;
      if (kc < kcs) st_shared_v4(sA + kmajor_off(TC_BM, r, kc), rg.v[e]);
    }
  }
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int ptid, const uint8_t* table,
                       uint64_t* full) const {
    const int* off = (const int*)table;
    if constexpr (!MN) {
      if (ptid == 0) {
        mbar_expect_tx(full, (uint32_t)BN * 128u);
        tma_load_2d(sB, &bmap, kb * TC_BK, c.n0, full);
      }
      // only the K16 steps the MMA issues are filled (Kp < 64: a single, partial K block)
      const int kcs = min(8, ((Kp - kb * TC_BK + 15) / 16) * 2);
      const int r = ptid & (TC_BM - 1), kc0 = ptid >> 7;
      const long long base = origin(c.m0 + r);
      uint4 vals[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kc = kc0 + 2 * e;
        vals[e] = kc < kcs ? chunk(base, kb * TC_BK + kc * 8, off) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kc = kc0 + 2 * e;
        if (kc < kcs) st_shared_v4(sA + kmajor_off(TC_BM, r, kc), vals[e]);
      }
    } else {
      // A: 16 groups of 8 kk rows x 64 pixels; thread -> one pixel, 4 kk groups (origin computed once)
      const int kr = ptid & (TC_BK - 1);
      const long long base = origin(kb * TC_BK + kr);
      uint4 vals[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) vals[e] = chunk(base, c.m0 + ((ptid >> 6) + 4 * e) * 8, off);
#pragma unroll
      for (int e = 0; e < 4; ++e) st_shared_v4(sA + mnmajor_off(TC_BM, (ptid >> 6) + 4 * e, kr), vals[e]);
      if constexpr (TMA_B) {
        if (ptid == 0) {
          mbar_expect_tx(full, (uint32_t)BN * TC_BK * 2u);
          for (int j = 0; j < BN / 64; ++j) tma_load_2d(sB + j * 8192, &bmap, c.n0 + 64 * j, kb * TC_BK, full);
        }
      } else {
        const int groups = BN / 8;
        for (int ch = ptid; ch < groups * TC_BK; ch += TC_PRODUCERS) {
          const int gq = ch % groups, kq = ch / groups;
          const int o0 = c.n0 + gq * 8, m = kb * TC_BK + kq;
          uint4 v = make_uint4(0u, 0u, 0u, 0u);
          if (o0 < g.co && m < rows) v = *(const uint4*)(dy + (size_t)m * g.co + o0);
          st_shared_v4(sB + mnmajor_off(BN, gq, kq), v);
        }
      }
    }
  }
};

// Packed first-layer forward without the HBM im2col (PackedTcLoader); pm: pooled epilogue
inline int conv_fwd_packed_implicit(const ConvGeom& g, const bf16* x, int c_real, int Kp, const bf16* wp,
                                    const float* bias, int relu, const PoolMap* pm, bf16* y, uint8_t* arg,
                                    int num_sms, cudaStream_t st) {
  const int M = pm ? pool_rows(*pm) : g.n * g.oh * g.ow;
  return with_bn(pick_bn((M + TC_BM - 1) / TC_BM, g.co, num_sms), [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    TcShape sh = tc_make_shape(M, g.co, Kp, BN, 1);
    auto fill = [&](auto& ld) {
      ld.x = x; ld.g = g; ld.c_real = c_real; ld.Kr = packed_kr(g, c_real); ld.Kp = Kp; ld.rows = M; ld.BN = BN;
      ld.d_ow = FastDiv(g.ow); ld.d_oh = FastDiv(g.oh);
      if (pm) ld.pm = *pm;
      return make_tmap_kmajor(&ld.bmap, wp, g.co, Kp, BN);
    };
    cudaError_t e;
    if (pm) {
      PackedTcLoader<false, true, true> ld{};
      if (!fill(ld)) return fail(CE_ECUDA, "conv_fwd_packed_implicit: tensor map encoding failed");
      e = (cudaError_t)with_pool_kk(pm->ps, [&](auto kkc) {
        constexpr int KK = decltype(kkc)::value;
        return (int)tc_launch<BN>(ld, FwdPoolEpi<KK>{y, arg, bias, g.co, relu, *pm}, sh, num_sms, st);
      });
    } else {
      PackedTcLoader<false, false, true> ld{};
      if (!fill(ld)) return fail(CE_ECUDA, "conv_fwd_packed_implicit: tensor map encoding failed");
      e = tc_launch<BN>(ld, FwdTcEpi{y, bias, M, g.co, relu}, sh, num_sms, st);
    }
    return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_fwd_packed_implicit: %s", cudaGetErrorString(e));
  });
}

// Packed first-layer weight gradient without the HBM im2col: part[split][co][Kp]
inline int conv_wgrad_packed_implicit(const ConvGeom& g, const bf16* x, int c_real, int Kp, const bf16* dy,
                                      const PoolMap* pm, float* part, int* splits_out, int num_sms, cudaStream_t st) {
  const int Mo = pm ? pool_rows(*pm) : g.n * g.oh * g.ow;
  return with_bn(g.co, [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    TcShape sh = tc_make_shape(Kp, g.co, Mo, BN, conv_wgrad_packed_splits(Kp, Mo, num_sms));
    *splits_out = sh.splits;
    WgradTcEpi ep{part, Kp, g.co};
    auto run = [&](auto& ld) {
      ld.x = x; ld.dy = dy; ld.g = g; ld.c_real = c_real; ld.Kr = packed_kr(g, c_real); ld.Kp = Kp; ld.rows = Mo;
      ld.BN = BN; ld.d_ow = FastDiv(g.ow); ld.d_oh = FastDiv(g.oh);
      if (pm) ld.pm = *pm;
      return tc_launch<BN>(ld, ep, sh, num_sms, st);
    };
    cudaError_t e;
    if constexpr (BN >= 64) {
      if (pm) {
        PackedTcLoader<true, true, true> ld{};
        if (!make_tmap_mn64(&ld.bmap, dy, Mo, g.co)) return fail(CE_ECUDA, "conv_wgrad_packed_implicit: tmap");
        e = run(ld);
      } else {
        PackedTcLoader<true, false, true> ld{};
        if (!make_tmap_mn64(&ld.bmap, dy, Mo, g.co)) return fail(CE_ECUDA, "conv_wgrad_packed_implicit: tmap");
        e = run(ld);
      }
    } else {
      if (pm) {
        PackedTcLoader<true, true, false> ld{};
        e = run(ld);
      } else {
        PackedTcLoader<true, false, false> ld{};
        e = run(ld);
      }
    }
    return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_wgrad_packed_implicit: %s", cudaGetErrorString(e));
  });
}

// A = xcol^T (MN-major over kk, 64x64 TMA boxes); B = dY (MN-major over C_out):
// TMA boxes when C_out >= 64, else cp.async chunks gathered by the producers.
template <bool TMA_B>
struct WgradPackedLoader {
  static constexpr int A_MN_MAJOR = 1, B_MN_MAJOR = 1;
  static constexpr bool A_TMA_SW128 = true, B_TMA_SW128 = TMA_B, PURE_TMA = TMA_B;
  CUtensorMap amap;  // xcol [Mo][Kp]
  CUtensorMap dmap;  // dY [Mo][co] (TMA_B)
  const bf16* dy;
  int co, Kp, Mo, BN;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int ptid, const uint8_t*,
                       uint64_t* full) const {
    if (ptid == 0) {
      const int nblk = (c.m0 + 64 < Kp) ? 2 : 1;  // a fully out-of-range 64-row block is not loaded
      mbar_expect_tx(full, (uint32_t)nblk * 64u * TC_BK * 2u + (TMA_B ? (uint32_t)BN * TC_BK * 2u : 0u));
      for (int blk = 0; blk < nblk; ++blk) tma_load_2d(sA + blk * 8192, &amap, c.m0 + 64 * blk, kb * TC_BK, full);
      if (TMA_B)
        for (int j = 0; j < BN / 64; ++j) tma_load_2d(sB + j * 8192, &dmap, c.n0 + 64 * j, kb * TC_BK, full);
    }
    if (TMA_B) return;
    const int groups = BN / 8;
    for (int ch = ptid; ch < groups * TC_BK; ch += TC_PRODUCERS) {
      const int grp = ch % groups, kr = ch / groups;
      const int o0 = c.n0 + grp * 8, m = kb * TC_BK + kr;
      const bool ok = o0 < co && m < Mo;
      cp_async16(sB + mnmajor_off(BN, grp, kr), ok ? (const void*)(dy + (size_t)m * co + o0) : (const void*)dy,
                 ok ? 16u : 0u);
    }
  }
};


// part[split][co][Kp]: split-K partial sums of D^T (row Kr = bias gradient)
// rows: reduction length (default n*oh*ow; pool_rows() for the window-major order)
inline int conv_wgrad_packed(const ConvGeom& g, const bf16* xcol, int Kp, const bf16* dy, float* part,
                             int* splits_out, int num_sms, cudaStream_t st, int rows = 0) {
  const int Mo = rows > 0 ? rows : g.n * g.oh * g.ow;
  return with_bn(g.co, [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    TcShape sh = tc_make_shape(Kp, g.co, Mo, BN, conv_wgrad_packed_splits(Kp, Mo, num_sms));
    *splits_out = sh.splits;
    WgradTcEpi ep{part, Kp, g.co};
    cudaError_t e;
    auto fill = [&](auto& ld) {
      ld.dy = dy; ld.co = g.co; ld.Kp = Kp; ld.Mo = Mo; ld.BN = BN;
    };
    if constexpr (BN >= 64) {
      WgradPackedLoader<true> ld{};
      fill(ld);
      if (!make_tmap_mn64(&ld.amap, xcol, Mo, Kp) || !make_tmap_mn64(&ld.dmap, dy, Mo, g.co))
        return fail(CE_ECUDA, "conv_wgrad_packed: tensor map encoding failed");
      e = tc_launch<BN>(ld, ep, sh, num_sms, st);
    } else {
      WgradPackedLoader<false> ld{};
      fill(ld);
      if (!make_tmap_mn64(&ld.amap, xcol, Mo, Kp)) return fail(CE_ECUDA, "conv_wgrad_packed: tensor map failed");
      e = tc_launch<BN>(ld, ep, sh, num_sms, st);
    }
    return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_wgrad_packed: %s", cudaGetErrorString(e));
  });
}

// Reduce the split partials (one warp per element, fixed order) and apply the
// momentum update (nn.py:306-322): kk < Kr -> master W[o][i][j][c] (+ packed
// bf16 mirror), kk == Kr -> bias.
template <class TW>
__global__ void __launch_bounds__(256) conv_sgd_packed_kernel(
    const float* __restrict__ part, int splits, int co, int Kp, int k, int cp, int c_real, float* __restrict__ w,
    float* __restrict__ vel, float* __restrict__ gw, TW* __restrict__ wp, float* __restrict__ b,
    float* __restrict__ vb, float* __restrict__ gb, float lr, float mu) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Kr = k * k * kPackedCpt;
  const size_t e = (size_t)blockIdx.x * 8 + warp;  // over co x (Kr + 1)
  if (e >= (size_t)co * (Kr + 1)) return;
  const int o = (int)(e / (Kr + 1)), kk = (int)(e % (Kr + 1));
  const float g = warp_sum_splits(part, splits, (size_t)co * Kp, (size_t)o * Kp + kk);
  if (lane != 0) return;
  if (kk == Kr) {
    if (gb) gb[o] = g;
    if (b) {
      float bv = b[o], v = vb[o];
      sgd_update(bv, v, g, lr, mu);
      b[o] = bv;
      vb[o] = v;
    }
    return;
  }
  const int tap = kk / kPackedCpt, c = kk - tap * kPackedCpt;
  if (c >= c_real) return;  // zero column of the packing: no parameter
  const size_t mi = ((size_t)o * k * k + tap) * cp + c;
  if (gw) gw[mi] = g;
  if (!w) return;
  float wv = w[mi], vv = vel[mi];
  sgd_update(wv, vv, g, lr, mu);
  w[mi] = wv;
  vel[mi] = vv;
  if (wp) stf(wp, (size_t)o * Kp + kk, wv);
}

template <class TW>
inline void launch_conv_sgd_packed(const float* part, int splits, const ConvGeom& g, int c_real, int Kp, float* w,
                                   float* vel, float* gw, TW* wp, float* b, float* vb, float* gb, float lr,
                                   float mu, cudaStream_t st) {
  const size_t elems = (size_t)g.co * (packed_kr(g, c_real) + 1);
  conv_sgd_packed_kernel<TW><<<(unsigned)((elems + 7) / 8), 256, 0, st>>>(part, splits, g.co, Kp, g.k, g.c, c_real,
                                                                          w, vel, gw, wp, b, vb, gb, lr, mu);
}

template <class T>
inline void launch_im2col_packed(const T* x, const ConvGeom& g, int c_real, int Kp, T* xcol, cudaStream_t st,
                                 const PoolMap* pm = nullptr) {
  if (pm) {
    const uint32_t rows = (uint32_t)pool_rows(*pm);
    im2col_packed_kernel<T, true><<<grid_for((size_t)rows * (Kp / 8)), 256, 0, st>>>(
        x, g, c_real, Kp, FastDiv(Kp / 8), FastDiv(g.ow), FastDiv(g.oh), xcol, *pm, rows);
    return;
  }
  const uint32_t rows = (uint32_t)g.n * g.oh * g.ow;
  im2col_packed_kernel<T, false><<<grid_for((size_t)rows * (Kp / 8)), 256, 0, st>>>(
      x, g, c_real, Kp, FastDiv(Kp / 8), FastDiv(g.ow), FastDiv(g.oh), xcol, PoolMap{}, rows);
}

// fp32 check mode: the same packed GEMMs on CUDA cores (simt_gemm over plain operands)
inline void conv_fwd_packed_simt(const ConvGeom& g, const float* xcol, int Kp, const float* wpf, const float* bias,
                                 int relu, float* y, cudaStream_t st) {
  const int M = g.n * g.oh * g.ow;
  simt_gemm(DenseXA<float>{xcol, Kp}, FwdB{wpf, Kp}, FwdEpi<float>{y, bias, g.co, relu != 0}, M, g.co, Kp, 1, st);
}
inline void conv_wgrad_packed_simt(const ConvGeom& g, const float* xcol, int Kp, const float* dy, float* part,
                                   int splits, cudaStream_t st) {
  const int Mo = g.n * g.oh * g.ow;
  simt_gemm(WgradA<float>{dy, g.co}, DenseXN<float>{xcol, Kp}, PartialEpi{part, g.co, Kp}, g.co, Kp, Mo, splits, st);
}

}  // namespace ce
