// Convolution forward / dgrad / wgrad as implicit GEMMs on the tcgen05 engine.
//
// All three passes put a channel count on the UMMA N axis (<= 256, so one N
// tile per problem) and gather 16-byte chunks of 8 consecutive channels:
//
//   fwd  : D[(n,p,q)][o]  = sum_{(i,j,c)} x[n, sp+i, sq+j, c] * W[o][i][j][c]      A,B K-major
//          epilogue: + bias, ReLU, bf16 NHWC store                 (nn.py:82-94, 178-180)
//   dgrad: D[(n,h,w)][c]  = sum_{(i,j,o)} dy[n, (h-i)/s, (w-j)/s, o] * Wt[c][i][j][o]   A,B K-major
//          one stride-1 GEMM per residue class (h mod s, w mod s) over that class's
//          taps only (sub-pixel decomposition); out-of-range taps are zero-filled;
//          epilogue: x ReLU mask of the input activation, bf16 store  (nn.py:112-113, 183)
//   wgrad: D[(i,j,c)][o]  = sum_{(n,p,q)} x[n, sp+i, sq+j, c] * dy[n,p,q,o]           A,B MN-major
//          reduction split across CTAs; epilogue writes fp32 partials part[split][o][(i,j,c)]
//          that conv_sgd_kernel reduces in fixed order and feeds to the momentum update
//          (nn.py:108-115, 306-322)
#pragma once
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "tc_engine.cuh"
#include "kernels.cuh"

namespace ce {

inline bool conv_tc_enabled() {
  const char* e = getenv("CE_DISABLE_TC");
  return !(e && e[0] == '1');
}

// TMA descriptor for a K-major bf16 operand [rows][K] (K contiguous, K % 8 == 0):
// box = 64 K-elements (128 B, SWIZZLE_128B) x `box_rows` rows; OOB reads are zeros.
inline bool make_tmap_kmajor(CUtensorMap* map, const bf16* base, int rows, int K, int box_rows, int row_stride = 0) {
  if (row_stride <= 0) row_stride = K;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_stride * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// TMA descriptor for an MN-major operand stored [K rows][MN] (MN contiguous):
// boxes of 64 MN-elements x 64 K-rows with SWIZZLE_128B.
inline bool make_tmap_mn64(CUtensorMap* map, const bf16* base, int krows, int mn) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)mn, (cuuint64_t)krows};
  cuuint64_t strides[1] = {(cuuint64_t)mn * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)base, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The same [K rows][MN] operand as `nslab` 64-wide MN slabs in ONE copy: a 3-D
// view {64 MN, K rows, MN / 64 slabs} (slab stride 128 B) whose box lands as
// nslab consecutive 8 KB SW128 blocks, the layout of nslab make_tmap_mn64 boxes.
// One TMA issue instead of nslab (the producer's per-copy issue cost dominates
// short k-blocks: profiles/r02_tc_trace/).
inline bool make_tmap_mn64_slabs(CUtensorMap* map, const bf16* base, int krows, int mn, int nslab) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
  }
  if (mn % 64 != 0 || nslab < 1) return false;
  cuuint64_t dims[3] = {64, (cuuint64_t)krows, (cuuint64_t)(mn / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)mn * 2, 128};
  cuuint32_t box[3] = {64, 64, (cuuint32_t)nslab};
  cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)base, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA im2col descriptor over an NHWC bf16 activation for a valid (unpadded)
// convolution with kernel k and stride s: `pixels` output pixels x 64 channels
// per copy (128 B rows, SWIZZLE_128B), receptive-field origins traversed in
// (n, p, q) order with stride s (bounding box shrunk by k-1 on the far side).
inline bool make_tmap_im2col(CUtensorMap* map, const bf16* x, const ConvGeom& g, int pixels, int cpp = 64) {
  static PFN_cuTensorMapEncodeIm2col_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
  }
  cuuint64_t dims[4] = {(cuuint64_t)g.c, (cuuint64_t)g.w, (cuuint64_t)g.h, (cuuint64_t)g.n};
  cuuint64_t strides[3] = {(cuuint64_t)g.c * 2, (cuuint64_t)g.w * g.c * 2, (cuuint64_t)g.h * g.w * g.c * 2};
  int lower[2] = {0, 0};
  int upper[2] = {-(g.k - 1), -(g.k - 1)};
  cuuint32_t estr[4] = {1, (cuuint32_t)g.s, (cuuint32_t)g.s, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)x, dims, strides, lower, upper,
                      (cuuint32_t)cpp, (cuuint32_t)pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      cpp == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                      : cpp == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  // driver <= 13.1 workaround (as in CUTLASS): small tensors must not set bit 21 of word 1
  int drv = 0;
  cudaDriverGetVersion(&drv);
  if (drv <= 13010 && (size_t)g.n * g.h * g.w * g.c * 2 < 131072) reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  return true;
}

// Output tiles as 2-D pixel blocks (stride-1 convolutions): a 128-row GEMM tile
// is a BH x BW block of output pixels of one image, rows row-major inside it,
// so the A operand of every (tap, 64-channel slab) is ONE tiled TMA box of the
// input {64 ch, BW, BH, 1} at the block origin shifted by the tap. The im2col
// TMA mode moves a 128-pixel column at ~7 SM cycles per pixel row (measured,
// tools/tc_trace.py), which capped every im2col k-block at ~900 cycles; tiled
// boxes stream at the TMA's full rate. Rows past the map edge are computed on
// zero-filled / neighbouring input and never stored.
struct PixelBlocks {
  int bh, bw_log2, oh, ow, n;
  FastDiv d_bw_tiles, d_bh_tiles;  // blocks per image row / column
  // block origin of tile t = m0 / 128; false past the last block
  __device__ __forceinline__ bool origin(int m0, int& img, int& p0, int& q0) const {
    uint32_t rest, qb, nn, pb;
    d_bw_tiles.divmod((uint32_t)m0 >> 7, rest, qb);
    d_bh_tiles.divmod(rest, nn, pb);
    img = (int)nn;
    p0 = (int)pb * bh;
    q0 = (int)qb << bw_log2;
    return img < n;
  }
  // output pixel index of row `row` of the tile at m0, or -1
  __device__ __forceinline__ int pixel(int m0, int row) const {
    int img, p0, q0;
    if (!origin(m0, img, p0, q0)) return -1;
    const int p = p0 + (row >> bw_log2), q = q0 + (row & ((1 << bw_log2) - 1));
    return (p < oh && q < ow) ? (img * oh + p) * ow + q : -1;
  }
};
// block shape minimising the padded tile count (ties: wider rows)
inline PixelBlocks make_pixel_blocks(int n, int oh, int ow) {
  PixelBlocks b{};
  long long best = -1;
  for (int l = 7; l >= 3; --l) {
    const int bw = 1 << l, bh = TC_BM / bw;
    const long long cost = (long long)((oh + bh - 1) / bh) * ((ow + bw - 1) / bw);
    if (best < 0 || cost < best) {
      best = cost;
      b.bw_log2 = l;
      b.bh = bh;
    }
  }
  b.oh = oh;
  b.ow = ow;
  b.n = n;
  b.d_bw_tiles = FastDiv((uint32_t)((ow + (1 << b.bw_log2) - 1) >> b.bw_log2));
  b.d_bh_tiles = FastDiv((uint32_t)((oh + b.bh - 1) / b.bh));
  return b;
}
inline int pixel_block_tiles(const PixelBlocks& b) {
  return b.n * ((b.oh + b.bh - 1) / b.bh) * ((b.ow + (1 << b.bw_log2) - 1) >> b.bw_log2);
}
// tiled 4-D map over an NHWC bf16 tensor: boxes {64 channels, bw, bh, 1}, SWIZZLE_128B
inline bool make_tmap_blocks(CUtensorMap* map, const bf16* x, int n, int h, int w, int c, int bh, int bw) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
  }
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, (cuuint64_t)h * w * c * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)bw, (cuuint32_t)bh, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)x, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// CE_PIXEL_BLOCKS=1 (opt-in): measured no faster than the im2col TMA once the MMA
// issue was made warp-converged, and the padded blocks waste rows on small maps
inline bool pixel_blocks_enabled() {
  static const bool on = [] {
    const char* e = getenv("CE_PIXEL_BLOCKS");
    return e && e[0] == '1';
  }();
  return on;
}

inline bool tma_disabled() {
  const char* e = getenv("CE_DISABLE_TMA");
  return e && e[0] == '1';
}
inline bool im2col_disabled() {
  const char* e = getenv("CE_DISABLE_IM2COL");
  return e && e[0] == '1';
}
// 8-channel im2col copies (C < 64) measured slower than the cp.async gather
// (16-byte TMA boxes); opt-in only.
inline bool narrow_im2col_enabled() {
  const char* e = getenv("CE_NARROW_IM2COL");
  return e && e[0] == '1';
}

// ------------------------------------------------------------------ pooled row order
// A conv whose output feeds a non-overlapping max-pool (stride >= window,
// nn.py:119-150) runs its GEMM rows in WINDOW-MAJOR order, so the epilogue sees
// every pool window inside one warp and emits the pooled value + argmax
// directly (FwdPoolEpi): the pre-pool activation is never written. Row r of
// tile t: warp quarter wq = r / 32, lane l = r % 32 -> window
// t*WPT + wq*WPW + l / KK, tap l % KK (row-major inside the window, the
// reference's first-max order); lanes >= WPW*KK of a quarter are padding.
// Conv outputs no window covers (stride > window gaps, ragged edges) are never
// computed: the reference routes them a zero gradient (nn.py:156-167).
struct PoolMap {
  int KK, WPW, WPT;  // taps per window; windows per 32-row warp quarter / per 128-row tile
  int ps, pst;       // pool window and stride
  int windows;       // n * PH * PW = pooled pixels
  FastDiv d_pw, d_ph, d_kk, d_ps;
  // conv output pixel (n, p, q) of row r of tile t; false for a padding row
  __device__ __forceinline__ bool pixel(int t, int r, uint32_t& n, uint32_t& p, uint32_t& q) const {
    uint32_t wl, tap;
    d_kk.divmod((uint32_t)(r & 31), wl, tap);
    if ((int)wl >= WPW) return false;
    const int window = t * WPT + (r >> 5) * WPW + (int)wl;
    if (window >= windows) return false;
    uint32_t rest, pw, ph, di, dj;
    d_pw.divmod((uint32_t)window, rest, pw);
    d_ph.divmod(rest, n, ph);
    d_ps.divmod(tap, di, dj);
    p = ph * pst + di;
    q = pw * pst + dj;
    return true;
  }
};

inline PoolMap make_pool_map(int n, int oh, int ow, int ps, int pst) {
  PoolMap pm{};
  const int PH = (oh - ps) / pst + 1, PW = (ow - ps) / pst + 1;
  pm.ps = ps;
  pm.pst = pst;
  pm.KK = ps * ps;
  pm.WPW = 32 / pm.KK;
  pm.WPT = 4 * pm.WPW;
  pm.windows = n * PH * PW;
  pm.d_pw = FastDiv(PW);
  pm.d_ph = FastDiv(PH);
  pm.d_kk = FastDiv(pm.KK);
  pm.d_ps = FastDiv(ps);
  return pm;
}
// GEMM rows of the pooled order (whole 128-row tiles)
inline int pool_rows(const PoolMap& pm) { return (pm.windows + pm.WPT - 1) / pm.WPT * TC_BM; }
inline bool pool_fusable(int ps, int pst) { return (ps == 2 || ps == 3) && pst >= ps; }

// ------------------------------------------------------------------ forward
// table: xoff[k8] = im2col offset of K chunk k8 = (tap, c0) relative to the
// output pixel's receptive-field origin: (i*W + j)*C + c0.
// POOL: rows in the window-major order of `pm` (gather modes 0 / 1 only).
template <int MODE, bool POOL = false>
struct FwdTcLoader;

// 32-channel im2col forward (C % 64 == 32, e.g. the FIXED genome's second layer):
// per k-block two TMA im2col boxes of 128 pixels x 32 channels (SWIZZLE_64B, one per
// 32-deep K half: tap 2kb and 2kb+1 when C = 32) + the weight box. Replaces the
// cp.async gather, whose 1,024 16-byte requests per k-block cost ~2,200 SM cycles
// (profiles/r02_tc_trace/).
struct FwdTcLoader32 {
  static constexpr int A_MN_MAJOR = 0, B_MN_MAJOR = 0;
  static constexpr bool A_TMA_SW128 = false, A_SW64 = true, B_TMA_SW128 = true, PURE_TMA = true, KB2 = true;
  CUtensorMap wmap, xmap;
  ConvGeom g;
  int K, M, BN;
  FastDiv d_ow, d_oh, d_c, d_k;
  __device__ void init(uint8_t*, int tid, int) const {
    if (tid == 0) {
      tma_prefetch_desc(&wmap);
      tma_prefetch_desc(&xmap);
    }
  }
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int, const uint8_t*,
                       uint64_t* full) const {
    uint32_t q, p, n, t;
    d_ow.divmod((uint32_t)c.m0, t, q);
    d_oh.divmod(t, n, p);
    mbar_expect_tx(full, (uint32_t)(2 * TC_BM * 64 + BN * 128));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t kk = (uint32_t)(kb * TC_BK + h * 32);
      uint32_t tap = 0, c0 = (uint32_t)g.c, i = 0, j = 0;  // past K: a fully out-of-bounds box zero-fills
      if ((int)kk < K) {
        d_c.divmod(kk, tap, c0);
        d_k.divmod(tap, i, j);
      }
      tma_load_im2col_4d(sA + (uint32_t)h * (TC_BM * 64), &xmap, (int)c0, (int)q * g.s, (int)p * g.s, (int)n,
                         (uint16_t)j, (uint16_t)i, full);
    }
    tma_load_2d(sB, &wmap, kb * TC_BK, c.n0, full);
  }
};

// 32-channel TMA path enabled (CE_IM2COL32=0: the cp.async gather, for comparison)
inline bool im2col32_enabled() {
  static const bool on = [] {
    const char* e = getenv("CE_IM2COL32");
    return !(e && e[0] == '0');
  }();
  return on;
}
inline bool im2col32_ok(const ConvGeom& g) {
  return im2col32_enabled() && g.c % 32 == 0 && g.c % 64 != 0 && !tma_disabled() && !im2col_disabled();
}

template <int MODE, bool POOL>
struct FwdTcLoader {
  // MODE 0: cp.async gather A + cp.async B; 1: gather A + TMA B;
  //      2: TMA im2col A (64-channel slabs, SW128) + TMA B;
  //      3: TMA im2col A in 8-channel chunks (C < 64, interleaved layout) + TMA B
  static constexpr bool TMA_B = MODE >= 1, IM2COL = MODE == 2, NARROW = MODE == 3;
  static constexpr int A_MN_MAJOR = 0, B_MN_MAJOR = 0;
  static constexpr bool A_TMA_SW128 = IM2COL, B_TMA_SW128 = TMA_B, PURE_TMA = IM2COL || NARROW;
  static constexpr bool KB2 = IM2COL;  // two k-blocks per pipeline stage (tc_engine)
  CUtensorMap wmap;  // B operand (weights) when TMA_B
  CUtensorMap xmap;  // im2col view of x when IM2COL
  const bf16* x;
  const bf16* w;  // [o][K]
  ConvGeom g;
  int K, M, BN;
  FastDiv d_ow, d_oh;
  PoolMap pm;  // POOL
  FastDiv d_cpb, d_k;  // k-block -> (tap, 64-channel slab), tap -> (i, j) (IM2COL)
  static_assert(!POOL || MODE <= 1, "the pooled row order needs the gather loader");
  __device__ void init(uint8_t* table, int tid, int nthreads) const {
    if ((IM2COL || NARROW) && tid == 0) {
      tma_prefetch_desc(&wmap);
      tma_prefetch_desc(&xmap);
    }
    if (IM2COL || NARROW) return;
    int* xoff = (int*)table;
    for (int k8 = tid; k8 < K / 8; k8 += nthreads) {
      const int kk = k8 * 8, tap = kk / g.c, c0 = kk - tap * g.c;
      const int i = tap / g.k, j = tap - i * g.k;
      xoff[k8] = (i * g.w + j) * g.c + c0;
    }
  }
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int ptid, const uint8_t* table,
                       uint64_t* full) const {
    const int* xoff = (const int*)table;
    if (IM2COL) {  // one thread: A via im2col TMA (tap, 64-channel slab), B via 2-D TMA
      uint32_t tap, slab, i, j;  // FastDiv: runtime integer divisions cost ~100 cycles each here
      d_cpb.divmod((uint32_t)kb, tap, slab);
      d_k.divmod(tap, i, j);
      const int c0 = (int)slab * 64;
      uint32_t q, p, n, t;
      d_ow.divmod((uint32_t)c.m0, t, q);
      d_oh.divmod(t, n, p);
      mbar_expect_tx(full, (uint32_t)(TC_BM + BN) * 128u);
      tma_load_im2col_4d(sA, &xmap, c0, (int)q * g.s, (int)p * g.s, (int)n, (uint16_t)j, (uint16_t)i, full);
      tma_load_2d(sB, &wmap, kb * TC_BK, c.n0, full);
      return;
    }
    if (NARROW) {  // one thread: 8 im2col copies of 128 pixels x 8 channels (one per 16-byte K chunk)
      uint32_t q, p, n, t;
      d_ow.divmod((uint32_t)c.m0, t, q);
      d_oh.divmod(t, n, p);
      mbar_expect_tx(full, (uint32_t)(8 * TC_BM * 16 + BN * 128));
#pragma unroll 1
      for (int kc = 0; kc < 8; ++kc) {
        const int kk = kb * TC_BK + kc * 8;
        int c0 = g.c, i = 0, j = 0;  // past K: a fully out-of-bounds copy zero-fills the chunk
        if (kk < K) {
          const int tap = kk / g.c;
          c0 = kk - tap * g.c;
          i = tap / g.k;
          j = tap - i * g.k;
        }
        tma_load_im2col_4d(sA + kmajor_off(TC_BM, 0, kc), &xmap, c0, (int)q * g.s, (int)p * g.s, (int)n,
                           (uint16_t)j, (uint16_t)i, full);
      }
      tma_load_2d(sB, &wmap, kb * TC_BK, c.n0, full);
      return;
    }
    if (TMA_B) {
      if (ptid == 0) {
        mbar_expect_tx(full, (uint32_t)BN * 128u);
        tma_load_2d(sB, &wmap, kb * TC_BK, c.n0, full);
      }
    }
    {
      const int r = ptid & (TC_BM - 1), kc0 = ptid >> 7;  // 256 producers: 2 threads per row
      const int m = c.m0 + r;
      uint32_t q = 0, p = 0, n = 0, t = 0;
      bool row_ok;
      if constexpr (POOL) {
        row_ok = pm.pixel(c.m0 / TC_BM, r, n, p, q);
        if (!row_ok) n = p = q = 0;
      } else {
        row_ok = m < M;
        if (row_ok) {
          d_ow.divmod((uint32_t)m, t, q);
          d_oh.divmod(t, n, p);
        }
      }
      const bf16* base = x + (((size_t)n * g.h + p * g.s) * g.w + q * g.s) * g.c;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kc = kc0 + 2 * e;
        const int k8 = kb * 8 + kc;
        const bool ok = row_ok && k8 * 8 < K;
        cp_async16(sA + kmajor_off(TC_BM, r, kc), ok ? (const void*)(base + xoff[k8]) : (const void*)x,
                   ok ? 16u : 0u);
      }
    }
    if (!TMA_B) {
      for (int ch = ptid; ch < BN * 8; ch += TC_PRODUCERS) {
        const int r = ch % BN, kc = ch / BN;
        const int o = c.n0 + r, kk = kb * TC_BK + kc * 8;
        const bool ok = o < g.co && kk < K;
        cp_async16(sB + kmajor_off(BN, r, kc), ok ? (const void*)(w + (size_t)o * K + kk) : (const void*)w,
                   ok ? 16u : 0u);
      }
    }
  }
};

// Stride-1 forward over pixel blocks (PixelBlocks): per k-block one tiled box
// of x at (c0, q0 + j, p0 + i, img) and one weight box. PAIR: the CTA-pair
// variant (rank r takes block 2t + r and weight rows n0 + r BN / 2; copies
// complete on rank 0's barrier).
template <bool PAIR>
struct FwdBlockLoader {
  static constexpr int A_MN_MAJOR = 0, B_MN_MAJOR = 0;
  static constexpr bool A_TMA_SW128 = true, B_TMA_SW128 = true, PURE_TMA = true;
  CUtensorMap wmap;  // box 64 K x (PAIR ? BN / 2 : BN) rows
  CUtensorMap xmap;  // make_tmap_blocks
  PixelBlocks pb;
  int cin, k, BN;
  FastDiv d_cpb, d_k;
  __device__ void init(uint8_t*, int tid, int) const {
    if (tid == 0) {
      tma_prefetch_desc(&wmap);
      tma_prefetch_desc(&xmap);
    }
  }
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int, const uint8_t*,
                       uint64_t* full) const {
    uint32_t tap, slab, i, j;
    d_cpb.divmod((uint32_t)kb, tap, slab);
    d_k.divmod(tap, i, j);
    const int c0 = (int)slab * 64;
    int img, p0, q0;
    pb.origin(c.m0, img, p0, q0);
    if constexpr (PAIR) {
      const uint32_t rank = cluster_ctarank();
      if (rank == 0) mbar_expect_tx(full, (uint32_t)(2 * TC_BM + BN) * 128u);
      tma_load_4d_pair(sA, &xmap, c0, q0 + j, p0 + i, img, full);
      tma_load_2d_pair(sB, &wmap, kb * TC_BK, c.n0 + (int)rank * (BN / 2), full);
    } else {
      mbar_expect_tx(full, (uint32_t)(TC_BM + BN) * 128u);
      tma_load_4d(sA, &xmap, c0, q0 + j, p0 + i, img, full);
      tma_load_2d(sB, &wmap, kb * TC_BK, c.n0, full);
    }
  }
};

// CTA-pair forward loader (tc_gemm_kernel<..., PAIR = true>): the im2col TMA of
// FwdTcLoader<2> for this CTA's 128 rows, and B rows n0 + rank * BN / 2 (a
// BN / 2-row weight box); every copy completes on rank 0's barrier, which
// rank 0 primes with the pair's total bytes.
struct FwdTcLoaderPair {
  static constexpr int A_MN_MAJOR = 0, B_MN_MAJOR = 0;
  static constexpr bool A_TMA_SW128 = true, B_TMA_SW128 = true, PURE_TMA = true, KB2 = true;
  CUtensorMap wmap;  // box: 64 K x BN / 2 rows
  CUtensorMap xmap;  // im2col, 128 pixels x 64 channels
  ConvGeom g;
  int K, M, BN;
  FastDiv d_ow, d_oh, d_cpb, d_k;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int, const uint8_t*,
                       uint64_t* full) const {
    const uint32_t rank = cluster_ctarank();
    uint32_t tap, slab, i, j;
    d_cpb.divmod((uint32_t)kb, tap, slab);
    d_k.divmod(tap, i, j);
    const int c0 = (int)slab * 64;
    uint32_t q, p, n, t;
    d_ow.divmod((uint32_t)c.m0, t, q);
    d_oh.divmod(t, n, p);
    if (rank == 0) mbar_expect_tx(full, (uint32_t)(2 * TC_BM + BN) * 128u);
    tma_load_im2col_4d_pair(sA, &xmap, c0, (int)q * g.s, (int)p * g.s, (int)n, (uint16_t)j, (uint16_t)i, full);
    tma_load_2d_pair(sB, &wmap, kb * TC_BK, c.n0 + (int)rank * (BN / 2), full);
  }
};

struct FwdTcEpi {
  static constexpr bool STAGED_BF16 = true;  // coalesced row stores through shared memory (tc_engine)
  // pure-TMA loaders (1 producer warp) leave room for 16 epilogue warps: the bf16
  // store stream is the limit of the wide forwards (gather loaders keep 8: registers)
  static constexpr int EPI_WARPS_TMA = 16;
  static constexpr int EPI_WARPS_SYNC = 16;  // implicit packed first layer: 8 producer warps, light registers
  bf16* y;
  const float* bias;
  int M, co, relu;
  PixelBlocks pb{};  // pb.bh > 0: rows are pixel blocks (FwdBlockLoader), else m = m0 + row
  __device__ __forceinline__ int row_pixel(const TileCoord& c, int row) const {
    if (pb.bh > 0) return pb.pixel(c.m0, row);
    const int m = c.m0 + row;
    return m < M ? m : -1;
  }
  // bias + ReLU of columns c.n0 + col .. +15 (row independent)
  // out[i] = bf16x2 of columns 2i, 2i+1
  __device__ void convert(const TileCoord& c, int col, const float (&v)[16], uint32_t (&out)[8]) const {
    const int o0 = c.n0 + col;
    float bv[16];
    if (o0 + 16 <= co) {  // co % 8 == 0 and o0 % 16 == 0: 16-byte aligned
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float4 b4 = __ldg((const float4*)(bias + o0) + h);
        bv[4 * h] = b4.x; bv[4 * h + 1] = b4.y; bv[4 * h + 2] = b4.z; bv[4 * h + 3] = b4.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) bv[i] = o0 + i < co ? __ldg(bias + o0 + i) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float t0 = v[2 * i] + bv[2 * i], t1 = v[2 * i + 1] + bv[2 * i + 1];
      if (relu) {
        t0 = t0 > 0.f ? t0 : 0.f;
        t1 = t1 > 0.f ? t1 : 0.f;
      }
      const __nv_bfloat162 h = __floats2bfloat162_rn(t0, t1);
      out[i] = *(const uint32_t*)&h;
    }
  }
  // destination of the 8-column half `half` of row `row` at columns col.., or null
  __device__ bf16* row_ptr(const TileCoord& c, int row, int col, int half) const {
    const int m = row_pixel(c, row), o = c.n0 + col + half * 8;
    return (m >= 0 && o < co) ? y + (size_t)m * co + o : nullptr;
  }
  __device__ void store(const TileCoord& c, int row, int col, const float (&v)[16]) const {
    const int m = row_pixel(c, row);
    const int o0 = c.n0 + col;
    if (m < 0 || o0 >= co) return;
    bf16* dst = y + (size_t)m * co + o0;
    __align__(16) bf16 out[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float t = v[i] + (o0 + i < co ? __ldg(bias + o0 + i) : 0.f);
      if (relu) t = t > 0.f ? t : 0.f;
      out[i] = __float2bfloat16_rn(t);
    }
    *(uint4*)dst = *(const uint4*)&out[0];
    if (o0 + 8 < co) *(uint4*)(dst + 8) = *(const uint4*)&out[8];
  }
  __device__ void finish(int, int) const {}
};

// Pooled forward epilogue (rows in PoolMap order): bias + ReLU, rounded to the
// bf16 the unfused path would store; each warp stages its 32 rows x 16 columns
// in shared memory and then every lane reduces (window, column) pairs over the
// window's KK rows: max with maxpool_fwd_kernel's first-max rule (a later tap
// wins only if strictly greater), argmax kPoolDead when the window came out of
// a ReLU and its max is not > 0. Stores the pooled bf16 value and the u8
// argmax in NHWC order of the pooled map (half-warps write 32 contiguous bytes).
template <int KK>
struct FwdPoolEpi {
  // the epilogue reads KK rows per output: 16 warps (4 per scheduler) keep it from limiting the kernel
  static constexpr int EPI_WARPS = 16;
  static constexpr int WPW = 32 / KK;
  static constexpr int ROW = 24;                 // staged row stride in bf16 (48 B: conflict-free window reads)
  static constexpr int WARP_SMEM = 32 * ROW * 2;  // per epilogue warp
  bf16* y;       // pooled [windows][co]
  uint8_t* arg;  // [windows][co]
  const float* bias;
  int co, relu;
  PoolMap pm;
  __device__ void store_warp(const TileCoord& c, int q, int col, const float (&v)[16], uint8_t* scratch) const {
    const int lane = threadIdx.x & 31;
    const int o0 = c.n0 + col;
    bf16* st = (bf16*)scratch;
    {
      float bv[16];
      if (o0 + 16 <= co) {  // co % 8 == 0, o0 % 16 == 0: 16-byte aligned
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float4 b4 = __ldg((const float4*)(bias + o0) + h);
          bv[4 * h] = b4.x; bv[4 * h + 1] = b4.y; bv[4 * h + 2] = b4.z; bv[4 * h + 3] = b4.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) bv[i] = o0 + i < co ? __ldg(bias + o0 + i) : 0.f;
      }
      uint32_t r[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float t0 = v[2 * i] + bv[2 * i], t1 = v[2 * i + 1] + bv[2 * i + 1];
        if (relu) {
          t0 = t0 > 0.f ? t0 : 0.f;
          t1 = t1 > 0.f ? t1 : 0.f;
        }
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(t0, t1);
        r[i] = *(const uint32_t*)&h2;
      }
      uint4* dst = (uint4*)(st + lane * ROW);
      dst[0] = make_uint4(r[0], r[1], r[2], r[3]);
      dst[1] = make_uint4(r[4], r[5], r[6], r[7]);
    }
    __syncwarp();
    const int window0 = (c.m0 / TC_BM) * (4 * WPW) + q * WPW;
#pragma unroll
    for (int p = lane; p < WPW * 16; p += 32) {
      const int wl = p >> 4, cc = p & 15;
      const int window = window0 + wl, o = o0 + cc;
      const bf16* src = st + wl * KK * ROW + cc;
      bf16 bb = src[0];
      float bv = __bfloat162float(bb);
      int b = 0;
#pragma unroll
      for (int k = 1; k < KK; ++k) {
        const bf16 ub = src[k * ROW];
        const float u = __bfloat162float(ub);
        if (u > bv) {
          bv = u;
          bb = ub;
          b = k;
        }
      }
      if (window < pm.windows && o < co) {
        const size_t off = (size_t)window * co + o;
        y[off] = bb;
        arg[off] = (relu && !(bv > 0.f)) ? kPoolDead : (uint8_t)b;
      }
    }
    __syncwarp();
  }
  __device__ void finish(int, int) const {}
};

template <class Fn>
inline int with_pool_kk(int ps, Fn&& fn) {
  if (ps == 2) return fn(std::integral_constant<int, 4>());
  return fn(std::integral_constant<int, 9>());
}

// ------------------------------------------------------------------ dgrad
// Sub-pixel decomposition: input positions (h, w) = (rh + s*hh, rw + s*ww) of one
// residue class (rh, rw) only receive taps i = rh + s*a, j = rw + s*b, from
// dy[n, hh - a, ww - b]; each class is a dense stride-1 implicit GEMM with
// K = ti*tj*C_out, so no MMA work is spent on off-lattice taps.
// table per K chunk k8 = (a, b, o0): dy offset delta, packed (a, b), Wt offset.
struct DgradClass {
  int rh, rw;   // residue class
  int ti, tj;   // valid taps per axis
  int hc, wc;   // positions of the class per axis
};

template <int MODE>
struct DgradTcLoader {
  // MODE as FwdTcLoader (3 = 8-channel im2col chunks for C_out < 64)
  static constexpr bool TMA_B = MODE >= 1, IM2COL = MODE == 2, NARROW = MODE == 3;
  static constexpr int A_MN_MAJOR = 0, B_MN_MAJOR = 0;
  static constexpr bool A_TMA_SW128 = IM2COL, B_TMA_SW128 = TMA_B, PURE_TMA = IM2COL || NARROW;
  static constexpr bool KB2 = IM2COL;
  CUtensorMap wmap;  // class block [c][K] when TMA_B
  CUtensorMap dmap;  // im2col view of dY for this class when IM2COL
  const bf16* dy;
  const bf16* wt;  // this class's block [c][K] of the class-blocked transpose
  ConvGeom g;
  DgradClass cl;
  int K, M, BN;    // K = ti*tj*co, M = n*hc*wc
  FastDiv d_wc, d_hc, d_cpb, d_tj;
  __device__ void init(uint8_t* table, int tid, int nthreads) const {
    if (IM2COL || NARROW) return;
    const int nk8 = K / 8;
    int* doff = (int*)table;
    int* dab = doff + nk8;
    int* woff = dab + nk8;
    for (int k8 = tid; k8 < nk8; k8 += nthreads) {
      const int kk = k8 * 8, tap = kk / g.co, o0 = kk - tap * g.co;
      const int a = cl.ti - 1 - tap / cl.tj, b = cl.tj - 1 - (tap - (tap / cl.tj) * cl.tj);  // flipped taps
      const int i = cl.rh + g.s * a, j = cl.rw + g.s * b;
      doff[k8] = o0 - (a * g.ow + b) * g.co;
      dab[k8] = (a << 16) | b;
      woff[k8] = kk;
      (void)i;
      (void)j;
    }
  }
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int ptid, const uint8_t* table,
                       uint64_t* full) const {
    const int nk8 = K / 8;
    if (IM2COL) {  // one thread: A = im2col of dY (flipped class taps, 64 channels), B = class weights
      uint32_t tap, slab, ap, bp;
      d_cpb.divmod((uint32_t)kb, tap, slab);
      d_tj.divmod(tap, ap, bp);
      const int o0 = (int)slab * 64;
      uint32_t ww, hh, n, t;
      d_wc.divmod((uint32_t)c.m0, t, ww);
      d_hc.divmod(t, n, hh);
      mbar_expect_tx(full, (uint32_t)(TC_BM + BN) * 128u);
      tma_load_im2col_4d(sA, &dmap, o0, (int)ww - (cl.tj - 1), (int)hh - (cl.ti - 1), (int)n, (uint16_t)bp,
                         (uint16_t)ap, full);
      tma_load_2d(sB, &wmap, kb * TC_BK, c.n0, full);
      return;
    }
    if (NARROW) {
      uint32_t ww, hh, n, t;
      d_wc.divmod((uint32_t)c.m0, t, ww);
      d_hc.divmod(t, n, hh);
      mbar_expect_tx(full, (uint32_t)(8 * TC_BM * 16 + BN * 128));
#pragma unroll 1
      for (int kc = 0; kc < 8; ++kc) {
        const int kk = kb * TC_BK + kc * 8;
        int o0 = g.co, ap = 0, bp = 0;  // past K: out-of-bounds copy zero-fills the chunk
        if (kk < K) {
          const int tap = kk / g.co;
          o0 = kk - tap * g.co;
          ap = tap / cl.tj;
          bp = tap - ap * cl.tj;
        }
        tma_load_im2col_4d(sA + kmajor_off(TC_BM, 0, kc), &dmap, o0, (int)ww - (cl.tj - 1), (int)hh - (cl.ti - 1),
                           (int)n, (uint16_t)bp, (uint16_t)ap, full);
      }
      tma_load_2d(sB, &wmap, kb * TC_BK, c.n0, full);
      return;
    }
    if (TMA_B && ptid == 0) {
      mbar_expect_tx(full, (uint32_t)BN * 128u);
      tma_load_2d(sB, &wmap, kb * TC_BK, c.n0, full);
    }
    const int* doff = (const int*)table;
    const int* dab = doff + nk8;
    const int* woff = dab + nk8;
    {
      const int r = ptid & (TC_BM - 1), kc0 = ptid >> 7;
      const int m = c.m0 + r;
      const bool row_ok = m < M;
      uint32_t ww = 0, hh = 0, n = 0, t = 0;
      if (row_ok) {
        d_wc.divmod((uint32_t)m, t, ww);
        d_hc.divmod(t, n, hh);
      }
      const bf16* row = dy + (((size_t)n * g.oh + hh) * g.ow + ww) * g.co;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kc = kc0 + 2 * e;
        const int k8 = kb * 8 + kc;
        bool ok = row_ok && k8 < nk8;
        const bf16* src = dy;
        if (ok) {
          const int ab = dab[k8], a = ab >> 16, b = ab & 0xFFFF;
          ok = (int)hh >= a && (int)ww >= b && (int)hh - a < g.oh && (int)ww - b < g.ow;
          if (ok) src = row + doff[k8];
        }
        cp_async16(sA + kmajor_off(TC_BM, r, kc), src, ok ? 16u : 0u);
      }
    }
    if (!TMA_B) {
      for (int ch = ptid; ch < BN * 8; ch += TC_PRODUCERS) {
        const int r = ch % BN, kc = ch / BN;
        const int cc = c.n0 + r, k8 = kb * 8 + kc;
        const bool ok = cc < g.c && k8 < nk8;
        cp_async16(sB + kmajor_off(BN, r, kc), ok ? (const void*)(wt + (size_t)cc * K + woff[k8]) : (const void*)wt,
                   ok ? 16u : 0u);
      }
    }
  }
};

// im2col view of dY for one dgrad residue class: a stride-1 "full" convolution
// with a ti x tj kernel, i.e. padding ti-1 / tj-1 on the near side and a far
// edge that yields exactly hc x wc receptive-field origins.
inline bool make_tmap_im2col_dgrad(CUtensorMap* map, const bf16* dy, const ConvGeom& g, const DgradClass& cl,
                                   int cpp = 64) {
  static PFN_cuTensorMapEncodeIm2col_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
  }
  cuuint64_t dims[4] = {(cuuint64_t)g.co, (cuuint64_t)g.ow, (cuuint64_t)g.oh, (cuuint64_t)g.n};
  cuuint64_t strides[3] = {(cuuint64_t)g.co * 2, (cuuint64_t)g.ow * g.co * 2, (cuuint64_t)g.oh * g.ow * g.co * 2};
  int lower[2] = {-(cl.tj - 1), -(cl.ti - 1)};
  int upper[2] = {cl.wc - g.ow - (cl.tj - 1), cl.hc - g.oh - (cl.ti - 1)};
  if (lower[0] < -128 || lower[1] < -128 || upper[0] < -128 || upper[1] < -128 || upper[0] > 127 || upper[1] > 127)
    return false;
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)dy, dims, strides, lower, upper,
                      (cuuint32_t)cpp, TC_BM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      cpp == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  int drv = 0;
  cudaDriverGetVersion(&drv);
  if (drv <= 13010 && (size_t)g.n * g.oh * g.ow * g.co * 2 < 131072)
    reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  return true;
}

// CTA-pair dgrad loader (one sub-pixel class): FwdTcLoaderPair's scheme over the
// class's im2col view of dY and its weight block
struct DgradTcLoaderPair {
  static constexpr int A_MN_MAJOR = 0, B_MN_MAJOR = 0;
  static constexpr bool A_TMA_SW128 = true, B_TMA_SW128 = true, PURE_TMA = true, KB2 = true;
  CUtensorMap wmap;  // class block [c][K], box 64 K x BN / 2 rows
  CUtensorMap dmap;
  ConvGeom g;
  DgradClass cl;
  int K, M, BN;
  FastDiv d_wc, d_hc, d_cpb, d_tj;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int, const uint8_t*,
                       uint64_t* full) const {
    const uint32_t rank = cluster_ctarank();
    uint32_t tap, slab, ap, bp;
    d_cpb.divmod((uint32_t)kb, tap, slab);
    d_tj.divmod(tap, ap, bp);
    const int o0 = (int)slab * 64;
    uint32_t ww, hh, n, t;
    d_wc.divmod((uint32_t)c.m0, t, ww);
    d_hc.divmod(t, n, hh);
    if (rank == 0) mbar_expect_tx(full, (uint32_t)(2 * TC_BM + BN) * 128u);
    tma_load_im2col_4d_pair(sA, &dmap, o0, (int)ww - (cl.tj - 1), (int)hh - (cl.ti - 1), (int)n, (uint16_t)bp,
                            (uint16_t)ap, full);
    tma_load_2d_pair(sB, &wmap, kb * TC_BK, c.n0 + (int)rank * (BN / 2), full);
  }
};

struct DgradTcEpi {
  bf16* dx;
  const bf16* mask;
  ConvGeom g;
  DgradClass cl;
  int M;
  FastDiv d_wc, d_hc;
  __device__ void store(const TileCoord& tc, int row, int col, const float (&v)[16]) const {
    const int m = tc.m0 + row;
    const int c0 = tc.n0 + col;
    if (m >= M || c0 >= g.c) return;
    uint32_t ww, hh, n, t;
    d_wc.divmod((uint32_t)m, t, ww);
    d_hc.divmod(t, n, hh);
    const size_t off = (((size_t)n * g.h + cl.rh + g.s * hh) * g.w + cl.rw + g.s * ww) * g.c + c0;
    __align__(16) bf16 out[16];
    __align__(16) bf16 mk[16];
    if (mask) {
      *(uint4*)&mk[0] = *(const uint4*)(mask + off);
      if (c0 + 8 < g.c) *(uint4*)&mk[8] = *(const uint4*)(mask + off + 8);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float t2 = v[i];
      if (mask && !(__bfloat162float(mk[i]) > 0.f)) t2 = 0.f;
      out[i] = __float2bfloat16_rn(t2);
    }
    *(uint4*)(dx + off) = *(const uint4*)&out[0];
    if (c0 + 8 < g.c) *(uint4*)(dx + off + 8) = *(const uint4*)&out[8];
  }
  __device__ void finish(int, int) const {}
};

// ------------------------------------------------------------------ wgrad
// 32-channel wgrad (C % 64 == 32): A = x patches, MN-major, as four 32-wide
// (tap, channel) blocks of 64 pixels per k-block (TMA im2col, SWIZZLE_64B, 4 KB
// each); B = dY as in WgradTcLoader<2>. Replaces the cp.async gather.
struct WgradTcLoader32 {
  static constexpr int A_MN_MAJOR = 1, B_MN_MAJOR = 1;
  static constexpr bool A_TMA_SW128 = false, A_SW64_MN = true, B_TMA_SW128 = true, PURE_TMA = true, KB2 = true;
  CUtensorMap dmap, dmap3, xmap;
  int slab3;
  ConvGeom g;
  int Kf, Mo, BN;
  FastDiv d_ow, d_oh, d_c, d_k;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int, const uint8_t*,
                       uint64_t* full) const {
    uint32_t q, p, n, t;
    d_ow.divmod((uint32_t)(kb * TC_BK), t, q);
    d_oh.divmod(t, n, p);
    int nblk = 0;
#pragma unroll
    for (int blk = 0; blk < 4; ++blk)
      if (c.m0 + 32 * blk < Kf) ++nblk;
    mbar_expect_tx(full, (uint32_t)BN * TC_BK * 2u + (uint32_t)nblk * 64u * 64u);
    for (int blk = 0; blk < nblk; ++blk) {
      uint32_t tap, c0, i, j;
      d_c.divmod((uint32_t)(c.m0 + 32 * blk), tap, c0);
      d_k.divmod(tap, i, j);
      tma_load_im2col_4d(sA + blk * 4096, &xmap, (int)c0, (int)q * g.s, (int)p * g.s, (int)n, (uint16_t)j,
                         (uint16_t)i, full);
    }
    if (slab3)
      tma_load_3d(sB, &dmap3, 0, kb * TC_BK, c.n0 / 64, full);
    else
      for (int jb = 0; jb < BN / 64; ++jb) tma_load_2d(sB + jb * 8192, &dmap, c.n0 + 64 * jb, kb * TC_BK, full);
  }
};

template <int MODE>
struct WgradTcLoader {
  static constexpr bool TMA_B = MODE >= 1, IM2COL = MODE == 2;
  static constexpr int A_MN_MAJOR = 1, B_MN_MAJOR = 1;
  static constexpr bool A_TMA_SW128 = IM2COL, B_TMA_SW128 = TMA_B, PURE_TMA = IM2COL;
  static constexpr bool KB2 = IM2COL;
  CUtensorMap dmap;  // dY [Mo][co] as 64x64 MN-major SW128 boxes when TMA_B
  CUtensorMap dmap3;  // dY as BN/64 slabs in one copy (make_tmap_mn64_slabs) when slab3
  int slab3;
  CUtensorMap xmap;  // im2col view of x (64 pixels x 64 channels) when IM2COL
  const bf16* x;
  const bf16* dy;
  ConvGeom g;
  int Kf;  // k*k*c (rows of D)
  int Mo;  // reduction length n*oh*ow
  int BN;
  FastDiv d_ow, d_oh, d_c, d_k;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int ptid, const uint8_t*,
                       uint64_t* full) const {
    if (IM2COL) {  // one thread: two 64-row (tap, channel-slab) blocks of A + BN/64 blocks of dY
      uint32_t q, p, n, t;
      d_ow.divmod((uint32_t)(kb * TC_BK), t, q);
      d_oh.divmod(t, n, p);
      uint32_t bytes = (uint32_t)BN * TC_BK * 2u;
      int nblk = 0;
      for (int blk = 0; blk < 2; ++blk)
        if (c.m0 + 64 * blk < Kf) ++nblk;
      bytes += (uint32_t)nblk * 64u * TC_BK * 2u;
      mbar_expect_tx(full, bytes);
      for (int blk = 0; blk < nblk; ++blk) {
        uint32_t tap, c0, i, j;
        d_c.divmod((uint32_t)(c.m0 + 64 * blk), tap, c0);
        d_k.divmod(tap, i, j);
        tma_load_im2col_4d(sA + blk * 8192, &xmap, c0, (int)q * g.s, (int)p * g.s, (int)n, (uint16_t)j,
                           (uint16_t)i, full);
      }
      if (slab3)
        tma_load_3d(sB, &dmap3, 0, kb * TC_BK, c.n0 / 64, full);
      else
        for (int jb = 0; jb < BN / 64; ++jb) tma_load_2d(sB + jb * 8192, &dmap, c.n0 + 64 * jb, kb * TC_BK, full);
      return;
    }
    // A: 16 groups of 8 (i,j,c) rows x 64 reduction indices; 256 producers -> 4 chunks each
    {
      const int grp = ptid & 15;
      const int kk0 = c.m0 + grp * 8;
      const bool grp_ok = kk0 < Kf;
      int tap_off = 0;
      if (grp_ok) {
        const int tap = kk0 / g.c, c0 = kk0 - tap * g.c;
        const int i = tap / g.k, j = tap - i * g.k;
        tap_off = (i * g.w + j) * g.c + c0;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kr = (ptid >> 4) + e * 16;  // 0..63
        const int m = kb * TC_BK + kr;
        const bool ok = grp_ok && m < Mo;
        const bf16* src = x;
        if (ok) {
          uint32_t t, q, p, n;
          d_ow.divmod((uint32_t)m, t, q);
          d_oh.divmod(t, n, p);
          src = x + (((size_t)n * g.h + p * g.s) * g.w + q * g.s) * g.c + tap_off;
        }
        cp_async16(sA + mnmajor_off(TC_BM, grp, kr), src, ok ? 16u : 0u);
      }
    }
    // B: BN/8 groups of 8 output channels x 64 reduction indices
    if (TMA_B) {
      if (ptid == 0) {
        mbar_expect_tx(full, (uint32_t)BN * TC_BK * 2u);
        for (int j = 0; j < BN / 64; ++j) tma_load_2d(sB + j * 8192, &dmap, c.n0 + 64 * j, kb * TC_BK, full);
      }
      return;
    }
    const int groups = BN / 8;
    for (int ch = ptid; ch < groups * TC_BK; ch += TC_PRODUCERS) {
      const int grp = ch % groups, kr = ch / groups;
      const int o0 = c.n0 + grp * 8, m = kb * TC_BK + kr;
      const bool ok = o0 < g.co && m < Mo;
      cp_async16(sB + mnmajor_off(BN, grp, kr), ok ? (const void*)(dy + (size_t)m * g.co + o0) : (const void*)dy,
                 ok ? 16u : 0u);
    }
  }
};

struct WgradTcEpi {
  float* part;  // [split][co][Kf]
  int Kf, co;
  __device__ void store(const TileCoord& c, int row, int col, const float (&v)[16]) const {
    const int kk = c.m0 + row;
    if (kk >= Kf) return;
    float* base = part + (size_t)c.split * co * Kf + kk;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int o = c.n0 + col + i;
      if (o < co) base[(size_t)o * Kf] = v[i];
    }
  }
  __device__ void finish(int, int) const {}
};

// ------------------------------------------------------------------ dispatch
// N-tile width: the smallest power of two >= n (16..256), halved while that
// lowers the wave-quantised cost  ceil(tiles / #SMs) * (BN + 32)  (the +32
// models the per-tile fixed cost: A loads, epilogue, pipeline ramp).
inline int pick_bn(int m_tiles, int n, int num_sms) {
  int bn = 16;
  while (bn < n && bn < 256) bn *= 2;
  auto cost = [&](int b) {
    const long long tiles = (long long)m_tiles * ((n + b - 1) / b);
    return ((tiles + num_sms - 1) / num_sms) * (long long)(b + 32);
  };
  while (bn > 64 && cost(bn / 2) < cost(bn)) bn /= 2;
  return bn;
}

// CTA-pair forward (cta_group::2, FwdTcLoaderPair): im2col-TMA layers (C % 64 == 0)
// with N >= 128 and at least one 256-row tile per pair of SMs. CE_CONV_PAIR=0
// keeps every forward on single-CTA tiles.
inline bool conv_pair_enabled() {
  static const bool on = [] {
    const char* e = getenv("CE_CONV_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}
// Measured (conv_bench, r02 notes): pairs win on large maps with N = 256 (SWEET fwd
// 1,407 -> 1,563 TF/s, dgrad 1,358 -> 1,460) and lose on the VGG16STYLE layers
// (<= 1.4 waves of pair tiles, or N = 128), so: N > 128 and >= 4 waves of pair tiles.
inline bool conv_pair_shape_ok(long long M, int n_cols, int num_sms) {
  const long long pair_tiles = (M + 2 * TC_BM - 1) / (2 * TC_BM);
  return n_cols > 128 && pair_tiles >= 4LL * (num_sms / 2);
}
inline bool conv_pair_ok(const ConvGeom& g, int num_sms) {
  const long long M = (long long)g.n * g.oh * g.ow;
  return conv_pair_enabled() && !tma_disabled() && !im2col_disabled() && g.c % 64 == 0 &&
         conv_pair_shape_ok(M, g.co, num_sms);
}
// N width of a pair tile (128 or 256) by the same wave-quantised cost as pick_bn over SM pairs
inline int pick_bn_pair(int m_tiles, int n, int num_sms) {
  (void)m_tiles;
  (void)num_sms;
  return n > 128 ? 256 : 128;
}

template <class Fn>
inline int with_bn(int n, Fn&& fn) {
  if (n <= 16) return fn(std::integral_constant<int, 16>());
  if (n <= 32) return fn(std::integral_constant<int, 32>());
  if (n <= 64) return fn(std::integral_constant<int, 64>());
  if (n <= 128) return fn(std::integral_constant<int, 128>());
  return fn(std::integral_constant<int, 256>());
}

// Split-K partials of a sub-wave conv forward: part[split][m][o] (fp32, o contiguous)
struct FwdPartialEpi {
  float* part;
  int M, co;
  __device__ void store(const TileCoord& c, int row, int col, const float (&v)[16]) const {
    const int m = c.m0 + row, o0 = c.n0 + col;
    if (m >= M || o0 >= co) return;
    float4* p = (float4*)(part + ((size_t)c.split * M + m) * co + o0);
    p[0] = make_float4(v[0], v[1], v[2], v[3]);
    p[1] = make_float4(v[4], v[5], v[6], v[7]);
    if (o0 + 8 < co) {
      p[2] = make_float4(v[8], v[9], v[10], v[11]);
      p[3] = make_float4(v[12], v[13], v[14], v[15]);
    }
  }
  __device__ void finish(int, int) const {}
};

// y[m][o] = ReLU?(sum over splits in order + bias) as bf16, 8 channels per thread
__global__ void __launch_bounds__(256) conv_fwd_reduce_kernel(const float* __restrict__ part, int splits, int M,
                                                              int co, const float* __restrict__ bias, int relu,
                                                              bf16* __restrict__ y) {
  const int cg = co / 8;
  const size_t total = (size_t)M * cg, plane = (size_t)M * co;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int o0 = (int)(e % cg) * 8;
    const size_t off = (e / cg) * co + o0;
    float acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.f;
    for (int s = 0; s < splits; ++s) {
      const float4 a = __ldcs((const float4*)(part + s * plane + off)), b = __ldcs((const float4*)(part + s * plane + off) + 1);
      acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
      acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
    }
    __align__(16) bf16 out[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float t = acc[u] + bias[o0 + u];
      if (relu) t = t > 0.f ? t : 0.f;
      out[u] = __float2bfloat16_rn(t);
    }
    *(uint4*)(y + off) = *(const uint4*)out;
  }
}

// Split count of a conv forward: 1 when its tiles fill at least half the GPU; else enough
// splits for about one wave, each keeping >= 8 K blocks (the partials cost 4 B per output
// per split, so long-K, small-M layers gain the most: late layers on small maps)
inline int conv_fwd_splits(const ConvGeom& g, int num_sms) {
  static const int off = [] {
    const char* e = getenv("CE_CONV_FWD_SPLITK");
    return e && e[0] == '0';
  }();
  const int M = g.n * g.oh * g.ow, K = g.k * g.k * g.c;
  const int m_tiles = (M + TC_BM - 1) / TC_BM, nkb = (K + TC_BK - 1) / TC_BK;
  const int tiles = m_tiles * ((g.co + 255) / 256);
  if (off || 2 * tiles >= num_sms || nkb < 16) return 1;
  int s = num_sms / tiles;
  s = std::min(s, nkb / 8);
  s = std::min(s, 16);
  return s < 2 ? 1 : s;
}
inline size_t conv_fwd_ws_bytes(const ConvGeom& g, int num_sms) {
  const int s = conv_fwd_splits(g, num_sms);
  return s > 1 ? (size_t)s * g.n * g.oh * g.ow * g.co * 4 : 0;
}

// ws / ws_bytes: split-K partials for sub-wave layers (nullptr: never split)
inline int conv_fwd_tc(const ConvGeom& g, const bf16* x, const bf16* w, const float* bias, int relu, bf16* y,
                       int num_sms, cudaStream_t st, float* ws = nullptr, size_t ws_bytes = 0) {
  const int M = g.n * g.oh * g.ow, K = g.k * g.k * g.c;
  if ((K / 8) * 4 > TC_TABLE_BYTES) return fail(CE_EINVAL, "conv_fwd_tc: K=%d exceeds the chunk table", K);
  int splits = ws ? conv_fwd_splits(g, num_sms) : 1;
  if (splits > 1 && (size_t)splits * M * g.co * 4 > ws_bytes) splits = 1;
  auto launch = [&](auto bn, const auto& ep, int nsplit) {
    constexpr int BN = decltype(bn)::value;
    TcShape sh = tc_make_shape(M, g.co, K, BN, nsplit);
    const bool tma = !tma_disabled();
    auto fill = [&](auto& ld) {
      ld.x = x; ld.w = w; ld.g = g; ld.K = K; ld.M = M; ld.BN = BN;
      ld.d_ow = FastDiv(g.ow); ld.d_oh = FastDiv(g.oh);
      ld.d_cpb = FastDiv((uint32_t)std::max(1, g.c / 64)); ld.d_k = FastDiv(g.k);
    };
    FwdTcLoader<2> ld2{};
    FwdTcLoader<3> ld3{};
    FwdTcLoader<1> ld1{};
    if (tma && g.c % 64 == 0 && !im2col_disabled() && make_tmap_kmajor(&ld2.wmap, w, g.co, K, BN) &&
        make_tmap_im2col(&ld2.xmap, x, g, TC_BM)) {
      fill(ld2);
      return tc_launch<BN>(ld2, ep, sh, num_sms, st);
    }
    if (tma && im2col32_ok(g)) {
      FwdTcLoader32 ld32{};
      if (make_tmap_kmajor(&ld32.wmap, w, g.co, K, BN) && make_tmap_im2col(&ld32.xmap, x, g, TC_BM, 32)) {
        ld32.g = g; ld32.K = K; ld32.M = M; ld32.BN = BN;
        ld32.d_ow = FastDiv(g.ow); ld32.d_oh = FastDiv(g.oh); ld32.d_c = FastDiv(g.c); ld32.d_k = FastDiv(g.k);
        return tc_launch<BN>(ld32, ep, sh, num_sms, st);
      }
    }
    if (tma && narrow_im2col_enabled() && make_tmap_kmajor(&ld3.wmap, w, g.co, K, BN) &&
        make_tmap_im2col(&ld3.xmap, x, g, TC_BM, 8)) {
      fill(ld3);
      return tc_launch<BN>(ld3, ep, sh, num_sms, st);
    }
    if (tma && make_tmap_kmajor(&ld1.wmap, w, g.co, K, BN)) {
      fill(ld1);
      return tc_launch<BN>(ld1, ep, sh, num_sms, st);
    }
    FwdTcLoader<0> ld{};
    fill(ld);
    return tc_launch<BN>(ld, ep, sh, num_sms, st);
  };
  if (splits > 1) {  // sub-wave layer: split-K partials, then bias + ReLU + bf16 in one pass
    return with_bn(g.co, [&](auto bn) {
      cudaError_t e = launch(bn, FwdPartialEpi{ws, M, g.co}, splits);
      if (e != cudaSuccess) return fail(CE_ECUDA, "conv_fwd_tc split-K: %s", cudaGetErrorString(e));
      conv_fwd_reduce_kernel<<<grid_for((size_t)M * (g.co / 8)), 256, 0, st>>>(ws, splits, M, g.co, bias, relu, y);
      e = cudaGetLastError();
      return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_fwd_reduce: %s", cudaGetErrorString(e));
    });
  }
  if (pixel_blocks_enabled() && g.s == 1 && g.c % 64 == 0 && !tma_disabled() && !im2col_disabled()) {
    // stride 1: pixel-block tiles, tiled TMA boxes (CTA pairs when wide and large enough)
    const PixelBlocks pbk = make_pixel_blocks(g.n, g.oh, g.ow);
    const int tiles = pixel_block_tiles(pbk);
    const bool pair = conv_pair_enabled() && conv_pair_shape_ok((long long)tiles * TC_BM, g.co, num_sms);
    auto go = [&](auto bnc, auto pairc) -> int {
      constexpr int BN = decltype(bnc)::value;
      constexpr bool P = decltype(pairc)::value;
      FwdBlockLoader<P> ld{};
      if (!make_tmap_kmajor(&ld.wmap, w, g.co, K, P ? BN / 2 : BN) ||
          !make_tmap_blocks(&ld.xmap, x, g.n, g.h, g.w, g.c, pbk.bh, 1 << pbk.bw_log2))
        return -1;
      ld.pb = pbk; ld.cin = g.c; ld.k = g.k; ld.BN = BN;
      ld.d_cpb = FastDiv(g.c / 64); ld.d_k = FastDiv(g.k);
      FwdTcEpi ep{y, bias, M, g.co, relu};
      ep.pb = pbk;
      TcShape sh = tc_make_shape(tiles * TC_BM, g.co, K, BN, 1);
      cudaError_t e;
      if constexpr (P) {
        sh.m_tiles = (tiles + 1) / 2;
        e = tc_launch_pair<BN>(ld, ep, sh, num_sms, st);
      } else {
        e = tc_launch<BN>(ld, ep, sh, num_sms, st);
      }
      return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_fwd_tc blocks: %s", cudaGetErrorString(e));
    };
    int r;
    if (pair) {
      const int bn = pick_bn_pair((tiles + 1) / 2, g.co, num_sms);
      r = bn == 256 ? go(std::integral_constant<int, 256>(), std::true_type())
                    : go(std::integral_constant<int, 128>(), std::true_type());
    } else {
      r = with_bn(pick_bn(tiles, g.co, num_sms), [&](auto bn) { return go(bn, std::false_type()); });
    }
    if (r >= 0) return r;
  }
  if (conv_pair_ok(g, num_sms)) {  // CTA-pair M=256 tiles over the im2col TMA path
    const int bn = pick_bn_pair((M + 2 * TC_BM - 1) / (2 * TC_BM), g.co, num_sms);
    auto go = [&](auto bnc) -> int {
      constexpr int BN = decltype(bnc)::value;
      FwdTcLoaderPair ld{};
      if (!make_tmap_kmajor(&ld.wmap, w, g.co, K, BN / 2) || !make_tmap_im2col(&ld.xmap, x, g, TC_BM)) return -1;
      ld.g = g; ld.K = K; ld.M = M; ld.BN = BN;
      ld.d_ow = FastDiv(g.ow); ld.d_oh = FastDiv(g.oh);
      ld.d_cpb = FastDiv(g.c / 64); ld.d_k = FastDiv(g.k);
      TcShape sh = tc_make_shape(M, g.co, K, BN, 1);
      sh.m_tiles = (M + 2 * TC_BM - 1) / (2 * TC_BM);
      cudaError_t e = tc_launch_pair<BN>(ld, FwdTcEpi{y, bias, M, g.co, relu}, sh, num_sms, st);
      return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_fwd_tc pair: %s", cudaGetErrorString(e));
    };
    const int r = bn == 256 ? go(std::integral_constant<int, 256>()) : go(std::integral_constant<int, 128>());
    if (r >= 0) return r;
  }
  return with_bn(pick_bn((M + TC_BM - 1) / TC_BM, g.co, num_sms), [&](auto bn) {
    cudaError_t e = launch(bn, FwdTcEpi{y, bias, M, g.co, relu}, 1);
    return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_fwd_tc: %s", cudaGetErrorString(e));
  });
}

// Conv forward + non-overlapping max-pool in one kernel (window-major rows,
// FwdPoolEpi): y / arg are the POOLED map [n][PH][PW][co] and its argmax.
// Sub-wave conv + pool: the split-K partials of the window-major rows are summed in
// split order, biased, ReLU'd and rounded to bf16 exactly as FwdPoolEpi does, then
// pooled with its first-max rule (one thread per window x 8 channels).
template <int KK>
__global__ void __launch_bounds__(256) conv_pool_reduce_kernel(const float* __restrict__ part, int splits, int rows,
                                                               int co, const float* __restrict__ bias, int relu,
                                                               PoolMap pm, bf16* __restrict__ y,
                                                               uint8_t* __restrict__ arg) {
  const int cg = co / 8;
  const size_t total = (size_t)pm.windows * cg, plane = (size_t)rows * co;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int o0 = (int)(e % cg) * 8;
    const int window = (int)(e / cg);
    const int t = window / pm.WPT, r = window - t * pm.WPT, wq = r / pm.WPW, wl = r - wq * pm.WPW;
    const int row0 = t * TC_BM + wq * 32 + wl * KK;
    float best[8];
    uint8_t bi[8];
#pragma unroll 1
    for (int tap = 0; tap < KK; ++tap) {
      const size_t off = (size_t)(row0 + tap) * co + o0;
      float acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = 0.f;
      for (int s = 0; s < splits; ++s) {
        const float4 a = __ldcs((const float4*)(part + s * plane + off));
        const float4 b = __ldcs((const float4*)(part + s * plane + off) + 1);
        acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
        acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float v = acc[u] + bias[o0 + u];
        if (relu) v = v > 0.f ? v : 0.f;
        v = __bfloat162float(__float2bfloat16_rn(v));
        if (tap == 0 || v > best[u]) {
          best[u] = v;
          bi[u] = (uint8_t)tap;
        }
      }
    }
    __align__(16) bf16 out[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      out[u] = __float2bfloat16_rn(best[u]);
      if (relu && !(best[u] > 0.f)) bi[u] = kPoolDead;
    }
    const size_t dst = (size_t)window * co + o0;
    *(uint4*)(y + dst) = *(const uint4*)out;
    *(uint2*)(arg + dst) = *(const uint2*)bi;
  }
}

inline int conv_pool_splits(const ConvGeom& g, const PoolMap& pm, int num_sms) {
  ConvGeom q = g;  // the split rule of conv_fwd_splits on the window-major row count
  const int rows = pool_rows(pm);
  q.n = 1;
  q.oh = rows;
  q.ow = 1;
  return conv_fwd_splits(q, num_sms);
}
inline size_t conv_pool_ws_bytes(const ConvGeom& g, int ps, int pst, int num_sms) {
  const PoolMap pm = make_pool_map(g.n, g.oh, g.ow, ps, pst);
  const int s = conv_pool_splits(g, pm, num_sms);
  return s > 1 ? (size_t)s * pool_rows(pm) * g.co * 4 : 0;
}

inline int conv_fwd_tc_pool(const ConvGeom& g, const bf16* x, const bf16* w, const float* bias, int relu, int ps,
                            int pst, bf16* y, uint8_t* arg, int num_sms, cudaStream_t st, float* ws = nullptr,
                            size_t ws_bytes = 0) {
  if (!pool_fusable(ps, pst)) return fail(CE_EINVAL, "pool epilogue needs a non-overlapping 2x2 or 3x3 window");
  const int K = g.k * g.k * g.c;
  if ((K / 8) * 4 > TC_TABLE_BYTES) return fail(CE_EINVAL, "conv_fwd_tc_pool: K=%d exceeds the chunk table", K);
  const PoolMap pm = make_pool_map(g.n, g.oh, g.ow, ps, pst);
  const int Mp = pool_rows(pm);
  int splits = ws ? conv_pool_splits(g, pm, num_sms) : 1;
  if (splits > 1 && (size_t)splits * Mp * g.co * 4 > ws_bytes) splits = 1;
  if (splits > 1) {  // sub-wave: split-K partials over the window-major rows, then pool in the reduce
    return with_bn(g.co, [&](auto bn) {
      constexpr int BN = decltype(bn)::value;
      TcShape sh = tc_make_shape(Mp, g.co, K, BN, splits);
      FwdPartialEpi ep{ws, Mp, g.co};
      auto fill = [&](auto& ld) {
        ld.x = x; ld.w = w; ld.g = g; ld.K = K; ld.M = Mp; ld.BN = BN; ld.pm = pm;
        ld.d_ow = FastDiv(g.ow); ld.d_oh = FastDiv(g.oh);
      };
      cudaError_t e;
      FwdTcLoader<1, true> ld1{};
      if (!tma_disabled() && make_tmap_kmajor(&ld1.wmap, w, g.co, K, BN)) {
        fill(ld1);
        e = tc_launch<BN>(ld1, ep, sh, num_sms, st);
      } else {
        FwdTcLoader<0, true> ld0{};
        fill(ld0);
        e = tc_launch<BN>(ld0, ep, sh, num_sms, st);
      }
      if (e != cudaSuccess) return fail(CE_ECUDA, "conv_fwd_tc_pool split-K: %s", cudaGetErrorString(e));
      const unsigned grid = grid_for((size_t)pm.windows * (g.co / 8));
      if (ps == 2)
        conv_pool_reduce_kernel<4><<<grid, 256, 0, st>>>(ws, splits, Mp, g.co, bias, relu, pm, y, arg);
      else
        conv_pool_reduce_kernel<9><<<grid, 256, 0, st>>>(ws, splits, Mp, g.co, bias, relu, pm, y, arg);
      e = cudaGetLastError();
      return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_pool_reduce: %s", cudaGetErrorString(e));
    });
  }
  return with_bn(pick_bn(Mp / TC_BM, g.co, num_sms), [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    return with_pool_kk(ps, [&](auto kkc) {
      constexpr int KK = decltype(kkc)::value;
      TcShape sh = tc_make_shape(Mp, g.co, K, BN, 1);
      FwdPoolEpi<KK> ep{y, arg, bias, g.co, relu, pm};
      auto fill = [&](auto& ld) {
        ld.x = x; ld.w = w; ld.g = g; ld.K = K; ld.M = Mp; ld.BN = BN; ld.pm = pm;
        ld.d_ow = FastDiv(g.ow); ld.d_oh = FastDiv(g.oh);
      };
      cudaError_t e;
      FwdTcLoader<1, true> ld1{};
      if (!tma_disabled() && make_tmap_kmajor(&ld1.wmap, w, g.co, K, BN)) {
        fill(ld1);
        e = tc_launch<BN>(ld1, ep, sh, num_sms, st);
      } else {
        FwdTcLoader<0, true> ld0{};
        fill(ld0);
        e = tc_launch<BN>(ld0, ep, sh, num_sms, st);
      }
      return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_fwd_tc_pool: %s", cudaGetErrorString(e));
    });
  });
}

// Auxiliary streams for independent launches of one layer pass (the stride^2
// dgrad classes): fork from the caller's stream with an event, join back
// with one event per branch. Per calling thread and device (a worker thread
// drives one net at a time); under graph capture the branches become
// parallel graph nodes. CE_SERIAL_CLASSES=1 keeps everything on one stream.
struct ForkStreams {
  static constexpr int N = 8;
  cudaStream_t aux[N] = {};
  cudaEvent_t done[N] = {};
  cudaEvent_t start = nullptr;
  int device = -1;
};
inline ForkStreams* fork_streams() {
  static const bool serial = [] {
    const char* e = getenv("CE_SERIAL_CLASSES");
    return e && e[0] == '1';
  }();
  if (serial) return nullptr;
  thread_local ForkStreams fs;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  if (fs.device != dev) {
    for (int i = 0; i < ForkStreams::N; ++i) {
      if (cudaStreamCreateWithFlags(&fs.aux[i], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&fs.done[i], cudaEventDisableTiming) != cudaSuccess)
        return nullptr;
    }
    if (cudaEventCreateWithFlags(&fs.start, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    fs.device = dev;
  }
  return &fs;
}

inline int conv_dgrad_tc(const ConvGeom& g, const bf16* dy, const bf16* wt, const bf16* mask, bf16* dx, int num_sms,
                         cudaStream_t st) {
  bool any_empty = false;
  for (int rh = 0; rh < g.s && rh < g.h; ++rh)
    for (int rw = 0; rw < g.s && rw < g.w; ++rw)
      if (rh >= g.k || rw >= g.k) any_empty = true;
  if (any_empty) {  // positions no tap reaches get a zero gradient (k < s)
    cudaError_t e = cudaMemsetAsync(dx, 0, (size_t)g.n * g.h * g.w * g.c * sizeof(bf16), st);
    if (e != cudaSuccess) return fail(CE_ECUDA, "conv_dgrad_tc memset: %s", cudaGetErrorString(e));
  }
  int n_cls = 0;
  for (int rh = 0; rh < g.s && rh < g.h; ++rh)
    for (int rw = 0; rw < g.s && rw < g.w; ++rw)
      if (rh < g.k && rw < g.k) ++n_cls;
  ForkStreams* fs = n_cls > 1 ? fork_streams() : nullptr;
  if (fs && cudaEventRecord(fs->start, st) != cudaSuccess) return fail(CE_ECUDA, "conv_dgrad_tc: fork");
  int ci = 0;
  const cudaStream_t home = st;
  for (int rh = 0; rh < g.s && rh < g.h; ++rh)
    for (int rw = 0; rw < g.s && rw < g.w; ++rw) {
      if (rh >= g.k || rw >= g.k) continue;
      st = (fs && ci > 0) ? fs->aux[ci - 1] : home;
      if (st != home && cudaStreamWaitEvent(st, fs->start, 0) != cudaSuccess)
        return fail(CE_ECUDA, "conv_dgrad_tc: fork wait");
      ++ci;
      DgradClass cl;
      cl.rh = rh;
      cl.rw = rw;
      cl.ti = rh < g.k ? (g.k - rh + g.s - 1) / g.s : 0;
      cl.tj = rw < g.k ? (g.k - rw + g.s - 1) / g.s : 0;
      cl.hc = (g.h - rh + g.s - 1) / g.s;
      cl.wc = (g.w - rw + g.s - 1) / g.s;
      if (cl.ti == 0 || cl.tj == 0) continue;
      const int M = g.n * cl.hc * cl.wc, K = cl.ti * cl.tj * g.co;
      if ((K / 8) * 12 > TC_TABLE_BYTES) return fail(CE_EINVAL, "conv_dgrad_tc: K=%d exceeds the chunk table", K);
      if (conv_pair_enabled() && !tma_disabled() && !im2col_disabled() && g.co % 64 == 0 &&
          conv_pair_shape_ok(M, g.c, num_sms)) {  // CTA-pair M=256 tiles
        const bf16* wcls = wt + dg_class_base(g.k, g.s, g.c, g.co, rh * g.s + rw);
        auto go = [&](auto bnc) -> int {
          constexpr int BN = decltype(bnc)::value;
          DgradTcLoaderPair ld{};
          if (!make_tmap_kmajor(&ld.wmap, wcls, g.c, K, BN / 2) || !make_tmap_im2col_dgrad(&ld.dmap, dy, g, cl))
            return -1;
          ld.g = g; ld.cl = cl; ld.K = K; ld.M = M; ld.BN = BN;
          ld.d_wc = FastDiv(cl.wc); ld.d_hc = FastDiv(cl.hc);
          ld.d_cpb = FastDiv(g.co / 64); ld.d_tj = FastDiv(cl.tj);
          TcShape sh = tc_make_shape(M, g.c, K, BN, 1);
          sh.m_tiles = (M + 2 * TC_BM - 1) / (2 * TC_BM);
          DgradTcEpi ep{dx, mask, g, cl, M, FastDiv(cl.wc), FastDiv(cl.hc)};
          cudaError_t e = tc_launch_pair<BN>(ld, ep, sh, num_sms, st);
          return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_dgrad_tc pair: %s", cudaGetErrorString(e));
        };
        const int bnp = pick_bn_pair((M + 2 * TC_BM - 1) / (2 * TC_BM), g.c, num_sms);
        const int r = bnp == 256 ? go(std::integral_constant<int, 256>()) : go(std::integral_constant<int, 128>());
        if (r > 0) return r;
        if (r == 0) continue;
      }
      int s = with_bn(pick_bn((M + TC_BM - 1) / TC_BM, g.c, num_sms), [&](auto bn) {
        constexpr int BN = decltype(bn)::value;
        TcShape sh = tc_make_shape(M, g.c, K, BN, 1);
        const bf16* wcls = wt + dg_class_base(g.k, g.s, g.c, g.co, rh * g.s + rw);
        DgradTcEpi ep{dx, mask, g, cl, M, FastDiv(cl.wc), FastDiv(cl.hc)};
        cudaError_t e;
        const bool tma = !tma_disabled();
        auto fill = [&](auto& ld) {
          ld.dy = dy; ld.wt = wcls; ld.g = g; ld.cl = cl; ld.K = K; ld.M = M; ld.BN = BN;
          ld.d_wc = FastDiv(cl.wc); ld.d_hc = FastDiv(cl.hc);
          ld.d_cpb = FastDiv((uint32_t)std::max(1, g.co / 64)); ld.d_tj = FastDiv(cl.tj);
        };
        DgradTcLoader<2> ld2{};
        DgradTcLoader<3> ld3{};
        DgradTcLoader<1> ld1{};
        if (tma && g.co % 64 == 0 && !im2col_disabled() && make_tmap_kmajor(&ld2.wmap, wcls, g.c, K, BN) &&
            make_tmap_im2col_dgrad(&ld2.dmap, dy, g, cl)) {
          fill(ld2);
          e = tc_launch<BN>(ld2, ep, sh, num_sms, st);
        } else if (tma && narrow_im2col_enabled() && make_tmap_kmajor(&ld3.wmap, wcls, g.c, K, BN) &&
                   make_tmap_im2col_dgrad(&ld3.dmap, dy, g, cl, 8)) {
          fill(ld3);
          e = tc_launch<BN>(ld3, ep, sh, num_sms, st);
        } else if (tma && make_tmap_kmajor(&ld1.wmap, wcls, g.c, K, BN)) {
          fill(ld1);
          e = tc_launch<BN>(ld1, ep, sh, num_sms, st);
        } else {
          DgradTcLoader<0> ld{};
          fill(ld);
          e = tc_launch<BN>(ld, ep, sh, num_sms, st);
        }
        return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_dgrad_tc: %s", cudaGetErrorString(e));
      });
      if (s != CE_OK) return s;
    }
  if (fs)  // join every branch back into the caller's stream
    for (int b = 1; b < ci; ++b)
      if (cudaEventRecord(fs->done[b - 1], fs->aux[b - 1]) != cudaSuccess ||
          cudaStreamWaitEvent(home, fs->done[b - 1], 0) != cudaSuccess)
        return fail(CE_ECUDA, "conv_dgrad_tc: join");
  return CE_OK;
}

inline int conv_wgrad_splits(const ConvGeom& g, int n, int num_sms) {
  // one wave: m_tiles * splits <= #SMs (a second, partial wave would double the
  // kernel time for a few CTAs), at least 4 k-blocks per split
  const int Kf = g.k * g.k * g.c;
  const long long Mo = (long long)n * g.oh * g.ow;
  const int m_tiles = (Kf + TC_BM - 1) / TC_BM;
  const long long nkb = (Mo + TC_BK - 1) / TC_BK;
  long long want = num_sms / m_tiles;
  if (want > nkb / 4) want = nkb / 4;
  if (want > 128) want = 128;
  if (want < 1) want = 1;
  if (nkb / want >= 256) {
    // long splits: wave balance outweighs the per-split fixed cost, so allow a few
    // (nearly full) waves; each extra wave is charged 4% (measured on SWEET:
    // 4 splits = 128/148 SMs 684 TF/s, 9 splits = 288/296 790 TF/s, 13 = 416/444 696 TF/s)
    double best = 0.0;
    long long pick = want;
    for (long long s = want; s <= 128 && s <= nkb / 64; ++s) {
      const long long units = (long long)m_tiles * s, waves = (units + num_sms - 1) / num_sms;
      const double score = (double)units / (double)(waves * num_sms) * (1.0 - 0.04 * (double)(waves - 1));
      if (score > best + 1e-9) best = score, pick = s;
    }
    want = pick;
  }
  static const int forced = [] {  // CE_WGRAD_SPLITS=N: measurement override
    const char* e = getenv("CE_WGRAD_SPLITS");
    return e ? atoi(e) : 0;
  }();
  if (forced > 0) want = std::min<long long>(forced, std::max<long long>(1, nkb));
  return (int)want;
}
inline int conv_wgrad_tc_max_splits(const ConvGeom& g, int n, int num_sms) { return conv_wgrad_splits(g, n, num_sms); }

inline int conv_wgrad_tc(const ConvGeom& g, const bf16* x, const bf16* dy, float* part, int* splits_out, int num_sms,
                         cudaStream_t st) {
  const int Kf = g.k * g.k * g.c, Mo = g.n * g.oh * g.ow;
  const int want = conv_wgrad_splits(g, g.n, num_sms);
  return with_bn(g.co, [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    TcShape sh = tc_make_shape(Kf, g.co, Mo, BN, want);
    *splits_out = sh.splits;
    WgradTcEpi ep{part, Kf, g.co};
    cudaError_t e;
    const bool tma = !tma_disabled() && BN >= 64;
    auto fill = [&](auto& ld) {
      ld.x = x; ld.dy = dy; ld.g = g; ld.Kf = Kf; ld.Mo = Mo; ld.BN = BN;
      ld.d_ow = FastDiv(g.ow); ld.d_oh = FastDiv(g.oh);
      ld.d_c = FastDiv(g.c); ld.d_k = FastDiv(g.k);
    };
    WgradTcLoader<2> ld2{};
    WgradTcLoader32 ld32{};
    WgradTcLoader<1> ld1{};
    if (tma && g.c % 64 == 0 && !im2col_disabled() && make_tmap_mn64(&ld2.dmap, dy, Mo, g.co) &&
        make_tmap_im2col(&ld2.xmap, x, g, TC_BK)) {
      fill(ld2);
      ld2.slab3 = BN > 64 && make_tmap_mn64_slabs(&ld2.dmap3, dy, Mo, g.co, BN / 64) ? 1 : 0;
      e = tc_launch<BN>(ld2, ep, sh, num_sms, st);
    } else if (tma && im2col32_ok(g) && make_tmap_mn64(&ld32.dmap, dy, Mo, g.co) &&
               make_tmap_im2col(&ld32.xmap, x, g, TC_BK, 32)) {
      ld32.g = g; ld32.Kf = Kf; ld32.Mo = Mo; ld32.BN = BN;
      ld32.d_ow = FastDiv(g.ow); ld32.d_oh = FastDiv(g.oh); ld32.d_c = FastDiv(g.c); ld32.d_k = FastDiv(g.k);
      ld32.slab3 = BN > 64 && make_tmap_mn64_slabs(&ld32.dmap3, dy, Mo, g.co, BN / 64) ? 1 : 0;
      e = tc_launch<BN>(ld32, ep, sh, num_sms, st);
    } else if (tma && make_tmap_mn64(&ld1.dmap, dy, Mo, g.co)) {
      fill(ld1);
      e = tc_launch<BN>(ld1, ep, sh, num_sms, st);
    } else {
      WgradTcLoader<0> ld{};
      fill(ld);
      e = tc_launch<BN>(ld, ep, sh, num_sms, st);
    }
    return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_wgrad_tc: %s", cudaGetErrorString(e));
  });
}

}  // namespace ce
