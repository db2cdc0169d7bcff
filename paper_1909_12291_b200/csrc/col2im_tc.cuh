// Small-channel stride-1 conv backward-data as GEMM + col2im (tcgen05).
//
// The implicit dgrad GEMM (conv_dgrad_tc) puts the input channel count on N;
// with few channels (C2 genome 8: 16 channels at k = 6, 64 at k = 7) N is
// 16-64, the M = 128 MMA runs at a sliver of its rate and every dY element is
// gathered k*k times. For stride 1 the same product is
//     Z[(n, p, q)][(i, j, c)] = sum_o dY[n, p, q, o] * W[o, i, j, c]   (plain GEMM)
//     dX[n, h, w, c] = sum_{i, j} Z[(n, h - i, w - j)][(i, j, c)]     (col2im gather)
// (Conv2d.backward, nn.py:112-113, taps summed in one pass): the GEMM has
// N = k*k*C_in (hundreds to thousands), A = dY read once per N tile by TMA, and
// B = the forward's bf16 weight mirror [o][i][j][c] read as an MN-major
// operand -- no extra weight layout. Z is stored bf16 through the staged
// epilogue (coalesced rows); the col2im kernel sums the k*k taps in fp32 and
// applies the ReLU mask of the layer input before the single bf16 rounding of dX.
#pragma once
#include "ops.cuh"
#include "conv_tc.cuh"

namespace ce {

inline bool col2im_dgrad_disabled() {  // CE_DISABLE_COL2IM=1: implicit dgrad everywhere (comparison)
  static const bool off = [] {
    const char* e = getenv("CE_DISABLE_COL2IM");
    return e && e[0] == '1';
  }();
  return off;
}
// stride 1, few channels, N wide enough for 64-column TMA boxes. Since the
// implicit dgrad's per-k-block cost came down (warp-converged MMA issue, two
// k-blocks per stage, FastDiv decode) it wins from 32 input channels up:
// FIXED's 32- and 64-channel layers took C1 from 404 to 322 us per step.
inline bool col2im_dgrad_eligible(const ConvGeom& g) {
  return g.s == 1 && g.c < 32 && g.k >= 2 && g.k * g.k * g.c >= 64 && !col2im_dgrad_disabled();
}

// A = dY [M][C_out] K-major (128 x 64 SW128 boxes); B = W [C_out rows (K)][k*k*C_in (N)] MN-major
struct Col2imGemmLoader {
  static constexpr int A_MN_MAJOR = 0, B_MN_MAJOR = 1;
  static constexpr bool A_TMA_SW128 = true, B_TMA_SW128 = true, PURE_TMA = true;
  CUtensorMap amap, bmap;
  int BN;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int, const uint8_t*,
                       uint64_t* full) const {
    mbar_expect_tx(full, (uint32_t)TC_BM * 128u + (uint32_t)BN * TC_BK * 2u);
    tma_load_2d(sA, &amap, kb * TC_BK, c.m0, full);
    for (int j = 0; j < BN / 64; ++j) tma_load_2d(sB + j * 8192, &bmap, c.n0 + 64 * j, kb * TC_BK, full);
  }
};

// Z[m][n] bf16, row-major [M][N] (N % 8 == 0), through the engine's staged path
struct Col2imZEpi {
  static constexpr bool STAGED_BF16 = true;
  bf16* z;
  int M, N;
  __device__ void convert(const TileCoord&, int, const float (&v)[16], uint32_t (&out)[8]) const {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      out[i] = *(const uint32_t*)&h;
    }
  }
  __device__ bf16* row_ptr(const TileCoord& c, int row, int col, int half) const {
    const int m = c.m0 + row, n = c.n0 + col + half * 8;
    return (m < M && n < N) ? z + (size_t)m * N + n : nullptr;
  }
  __device__ void store(const TileCoord&, int, int, const float (&)[16]) const {}
  __device__ void finish(int, int) const {}
};

// dX[n][h][w][c0..c0+7] = sum over taps (i, j) with 0 <= h-i < oh, 0 <= w-j < ow
// of Z[(n, h-i, w-j)][(i*k + j)*C + c0..]; gated by (mask > 0)
__global__ void __launch_bounds__(256) col2im_dgrad_kernel(const bf16* __restrict__ z, ConvGeom g,
                                                           const bf16* __restrict__ mask, bf16* __restrict__ dx) {
  const int cg = g.c / 8, N = g.k * g.k * g.c;
  const size_t total = (size_t)g.n * g.h * g.w * cg;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(e % cg) * 8;
    size_t t = e / cg;
    const int w = (int)(t % g.w);
    t /= g.w;
    const int h = (int)(t % g.h), n = (int)(t / g.h);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const int i_lo = max(0, h - g.oh + 1), i_hi = min(g.k - 1, h);
    const int j_lo = max(0, w - g.ow + 1), j_hi = min(g.k - 1, w);
    for (int i = i_lo; i <= i_hi; ++i) {
      const bf16* zr = z + ((size_t)n * g.oh + (h - i)) * g.ow * N;
      for (int j = j_lo; j <= j_hi; ++j) {
        float v[8];
        load8(zr + (size_t)(w - j) * N + (i * g.k + j) * g.c + c0, v);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += v[u];
      }
    }
    const size_t off = (((size_t)n * g.h + h) * g.w + w) * g.c + c0;
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

inline size_t col2im_dgrad_zbytes(const ConvGeom& g, int n) {
  return (size_t)n * g.oh * g.ow * g.k * g.k * g.c * 2;
}

// wbf: forward bf16 mirror [C_out][k][k][C]; z: col2im_dgrad_zbytes(g, g.n) bytes
inline int conv_dgrad_col2im(const ConvGeom& g, const bf16* dy, const bf16* wbf, const bf16* mask, bf16* dx, bf16* z,
                             int num_sms, cudaStream_t st) {
  const int M = g.n * g.oh * g.ow, N = g.k * g.k * g.c, K = g.co;
  int s = with_bn(pick_bn((M + TC_BM - 1) / TC_BM, N, num_sms) < 64 ? 64 : pick_bn((M + TC_BM - 1) / TC_BM, N, num_sms),
                  [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    if constexpr (BN < 64) {
      return fail(CE_EINVAL, "col2im dgrad needs 64-wide N tiles");
    } else {
      TcShape sh = tc_make_shape(M, N, K, BN, 1);
      Col2imGemmLoader ld{};
      ld.BN = BN;
      if (!make_tmap_kmajor(&ld.amap, dy, M, K, TC_BM) || !make_tmap_mn64(&ld.bmap, wbf, K, N))
        return fail(CE_ECUDA, "conv_dgrad_col2im: tensor map encoding failed");
      Col2imZEpi ep{z, M, N};
      cudaError_t e = tc_launch<BN>(ld, ep, sh, num_sms, st);
      return e == cudaSuccess ? CE_OK : fail(CE_ECUDA, "conv_dgrad_col2im: %s", cudaGetErrorString(e));
    }
  });
  if (s != CE_OK) return s;
  col2im_dgrad_kernel<<<grid_for((size_t)g.n * g.h * g.w * (g.c / 8)), 256, 0, st>>>(z, g, mask, dx);
  return cudaGetLastError() == cudaSuccess ? CE_OK : fail(CE_ECUDA, "col2im_dgrad_kernel launch");
}

}  // namespace ce
