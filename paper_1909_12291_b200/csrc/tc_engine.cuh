// Warp-specialised tcgen05 implicit-GEMM engine (sm_100a, cta_group::1).
//
//   D[m, n] = sum_k A[m, k] * B[n, k]     (bf16 operands, fp32 accumulate in TMEM)
//
// The engine knows nothing about convolutions: a Loader policy gathers 16-byte
// chunks of A and B for one (tile, k-block) into shared memory with cp.async
// (zero-fill for padding / invalid taps), and an Epilogue policy consumes the
// fp32 accumulator rows. Roles per CTA (persistent, grid <= #SMs):
//
//   warps 0-7   producers: cp.async gather into an S-stage smem ring
//   warps 8-15  epilogue : tcgen05.ld TMEM -> registers -> Epilogue::store
//                          (warp w reads TMEM lane quarter w%4, column half (w-8)/4)
//   warp  16    MMA      : TMEM alloc + one elected thread issuing tcgen05.mma
//
// Before the role split every thread helps the Loader fill a small shared
// table (Loader::init), e.g. the im2col offset of every 16-byte K chunk, so the
// producers' inner loop is a table lookup instead of runtime divisions.
//
// Two TMEM accumulators (2 x BN columns) let the epilogue of tile t overlap the
// MMAs of tile t+1. Shared-memory tiles use the SWIZZLE_NONE canonical layouts
// (see ptx.cuh::make_sdesc): a stage holds A as [kchunk][128 rows][16 B] and B
// as [kchunk][BN rows][16 B] (K-major) or the MN-major analogue.
#pragma once
#include <type_traits>
#include "ptx.cuh"

namespace ce {

constexpr int TC_BM = 128;  // UMMA M (rows per tile = TMEM lanes)
constexpr int TC_BK = 64;   // K elements per pipeline stage (8 x 16-byte chunks)
constexpr int TC_PRODUCERS = 256;  // producer threads of gather (cp.async) loaders

// Warp roles per (Loader, Epilogue) pair: gather loaders use 8 producer warps,
// pure-TMA loaders one (a single thread issues every copy); epilogues default
// to 8 warps (2 per TMEM lane quarter) and may ask for more via Epi::EPI_WARPS.
template <class Loader>
struct ProducerWarps {
  static constexpr int value = Loader::PURE_TMA ? 1 : TC_PRODUCERS / 32;
};
template <class Epi, class = void>
struct EpiWarps {
  static constexpr int value = 8;
};
template <class Epi>
struct EpiWarps<Epi, std::void_t<decltype(Epi::EPI_WARPS)>> {
  static constexpr int value = Epi::EPI_WARPS;
};
// Epilogues writing a row-major bf16 output may set STAGED_BF16: the engine then
// converts 16 columns with epi.convert(), bounces the warp's 32 x 16 block
// through shared memory and stores it two lanes per row (full 32-byte
// sectors) instead of one 16-byte piece per row per lane.
template <class Epi, class = void>
struct EpiStaged : std::false_type {};
template <class Epi>
struct EpiStaged<Epi, std::void_t<decltype(Epi::STAGED_BF16)>> : std::bool_constant<Epi::STAGED_BF16> {};

// Epi::EPI_WARPS_TMA: epilogue warps when the loader is pure TMA (one producer warp)
template <class Epi, class = void>
struct EpiWarpsTma {
  static constexpr int value = 0;
};
template <class Epi>
struct EpiWarpsTma<Epi, std::void_t<decltype(Epi::EPI_WARPS_TMA)>> {
  static constexpr int value = Epi::EPI_WARPS_TMA;
};

// Epi::WARP_SMEM: bytes of shared-memory scratch per epilogue warp for epilogues
// that combine rows (the pooled forward); the engine then calls
// epi.store_warp(c, quarter, col, v, scratch) instead of epi.store.
template <class Epi, class = void>
struct EpiWarpSmem {
  static constexpr int value = 0;
};
template <class Epi>
struct EpiWarpSmem<Epi, std::void_t<decltype(Epi::WARP_SMEM)>> {
  static constexpr int value = Epi::WARP_SMEM;
};

// Loader::SYNC_FILL: the producers write the stage with plain shared-memory
// stores (values computed in registers, e.g. the implicit packed im2col of the
// first layer); the engine fences them to the async proxy and arrives right
// after load() instead of tracking cp.async groups.
template <class Loader, class = void>
struct SyncFill : std::false_type {};
template <class Loader>
struct SyncFill<Loader, std::void_t<decltype(Loader::SYNC_FILL)>> : std::bool_constant<Loader::SYNC_FILL> {};

// Loader::PIPE (with SYNC_FILL): the fill is split into fetch() -> registers and
// put() -> shared memory, and the producer fetches the NEXT k-block right after
// putting the current one, so its global-load round trip overlaps the wait for a
// free stage and the MMAs instead of being paid once per k-block.
template <class Loader, class = void>
struct SyncPipe : std::false_type {};
template <class Loader>
struct SyncPipe<Loader, std::void_t<decltype(Loader::PIPE)>> : std::bool_constant<Loader::PIPE> {};

// Epi::EPI_WARPS_SYNC: epilogue warps when the loader fills stages with st.shared (SyncFill)
template <class Epi, class = void>
struct EpiWarpsSync {
  static constexpr int value = 0;
};
template <class Epi>
struct EpiWarpsSync<Epi, std::void_t<decltype(Epi::EPI_WARPS_SYNC)>> {
  static constexpr int value = Epi::EPI_WARPS_SYNC;
};

// Loader::SPLIT3: fp32-accurate GEMM on the bf16 tensor cores (fp32 check mode).
// The producers store every fp32 operand value as three bf16 planes
// (v = hi + mid + lo, each the bf16 rounding of the remainder), and every K=16
// step issues the six products with a combined weight >= 2^-16:
//   lo*hi + mid*mid + hi*lo + mid*hi + hi*mid + hi*hi   (smallest first)
// accumulated in fp32 in TMEM; the dropped terms are below 2^-24 relative.
template <class Loader, class = void>
struct Split3 : std::false_type {};
template <class Loader>
struct Split3<Loader, std::void_t<decltype(Loader::SPLIT3)>> : std::bool_constant<Loader::SPLIT3> {};

// Loader::KB2: a pipeline stage holds TWO consecutive 64-deep k-blocks (pure-TMA
// loaders): one barrier round trip, arrive and commit per 128 of K. The trace
// (profiles/r02_tc_trace/) shows ~650-700 SM cycles of fixed producer / MMA-warp
// cost per stage, more than a 128 x 128 x 64 block's 256 cycles of MMA work.
template <class Loader, class = void>
struct Kb2 : std::false_type {};
template <class Loader>
struct Kb2<Loader, std::void_t<decltype(Loader::KB2)>> : std::bool_constant<Loader::KB2> {};

// Loader::A_SW64: A arrives as two 32-wide K-major SWIZZLE_64B regions per k-block
// (128 rows x 64 B each, 8 KB apart): 32-channel im2col boxes (C % 64 == 32)
template <class Loader, class = void>
struct ASw64 : std::false_type {};
template <class Loader>
struct ASw64<Loader, std::void_t<decltype(Loader::A_SW64)>> : std::bool_constant<Loader::A_SW64> {};

// Loader::A_SW64_MN: A is MN-major in 32-wide SWIZZLE_64B blocks of 64 K-rows (4 KB
// apart): 32-channel im2col patches of the wgrad (C % 64 == 32)
template <class Loader, class = void>
struct ASw64Mn : std::false_type {};
template <class Loader>
struct ASw64Mn<Loader, std::void_t<decltype(Loader::A_SW64_MN)>> : std::bool_constant<Loader::A_SW64_MN> {};

template <class Loader, class Epi>
struct TcRoles {
  static constexpr int PW = ProducerWarps<Loader>::value;
  static constexpr int EW = (Loader::PURE_TMA && EpiWarpsTma<Epi>::value)        ? EpiWarpsTma<Epi>::value
                            : (SyncFill<Loader>::value && EpiWarpsSync<Epi>::value) ? EpiWarpsSync<Epi>::value
                                                                                   : EpiWarps<Epi>::value;
  static constexpr int MMA_WARP = PW + EW;
  static constexpr int THREADS = (MMA_WARP + 1) * 32;
  static_assert(EW % 4 == 0, "epilogue warps must cover the 4 TMEM lane quarters equally");
  // shared-memory staging of the epilogue warps (STAGED_BF16: 1 KB each; WARP_SMEM scratch)
  static constexpr int EPI_STAGE = EpiStaged<Epi>::value ? EW * 1024 : EW * EpiWarpSmem<Epi>::value;
};
constexpr int TC_TABLE_BYTES = 20480;              // loader lookup tables

// Pipeline event trace (debug builds with -DCE_TC_TRACE, tools/tc_trace.py): the
// first 4 CTAs record clock64 at every producer issue, MMA full-barrier pass and
// epilogue drain, one region per role: [kind:4][tile:14][kb:14][clock:32].
#ifdef CE_TC_TRACE
__device__ unsigned long long g_tc_trace[4][3][4096];
__device__ unsigned int g_tc_trace_n[4][3];
// one recording thread per role: the index lives in a register, stores are fire-and-forget
__device__ __forceinline__ void tc_trace(unsigned int& i, int role, int kind, int tile, int kb) {
  if (blockIdx.x < 4 && i < 4096)
    g_tc_trace[blockIdx.x][role][i] = ((unsigned long long)kind << 60) | ((unsigned long long)(tile & 0x3FFF) << 46) |
                                      ((unsigned long long)(kb & 0x3FFF) << 32) | (clock64() & 0xFFFFFFFFull);
  ++i;
}
__device__ __forceinline__ void tc_trace_done(unsigned int i, int role) {
  if (blockIdx.x < 4) g_tc_trace_n[blockIdx.x][role] = i;
}
__device__ int g_tc_fake_load;  // 1: producers skip the copies (MMA / barrier rate without memory)
#define TC_TRACE(role, kind, tile, kb) tc_trace(trace_i, role, kind, tile, kb)
#define TC_TRACE_DONE(role) tc_trace_done(trace_i, role)
#else
#define TC_TRACE(role, kind, tile, kb) ((void)0)
#define TC_TRACE_DONE(role) ((void)0)
#endif
constexpr int TC_MAX_LAG = 8;


// Tile coordinates handed to loaders / epilogues.
struct TileCoord {
  int m0;     // first row of the tile
  int n0;     // first column (output channel) of the tile
  int split;  // reduction split index
  int kb0;    // first k-block of this split
  int nkb;    // number of k-blocks of this split
};

struct TcShape {
  int M, N;          // problem rows / columns
  int K;             // reduction length (elements)
  int m_tiles, n_tiles, splits;
  int kb_per_split;  // k-blocks per split (last split may have fewer)
};

__host__ __device__ inline TcShape tc_make_shape(int M, int N, int K, int BN, int splits) {
  TcShape s;
  s.M = M;
  s.N = N;
  s.K = K;
  s.m_tiles = (M + TC_BM - 1) / TC_BM;
  s.n_tiles = (N + BN - 1) / BN;
  int nkb = (K + TC_BK - 1) / TC_BK;
  if (splits < 1) splits = 1;
  if (splits > nkb) splits = nkb;
  s.kb_per_split = (nkb + splits - 1) / splits;
  s.splits = (nkb + s.kb_per_split - 1) / s.kb_per_split;
  return s;
}

__device__ inline TileCoord tc_tile(const TcShape& s, int t, int bn) {
  TileCoord c;
  int per_split = s.m_tiles * s.n_tiles;
  c.split = t / per_split;
  int r = t - c.split * per_split;
  int nt = r / s.m_tiles;
  int mt = r - nt * s.m_tiles;
  c.m0 = mt * TC_BM;
  c.n0 = nt * bn;
  int nkb = (s.K + TC_BK - 1) / TC_BK;
  c.kb0 = c.split * s.kb_per_split;
  int end = c.kb0 + s.kb_per_split;
  if (end > nkb) end = nkb;
  c.nkb = end - c.kb0;
  return c;
}

// BROWS: B rows held per CTA (BN, or BN / 2 for a CTA pair). TABLE: loader table
// bytes (pure-TMA loaders use none, which leaves that space to the ring).
template <int BN, int EPI_STAGE = 0, int PLANES = 1, int BROWS = BN, int TABLE = TC_TABLE_BYTES>
struct TcSmemLayout {
  static constexpr int A_PLANE = TC_BM * TC_BK * 2;  // 16 KB
  static constexpr int B_PLANE = BROWS * TC_BK * 2;
  static constexpr int A_BYTES = A_PLANE * PLANES;
  static constexpr int B_BYTES = B_PLANE * PLANES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // pipeline budget: 196 KB less any epilogue staging beyond the 8 KB of 8 staged warps
  static constexpr int RING = 196 * 1024 + (TC_TABLE_BYTES - TABLE) - (EPI_STAGE > 8192 ? EPI_STAGE - 8192 : 0);
  static constexpr int STAGES = (RING / STAGE_BYTES) > 8 ? 8 : (RING / STAGE_BYTES);
  static constexpr int LAG = STAGES - 1 > TC_MAX_LAG ? TC_MAX_LAG : STAGES - 1;  // cp.async groups in flight
  // SPLIT3 keeps two accumulators per buffer (hi*hi and the cross terms)
  static constexpr int ACC_COLS = (PLANES == 3 ? 2 : 1) * BN;
  static constexpr int TMEM_COLS = (2 * ACC_COLS <= 32) ? 32 : (2 * ACC_COLS <= 64) ? 64 : (2 * ACC_COLS <= 128) ? 128
                                   : (2 * ACC_COLS <= 256) ? 256 : 512;
  static constexpr int BAR_BYTES = 8 * (2 * STAGES + 4) + 16;
  static constexpr int TABLE_BYTES = TABLE;
  static constexpr int TOTAL = STAGES * STAGE_BYTES + TABLE + BAR_BYTES + EPI_STAGE + 1024;  // + slack
};

// Shared-memory layout of one (BN, Loader, Epi, PAIR) kernel: KB2 stages (two
// k-blocks) where the ring still holds >= 3 of them, i.e. <= 128 B rows per CTA
template <int BN, class Loader, class Epi, bool PAIR>
struct TcKernelLayout {
  static constexpr bool SPLIT = Split3<Loader>::value;
  static constexpr int BROWS = PAIR ? BN / 2 : BN;
  static constexpr bool KB2 = Kb2<Loader>::value && !SPLIT && Loader::PURE_TMA && BROWS <= 128;
  using type = TcSmemLayout<BN, TcRoles<Loader, Epi>::EPI_STAGE, SPLIT ? 3 : (KB2 ? 2 : 1), BROWS,
                            Loader::PURE_TMA ? 0 : TC_TABLE_BYTES>;
};

// PAIR: the CTA-pair variant (cta_group::2, launched as (2,1,1) clusters). A
// tile is 256 rows x BN; rank r of the pair loads rows m0 + 128 r of A and B
// rows n0 + r BN/2, rank 0 issues M=256 MMAs over both CTAs' shared memory and
// each CTA drains its own 128 TMEM lanes. Per SM the B operand bytes read by the
// tensor core per FLOP halve, which is what bounds BN <= 128 tiles on one SM.
// Shape: m_tiles counts 256-row tiles. Pure-TMA loaders only.
template <int BN, class Loader, class Epi, bool PAIR = false>
__global__ void __launch_bounds__(TcRoles<Loader, Epi>::THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ Loader ld, const __grid_constant__ Epi epi, const TcShape shape) {
  using R = TcRoles<Loader, Epi>;
  constexpr bool STAGED = EpiStaged<Epi>::value;
  constexpr int WSM = EpiWarpSmem<Epi>::value;
  constexpr bool SPLIT = Split3<Loader>::value;
  static_assert(!PAIR || (Loader::PURE_TMA && !SPLIT && BN >= 32), "CTA pairs: pure-TMA loaders, BN >= 32");
  using L = typename TcKernelLayout<BN, Loader, Epi, PAIR>::type;
  constexpr bool KB2 = TcKernelLayout<BN, Loader, Epi, PAIR>::KB2;
  constexpr int KPS = KB2 ? 2 : 1;  // k-blocks per stage (planes of the stage)
  constexpr int S = L::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* table = smem + S * L::STAGE_BYTES;
  uint64_t* full = (uint64_t*)(table + L::TABLE_BYTES);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_base_slot = (uint32_t*)(tempty + 2);
  uint8_t* epi_stage = table + L::TABLE_BYTES + L::BAR_BYTES;  // epilogue warp staging / scratch (16-B aligned)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int total_tiles = shape.m_tiles * shape.n_tiles * shape.splits;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
#ifdef CE_TC_TRACE
  unsigned int trace_i = 0;
#endif
  const int tile0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // first tile / stride of this CTA (pair)
  const int tstep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  auto tile_at = [&](int t) {
    TileCoord c = tc_tile(shape, t, BN);
    if (PAIR) c.m0 = c.m0 * 2 + (int)rank * TC_BM;
    return c;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], Loader::PURE_TMA ? 1 : TC_PRODUCERS);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], PAIR ? 2 * R::EW : R::EW * 32);  // pair: one arrival per epilogue warp of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == R::MMA_WARP) {
    if constexpr (PAIR)
      tmem_alloc_pair(tmem_base_slot, L::TMEM_COLS);
    else
      tmem_alloc(tmem_base_slot, L::TMEM_COLS);
  }
  ld.init(table, threadIdx.x, R::THREADS);
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // the peer's barriers exist before any copy or commit targets them
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  const uint32_t smem_base = smem_u32(smem);

  if (warp < R::PW) {
    // ------------------------------------------------------------ producers
    if (Loader::PURE_TMA && threadIdx.x != 0) goto teardown;  // one thread issues every copy
    constexpr int LAG = L::LAG;
    const int ptid = threadIdx.x;
    int stage = 0;
    uint32_t phase = 0;
    int pending_stage[TC_MAX_LAG + 1];
    int npending = 0;
    if constexpr (SyncPipe<Loader>::value) {  // register-pipelined st.shared fill
      typename Loader::Regs regs;
      int t = tile0, kb = 0;
      TileCoord c = tile_at(t < total_tiles ? t : 0);
      if (t < total_tiles) ld.fetch(c, c.kb0, ptid, table, regs);
      while (t < total_tiles) {
        if (threadIdx.x == 0) TC_TRACE(0, 1, t, kb);
        mbar_wait(&empty[stage], phase ^ 1);
        if (threadIdx.x == 0) TC_TRACE(0, 2, t, kb);
        const uint32_t sA = smem_base + stage * L::STAGE_BYTES;
        const uint32_t sB = sA + L::A_BYTES;
        ld.put(c, c.kb0 + kb, sA, sB, ptid, regs, &full[stage]);
        if (threadIdx.x == 0) TC_TRACE(0, 7, t, kb);
        fence_proxy_async();
        mbar_arrive(&full[stage]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
        if (++kb == c.nkb) {  // next k-block: this tile's, or the first of the next tile
          kb = 0;
          t += tstep;
          if (t < total_tiles) c = tile_at(t);
        }
        if (t < total_tiles) ld.fetch(c, c.kb0 + kb, ptid, table, regs);
      }
      goto producer_done;
    }
    for (int t = tile0; t < total_tiles; t += tstep) {
      TileCoord c = tile_at(t);
      for (int kb = 0; kb < c.nkb; kb += KPS) {
        if (threadIdx.x == 0) TC_TRACE(0, 1, t, kb);
        mbar_wait(&empty[stage], phase ^ 1);
        if (threadIdx.x == 0) TC_TRACE(0, 2, t, kb);
        const uint32_t sA = smem_base + stage * L::STAGE_BYTES;
        const uint32_t sB = sA + L::A_BYTES;
        if (Loader::PURE_TMA) {  // copies complete on the barrier themselves (pair: rank 0's)
#ifdef CE_TC_TRACE
          if (!g_tc_fake_load)
#endif
          {
            ld.load(c, c.kb0 + kb, sA, sB, ptid, table, &full[stage]);
            if (KB2 && kb + 1 < c.nkb)  // second k-block into the stage's second planes
              ld.load(c, c.kb0 + kb + 1, sA + L::A_PLANE, sB + L::B_PLANE, ptid, table, &full[stage]);
          }
          TC_TRACE(0, 7, t, kb);
          if (!PAIR || rank == 0) mbar_arrive(&full[stage]);
        } else if constexpr (SyncFill<Loader>::value) {  // st.shared fill: visible to the MMA after the fence
          ld.load(c, c.kb0 + kb, sA, sB, ptid, table, &full[stage]);
          fence_proxy_async();
          mbar_arrive(&full[stage]);
        } else {
          ld.load(c, c.kb0 + kb, sA, sB, ptid, table, &full[stage]);
          if (threadIdx.x == 0) TC_TRACE(0, 7, t, kb);
          cp_async_commit();
          // retire the oldest group once LAG newer ones are in flight
          if (npending == LAG) {
            cp_async_wait<LAG>();
            fence_proxy_async();
            mbar_arrive(&full[pending_stage[0]]);
#pragma unroll
            for (int i = 0; i < LAG - 1; ++i) pending_stage[i] = pending_stage[i + 1];
            --npending;
          }
          pending_stage[npending++] = stage;
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    cp_async_wait_all();
    fence_proxy_async();
    for (int i = 0; i < npending; ++i) mbar_arrive(&full[pending_stage[i]]);
  producer_done:
    if (threadIdx.x == 0) TC_TRACE_DONE(0);
  } else if (warp < R::MMA_WARP) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter (warp % 4 == q)
    const int grp = (warp - R::PW) >> 2;  // column group of this warp
    constexpr int GROUPS = R::EW / 4;
    constexpr int GCOLS = (BN / GROUPS) >= 16 ? BN / GROUPS : 16;  // multiple of 16
    const int col_begin = grp * GCOLS;
    const int col_end = col_begin + GCOLS < BN ? col_begin + GCOLS : BN;
    const int row_in_tile = q * 32 + lane;
    int lt = 0;
    for (int t = tile0; t < total_tiles; t += tstep, ++lt) {
      TileCoord c = tile_at(t);
      const int acc = lt & 1;
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      if (warp == R::PW && lane == 0) TC_TRACE(2, 5, t, 0);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * L::ACC_COLS);
      if constexpr (STAGED) {
        // software-pipelined: the TMEM load of the next chunk is in flight while this
        // one is converted, staged (XOR-swizzled halves: conflict-free both ways) and
        // stored; two named register sets, no runtime-indexed arrays
        uint4* stage = (uint4*)(epi_stage + (warp - R::PW) * 1024);
        auto emit = [&](int col, uint32_t (&r)[16]) {
          if (warp == R::PW && lane == 0) TC_TRACE(2, 9, t, col);
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
          uint32_t out[8];
          epi.convert(c, col, v, out);
          if (warp == R::PW && lane == 0) TC_TRACE(2, 10, t, col);
          const int sw = (lane >> 2) & 1;
          stage[lane * 2 + sw] = make_uint4(out[0], out[1], out[2], out[3]);
          stage[lane * 2 + (sw ^ 1)] = make_uint4(out[4], out[5], out[6], out[7]);
          __syncwarp();
#pragma unroll
          for (int it = 0; it < 2; ++it) {
            const int row = it * 16 + (lane >> 1), half = lane & 1;
            bf16* dst = epi.row_ptr(c, q * 32 + row, col, half);
            if (dst) *(uint4*)dst = stage[row * 2 + (half ^ ((row >> 2) & 1))];
          }
          __syncwarp();
          if (warp == R::PW && lane == 0) TC_TRACE(2, 11, t, col);
        };
        uint32_t ra[16], rb[16];
        if (col_begin < col_end) tmem_ld16(tbase + col_begin, ra);
#pragma unroll 1
        for (int col = col_begin; col < col_end; col += 32) {
          tmem_ld_wait();
          tmem_regs_fence(ra);
          const bool more = col + 16 < col_end;
          if (more) tmem_ld16(tbase + col + 16, rb);
          emit(col, ra);
          if (!more) break;
          tmem_ld_wait();
          tmem_regs_fence(rb);
          if (col + 32 < col_end) tmem_ld16(tbase + col + 32, ra);
          emit(col + 16, rb);
        }
      } else {
#pragma unroll 1
        for (int col = col_begin; col < col_end; col += 16) {
          uint32_t r[16];
          tmem_ld16(tbase + col, r);
          float v[16];
          if constexpr (SPLIT) {  // hi*hi + cross terms, added in IEEE fp32
            uint32_t r2[16];
            tmem_ld16(tbase + BN + col, r2);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]) + __uint_as_float(r2[i]);
          } else {
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
          }
          if constexpr (WSM > 0)
            epi.store_warp(c, q, col, v, epi_stage + (warp - R::PW) * WSM);
          else
            epi.store(c, row_in_tile, col, v);
        }
      }
      if (warp == R::PW && lane == 0) TC_TRACE(2, 6, t, 0);
      tc_fence_before();
      if constexpr (PAIR) {  // one arrival per warp on rank 0's barrier
        __syncwarp();
        if (lane == 0) {
          if (rank == 0)
            mbar_arrive(&tempty[acc]);
          else
            mbar_arrive_cluster(&tempty[acc], 0);
        }
      } else {
        mbar_arrive(&tempty[acc]);
      }
    }
    if (warp == R::PW && lane == 0) TC_TRACE_DONE(2);
    epi.finish(lane, q);
  } else if (!PAIR || rank == 0) {
    // ------------------------------------------------------------ MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    int lt = 0;
    constexpr uint32_t idesc = make_idesc_bf16(PAIR ? 2 * TC_BM : TC_BM, BN, Loader::A_MN_MAJOR, Loader::B_MN_MAJOR);
    const int k16_total = (shape.K + 15) / 16;
    for (int t = tile0; t < total_tiles; t += tstep, ++lt) {
      TileCoord c = tile_at(t);
      const int acc = lt & 1;
      if constexpr (PAIR)
        mbar_wait_cluster(&tempty[acc], ((lt >> 1) & 1) ^ 1);
      else
        mbar_wait_warp(&tempty[acc], ((lt >> 1) & 1) ^ 1);
      __syncwarp();
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * L::ACC_COLS);
      if (lane == 0) TC_TRACE(1, 4, t, 0);
      for (int kb = 0; kb < c.nkb; kb += KPS) {
        mbar_wait_warp(&full[stage], phase);
        if (lane == 0) TC_TRACE(1, 3, t, kb);
        tc_fence_after();
        const uint32_t sA = smem_base + stage * L::STAGE_BYTES;
        const uint32_t sB = sA + L::A_BYTES;
        const int gkb = c.kb0 + kb;
        int nk16 = k16_total - gkb * (TC_BK / 16);
        if (nk16 > TC_BK / 16) nk16 = TC_BK / 16;
        const bool last_stage = kb + KPS >= c.nkb;
        if constexpr (SPLIT) {
          if (lane == 0) {
#pragma unroll 1
            for (int k = 0; k < nk16; ++k) {
              // six plane products (no-swizzle canonical layouts): the five cross terms,
              // smallest first, into a second accumulator so the hi*hi chain (the large
              // one) takes a single accumulation per K=16 step; the epilogue adds the two
              constexpr int PA[6] = {2, 1, 0, 1, 0, 0}, PB[6] = {0, 1, 2, 0, 1, 0};
#pragma unroll
              for (int q = 0; q < 6; ++q) {
                const uint64_t ad =
                    make_sdesc(sA + (uint32_t)PA[q] * L::A_PLANE + (uint32_t)(2 * k) * (TC_BM * 16), TC_BM * 16, 128);
                const uint64_t bd =
                    make_sdesc(sB + (uint32_t)PB[q] * L::B_PLANE + (uint32_t)(2 * k) * (BN * 16), BN * 16, 128);
                const bool big = q == 5;
                umma_bf16(d_tmem + (big ? 0u : (uint32_t)BN), ad, bd, idesc,
                          (kb > 0 || k > 0 || (!big && q > 0)) ? 1u : 0u);
              }
            }
            umma_commit(&empty[stage]);
            if (kb == c.nkb - 1) umma_commit(&tfull[acc]);
          }
        } else {
          // warp-converged issue (umma_*_warp): descriptors at K step 0, advanced linearly.
          // K-major SW128: +32 B per K=16 step; MN-major SW128: +2 K groups (2048 B);
          // no-swizzle K-major: +2 chunk columns (2 x rows x 16 B). Descriptor address field = bytes >> 4.
          constexpr uint32_t A_STEP = ASw64Mn<Loader>::value ? 1024u
                                      : Loader::A_TMA_SW128 ? (Loader::A_MN_MAJOR ? 2048u : 32u)
                                                            : 2u * TC_BM * 16u;
          constexpr uint32_t B_STEP = Loader::B_TMA_SW128 ? (Loader::B_MN_MAJOR ? 2048u : 32u) : 2u * BN * 16u;
          // one 64-deep k-block (planes h of the stage): MMAs over its nk K=16 steps
          auto kblock = [&](int h, int kbi, int nk) {
            const uint32_t pA = sA + (uint32_t)h * L::A_PLANE, pB = sB + (uint32_t)h * L::B_PLANE;
            const uint64_t ad0 = ASw64Mn<Loader>::value ? make_sdesc_sw64_mn(pA, 64 * 64)
                                 : Loader::A_TMA_SW128
                                     ? (Loader::A_MN_MAJOR ? make_sdesc_sw128_mn(pA, 64 * 128) : make_sdesc_sw128(pA))
                                     : make_sdesc(pA, TC_BM * 16, 128);
            const uint64_t bd0 = Loader::B_TMA_SW128
                                     ? (Loader::B_MN_MAJOR ? make_sdesc_sw128_mn(pB, 64 * 128) : make_sdesc_sw128(pB))
                                     : make_sdesc(pB, BN * 16, 128);
            if constexpr (ASw64<Loader>::value) {  // A: region k/2 (8 KB apart), +32 B for odd k
#pragma unroll 1
              for (int k = 0; k < nk; ++k) {
                const uint64_t ad = make_sdesc_sw64(pA + (uint32_t)(k >> 1) * (TC_BM * 64) + (uint32_t)(k & 1) * 32);
                const uint64_t bd = bd0 + (uint64_t)((B_STEP >> 4) * (uint32_t)k);
                const uint32_t accum = (kbi > 0 || k > 0) ? 1u : 0u;
                if constexpr (PAIR)
                  umma_bf16_pair_warp(d_tmem, ad, bd, idesc, accum);
                else
                  umma_bf16_warp(d_tmem, ad, bd, idesc, accum);
              }
              (void)ad0;
            } else if (nk == TC_BK / 16) {  // full k-block: one asm block of four MMAs
              const uint32_t accum = kbi > 0 ? 1u : 0u;
              if constexpr (PAIR)
                umma4_pair_warp(d_tmem, ad0, bd0, idesc, accum, A_STEP >> 4, B_STEP >> 4);
              else
                umma4_warp(d_tmem, ad0, bd0, idesc, accum, A_STEP >> 4, B_STEP >> 4);
            } else {
#pragma unroll 1
              for (int k = 0; k < nk; ++k) {
                const uint64_t ad = ad0 + (uint64_t)((A_STEP >> 4) * (uint32_t)k);
                const uint64_t bd = bd0 + (uint64_t)((B_STEP >> 4) * (uint32_t)k);
                const uint32_t accum = (kbi > 0 || k > 0) ? 1u : 0u;
                if constexpr (PAIR)
                  umma_bf16_pair_warp(d_tmem, ad, bd, idesc, accum);
                else
                  umma_bf16_warp(d_tmem, ad, bd, idesc, accum);
              }
            }
          };
          kblock(0, kb, nk16);
          if (KB2 && kb + 1 < c.nkb) {
            int nk2 = k16_total - (gkb + 1) * (TC_BK / 16);
            if (nk2 > TC_BK / 16) nk2 = TC_BK / 16;
            kblock(1, kb + 1, nk2);
          }
          if (lane == 0) TC_TRACE(1, 8, t, kb);
          if constexpr (PAIR) {
            umma_commit_pair_warp(&empty[stage]);
            if (last_stage) umma_commit_pair_warp(&tfull[acc]);
          } else {
            umma_commit_warp(&empty[stage]);
            if (last_stage) umma_commit_warp(&tfull[acc]);
          }
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    if (lane == 0) TC_TRACE_DONE(1);
  }
teardown:
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // rank 0's last MMAs and commits target the peer
  if (warp == R::MMA_WARP) {
    tc_fence_after();
    if constexpr (PAIR)
      tmem_dealloc_pair(tmem_base, L::TMEM_COLS);
    else
      tmem_dealloc(tmem_base, L::TMEM_COLS);
  }
}

// Byte offset of a 16-byte chunk inside a stage tile with R rows.
//   K-major : chunk (row r, kchunk kc)          -> (kc * R + r) * 16
//   MN-major: chunk (MN group g, k index kk)    -> (kk/8) * R*16 + g*128 + (kk%8)*16
__device__ __forceinline__ uint32_t kmajor_off(int R, int r, int kc) { return (uint32_t)(kc * R + r) * 16u; }
__device__ __forceinline__ uint32_t mnmajor_off(int R, int g, int kk) {
  return (uint32_t)((kk >> 3) * R * 16 + g * 128 + (kk & 7) * 16);
}

template <int BN, class Loader, class Epi>
inline cudaError_t tc_launch(const Loader& ld, const Epi& epi, const TcShape& shape, int num_sms, cudaStream_t st) {
  using L = typename TcKernelLayout<BN, Loader, Epi, false>::type;
  auto kern = tc_gemm_kernel<BN, Loader, Epi>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
  if (e != cudaSuccess) return e;
  int tiles = shape.m_tiles * shape.n_tiles * shape.splits;
  int grid = tiles < num_sms ? tiles : num_sms;
  if (grid < 1) grid = 1;
  kern<<<grid, TcRoles<Loader, Epi>::THREADS, L::TOTAL, st>>>(ld, epi, shape);
  return cudaGetLastError();
}

// CTA-pair launch: (2,1,1) clusters, one pair per 256-row x BN tile, grid <= the SM count
template <int BN, class Loader, class Epi>
inline cudaError_t tc_launch_pair(const Loader& ld, const Epi& epi, const TcShape& shape, int num_sms,
                                  cudaStream_t st) {
  using L = typename TcKernelLayout<BN, Loader, Epi, true>::type;
  auto kern = tc_gemm_kernel<BN, Loader, Epi, true>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
  if (e != cudaSuccess) return e;
  const int tiles = shape.m_tiles * shape.n_tiles * shape.splits;
  int pairs = tiles < num_sms / 2 ? tiles : num_sms / 2;
  if (pairs < 1) pairs = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs, 1, 1);
  cfg.blockDim = dim3(TcRoles<Loader, Epi>::THREADS, 1, 1);
  cfg.dynamicSmemBytes = L::TOTAL;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, ld, epi, shape);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace ce
