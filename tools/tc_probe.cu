// Standalone probe for the tcgen05 engine: plain GEMMs with K-major and MN-major
// operand layouts checked against a CPU reference, plus a throughput sample.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1909_12291_b200/csrc tc_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "tc_engine.cuh"

using namespace ce;

// A: K-major -> stored [M][K]; MN-major -> stored [K][M]. Same for B with N.
template <int AMN, int BMN>
struct PlainLoader {
  static constexpr int A_MN_MAJOR = AMN;
  static constexpr int B_MN_MAJOR = BMN;
  static constexpr bool A_TMA_SW128 = false, B_TMA_SW128 = false, PURE_TMA = false;
  const __nv_bfloat16* A;
  const __nv_bfloat16* B;
  int M, N, K;
  int BN;
  __device__ void init(uint8_t*, int, int) const {}
  __device__ void load(const TileCoord& c, int kb, uint32_t sA, uint32_t sB, int ptid, const uint8_t*,
                       uint64_t*) const {
    const int k0 = kb * TC_BK;
    // A tile: 128 rows x 64 k = 1024 chunks
    for (int ch = ptid; ch < TC_BM * 8; ch += TC_PRODUCERS) {
      if (!AMN) {
        int r = ch % TC_BM, kc = ch / TC_BM;
        int m = c.m0 + r, k = k0 + kc * 8;
        bool ok = m < M && k < K;
        const void* src = ok ? (const void*)(A + (size_t)m * K + k) : (const void*)A;
        cp_async16(sA + kmajor_off(TC_BM, r, kc), src, ok ? 16 : 0);
      } else {
        int g = ch % (TC_BM / 8), kk = ch / (TC_BM / 8);
        int m = c.m0 + g * 8, k = k0 + kk;
        bool ok = m < M && k < K;
        const void* src = ok ? (const void*)(A + (size_t)k * M + m) : (const void*)A;
        cp_async16(sA + mnmajor_off(TC_BM, g, kk), src, ok ? 16 : 0);
      }
    }
    for (int ch = ptid; ch < BN * 8; ch += TC_PRODUCERS) {
      if (!BMN) {
        int r = ch % BN, kc = ch / BN;
        int n = c.n0 + r, k = k0 + kc * 8;
        bool ok = n < N && k < K;
        const void* src = ok ? (const void*)(B + (size_t)n * K + k) : (const void*)B;
        cp_async16(sB + kmajor_off(BN, r, kc), src, ok ? 16 : 0);
      } else {
        int g = ch % (BN / 8), kk = ch / (BN / 8);
        int n = c.n0 + g * 8, k = k0 + kk;
        bool ok = n < N && k < K;
        const void* src = ok ? (const void*)(B + (size_t)k * N + n) : (const void*)B;
        cp_async16(sB + mnmajor_off(BN, g, kk), src, ok ? 16 : 0);
      }
    }
  }
};

struct PlainEpi {
  float* D;
  int M, N, splits;
  __device__ void store(const TileCoord& c, int row, int col, const float (&v)[16]) const {
    int m = c.m0 + row;
    if (m >= M) return;
    for (int i = 0; i < 16; ++i) {
      int n = c.n0 + col + i;
      if (n < N) D[((size_t)c.split * M + m) * N + n] = v[i];
    }
  }
  __device__ void finish(int, int) const {}
};

static float bf(float x) {  // round to bf16 and back
  __nv_bfloat16 b = __float2bfloat16(x);
  return __bfloat162float(b);
}

template <int BN, int AMN, int BMN>
int run_case(int M, int N, int K, int splits, bool timeit) {
  std::vector<float> a((size_t)M * K), b((size_t)N * K);
  srand(M * 7 + N * 13 + K);
  for (auto& x : a) x = bf((rand() / (float)RAND_MAX - 0.5f));
  for (auto& x : b) x = bf((rand() / (float)RAND_MAX - 0.5f));
  std::vector<__nv_bfloat16> ha((size_t)M * K), hb((size_t)N * K);
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) ha[AMN ? (size_t)k * M + m : (size_t)m * K + k] = __float2bfloat16(a[(size_t)m * K + k]);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) hb[BMN ? (size_t)k * N + n : (size_t)n * K + k] = __float2bfloat16(b[(size_t)n * K + k]);
  __nv_bfloat16 *dA, *dB;
  float* dD;
  TcShape sh = tc_make_shape(M, N, K, BN, splits);
  cudaMalloc(&dA, ha.size() * 2);
  cudaMalloc(&dB, hb.size() * 2);
  cudaMalloc(&dD, (size_t)sh.splits * M * N * 4);
  cudaMemcpy(dA, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  PlainLoader<AMN, BMN> ld{dA, dB, M, N, K, BN};
  PlainEpi ep{dD, M, N, sh.splits};
  int sms = 148;
  cudaError_t e = tc_launch<BN>(ld, ep, sh, sms, 0);
  cudaError_t e2 = cudaDeviceSynchronize();
  if (e != cudaSuccess || e2 != cudaSuccess) {
    printf("launch error %s / %s\n", cudaGetErrorString(e), cudaGetErrorString(e2));
    return 1;
  }
  std::vector<float> d((size_t)sh.splits * M * N);
  cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost);
  // check (sum splits); sample rows for big cases
  double num = 0, den = 0;
  int step = M > 4096 ? 37 : 1;
  for (int m = 0; m < M; m += step)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)a[(size_t)m * K + k] * b[(size_t)n * K + k];
      double got = 0;
      for (int s = 0; s < sh.splits; ++s) got += d[((size_t)s * M + m) * N + n];
      num += (got - ref) * (got - ref);
      den += ref * ref;
    }
  double rel = sqrt(num / (den + 1e-30));
  printf("case BN=%d AMN=%d BMN=%d M=%d N=%d K=%d splits=%d : rel_err=%.3e %s\n", BN, AMN, BMN, M, N, K, sh.splits, rel,
         rel < 1e-3 ? "OK" : "FAIL");
  if (timeit) {
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    for (int i = 0; i < 3; ++i) tc_launch<BN>(ld, ep, sh, sms, 0);
    cudaEventRecord(t0);
    int reps = 20;
    for (int i = 0; i < reps; ++i) tc_launch<BN>(ld, ep, sh, sms, 0);
    cudaEventRecord(t1);
    cudaEventSynchronize(t1);
    float ms;
    cudaEventElapsedTime(&ms, t0, t1);
    ms /= reps;
    double tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12;
    printf("   time %.3f ms  -> %.1f TFLOP/s\n", ms, tf);
  }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return rel < 1e-3 ? 0 : 1;
}

int main() {
  int fails = 0;
  fails += run_case<16, 0, 0>(128, 16, 64, 1, false);
  fails += run_case<64, 0, 0>(300, 50, 200, 1, false);
  fails += run_case<128, 0, 0>(1000, 128, 512, 1, false);
  fails += run_case<256, 0, 0>(1000, 256, 336, 1, false);
  fails += run_case<256, 0, 0>(777, 200, 1000, 3, false);
  fails += run_case<64, 1, 1>(256, 64, 128, 1, false);
  fails += run_case<128, 1, 1>(1000, 128, 640, 2, false);
  fails += run_case<256, 1, 0>(512, 256, 256, 1, false);
  fails += run_case<32, 0, 1>(512, 32, 256, 1, false);
  fails += run_case<256, 0, 0>(65536, 256, 4096, 1, true);
  fails += run_case<128, 0, 0>(65536, 128, 1024, 1, true);
  printf("fails=%d\n", fails);
  return fails;
}
