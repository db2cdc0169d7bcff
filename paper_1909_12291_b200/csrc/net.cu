// Candidate runtime behind the C ABI (include/menndl_sm100.h).
//
// A ce_net is one instantiated genome on one device: parameters (fp32 master
// weights + momentum, bf16 mirrors for the tensor-core path), per-layer
// activations for backward, ping-pong gradient buffers and a split-K
// workspace. ce_train captures one training step (gather -> forward -> xent ->
// backward + fused SGD) into a CUDA graph and replays it; a device step counter
// selects the permutation slice and loss slot, so the whole budget runs without
// host round trips (evaluator.py:160-170 in one call).
#include <cstdarg>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cmath>
#include <atomic>
#include <condition_variable>
#include <map>
#include <mutex>
#include <nvtx3/nvToolsExt.h>
#include "ops.cuh"
#include "conv_tc.cuh"
#include "dense_tc.cuh"
#include "dense_simt.cuh"
#include "first_layer_tc.cuh"
#include "head.cuh"
#include "col2im_tc.cuh"
#include "init.cuh"

namespace ce {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

struct Layer {
  int kind = 0, relu = 0;
  ConvGeom g{};          // conv / pool geometry (n set per launch)
  int c_real = 0;        // real channels of the input (first layer: 3 of 8 stored)
  int out_c_store = 0, out_c_real = 0;
  int in_units = 0, out_units = 0;  // dense (in_units = stored flat width)
  int hw_in = 0;         // dense after features: h*w of the flattened input
  bool in_is_act = true; // dense: input is a T activation (features / image), else fp32 dense output
  bool need_dx = false, mask_in = false;
  int pidx = -1;
  float *W = nullptr, *b = nullptr, *VW = nullptr, *Vb = nullptr, *GW = nullptr, *Gb = nullptr;
  bf16 *Wbf = nullptr, *Wtbf = nullptr;
  bool head = false;      // final Dense with <= kHeadMaxOut outputs: fused forward+loss / backward (head.cuh)
  bool packed = false;    // conv over channel-padded input without dX: packed im2col GEMMs (first_layer_tc.cuh)
  bool pool_fused = false;  // conv: the next (non-overlapping) max-pool runs in this conv's epilogue, the
                            // pre-pool activation is never materialised (conv_tc.cuh FwdPoolEpi)
  bool fused = false;       // pool: its forward is done by the previous conv
  bool col2im = false;    // stride-1 few-channel dgrad as GEMM + col2im (col2im_tc.cuh)
  int Kp = 0;             // packed: im2col row width
  bf16* Wp = nullptr;     // packed (bf16 mode): bf16 mirror [co][Kp]
  float* Wpf = nullptr;   // packed (fp32 check mode): fp32 mirror [co][Kp]
  void* xcol = nullptr;   // packed: im2col matrix [B*oh*ow][Kp] (activation type) of the last forward
  bf16* Wbp = nullptr;    // dense: bf16 mirror [out][in_pad]
  bf16* x16 = nullptr;    // dense after dense: bf16 copy of the fp32 input [B][in_pad]
  int in_pad = 0, out_pad = 0;
  size_t wn = 0;
  int bn = 0;
  void* out = nullptr;
  uint8_t* arg = nullptr;
  size_t out_per_sample = 0;  // elements
};

}  // namespace ce

using namespace ce;

struct ce_dataset {
  int device = 0;
  uint8_t* pix = nullptr;
  uint8_t* lab = nullptr;
  int n = 0, c = 0, h = 0, w = 0;
};

// Per-kernel-class profiling (bench.py roofline): when enabled, ce_train runs
// its steps eagerly and brackets every launch of a class with CUDA events on
// the launching stream; durations, algorithmic FLOPs and bytes accumulate.
enum ProfClass { P_CONV_FWD = 0, P_CONV_DGRAD, P_CONV_WGRAD, P_CONV_SGD, P_DENSE_FWD, P_DENSE_BWD, P_POOL,
                 P_LOSS, P_GATHER, P_NCLASS };
static const char* kProfNames[P_NCLASS] = {"conv_fwd", "conv_dgrad", "conv_wgrad", "conv_sgd", "dense_fwd",
                                           "dense_bwd", "pool", "loss", "gather"};
struct ProfEvent {
  int cls, layer;
  double flops, bytes;
  cudaEvent_t a, b;
};
struct ProfTotals {
  long long launches = 0;
  double ms = 0, flops = 0, bytes = 0;
  double ideal_ms = 0;  // sum over launches of max(flops / P, bytes / BW): SURVEY §8(d) roofline time
};
static std::atomic<long long> g_launches{0};
// roofline peaks for ideal_ms (ce_prof_set_peaks): sustained bf16 FLOP/s and HBM B/s
static double g_peak_flops = 1.3877e15, g_peak_bytes = 6.5504e12;

struct ce_net {
  int device = 0, prec = CE_PREC_BF16, num_sms = 148;
  bool prof_on = false;
  bool prof_in_train = false;  // NVTX class ranges only around ce_train's own steps (what prof_collect counts)
  bool prof_capturing = false;  // Prof events become event-record nodes of the captured step graph
  std::vector<ProfEvent> prof_pending;
  ProfTotals prof[P_NCLASS];
  std::map<std::pair<int, int>, ProfTotals> prof_layers;  // (layer, class) -> totals; layer -1 = gather / loss
  int prof_layer_cur = -1;                                 // layer being enqueued (set by the layer loops)
  long long acc = 0;  // kernels enqueued since the last reset
  cudaStream_t st = nullptr;
  int in_c = 3, in_cp = 8, in_h = 100, in_w = 100, max_batch = 0, classes = 2;
  std::vector<Layer> L;
  std::vector<int> params;
  void* x0 = nullptr;
  int32_t* ybatch = nullptr;
  void* gbuf[2] = {nullptr, nullptr};
  bf16* gbf = nullptr;  // bf16 copy of a dense output gradient [B][out_pad]
  size_t gbytes = 0;
  float* ws = nullptr;
  bf16* zbuf = nullptr;  // col2im dgrad: Z [pixels][k*k*C] of the largest eligible layer
  size_t ws_bytes = 0;
  int* d_step = nullptr;   // [0] step counter, [1] non-finite flag
  int* h_flags = nullptr;  // pinned: non-finite flag snapshots of in-flight chunks
  float* d_losses = nullptr;
  int losses_cap = 0;
  int32_t* d_perm = nullptr;
  size_t perm_cap = 0;
  double* d_scores = nullptr;
  int64_t* d_preds = nullptr;
  size_t pred_cap = 0;
  float* d_xhost = nullptr;
  size_t xhost_cap = 0;
  std::vector<void*> allocs;
  size_t bytes = 0;
  bool keep_grads = false;
  bool use_tc = false;
};

namespace {

int dev_alloc(ce_net* net, void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~(size_t)255;
  cudaError_t e = cudaMallocAsync(p, bytes, net->st);
  if (e == cudaErrorMemoryAllocation) {
    // the pool keeps freed memory cached (keep_pool_memory): after a giant
    // candidate it can be held in blocks of the wrong size, so hand the unused
    // part back to the driver and retry once before reporting OOM
    cudaGetLastError();
    int dev = 0;
    cudaMemPool_t pool;
    cudaStreamSynchronize(net->st);
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
      cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(p, bytes, net->st);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CE_ENOMEM, "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
  }
  net->allocs.push_back(*p);
  net->bytes += bytes;
  return CE_OK;
}
// stream-ordered free of a buffer the net outgrew (it leaves the net's alloc list)
void release_alloc(ce_net* net, void* p) {
  if (!p) return;
  auto it = std::find(net->allocs.begin(), net->allocs.end(), p);
  if (it == net->allocs.end()) return;
  net->allocs.erase(it);
  cudaFreeAsync(p, net->st);
}
#define ALLOC(ptr, bytes)                                             \
  do {                                                                \
    int s_ = dev_alloc(net, (void**)&(ptr), (bytes));                 \
    if (s_ != CE_OK) return s_;                                       \
  } while (0)

// Per-device execution gate (latency is measured in an
// exclusive per-GPU window). Candidate work on a device -- each ce_train replay
// chunk, predict, forward, parameter upload -- holds the gate shared and
// releases it only after that work has completed (or, for the train loop,
// with at most one chunk in flight, which ce_latency drains with a device
// synchronize). ce_latency holds it exclusively; a waiting measurement blocks
// new shared entries (writer preference), so it waits at most one chunk per
// concurrent slot. Only the library's own entry points take the gate; it is
// never taken twice on one thread.
struct DeviceGate {
  std::mutex m;
  std::condition_variable cv;
  int readers = 0, writers_waiting = 0;
  bool writer = false;
  void lock_shared() {
    std::unique_lock<std::mutex> l(m);
    cv.wait(l, [&] { return !writer && writers_waiting == 0; });
    ++readers;
  }
  void unlock_shared() {
    std::lock_guard<std::mutex> l(m);
    if (--readers == 0) cv.notify_all();
  }
  void lock() {
    std::unique_lock<std::mutex> l(m);
    ++writers_waiting;
    cv.wait(l, [&] { return !writer && readers == 0; });
    --writers_waiting;
    writer = true;
  }
  void unlock() {
    std::lock_guard<std::mutex> l(m);
    writer = false;
    cv.notify_all();
  }
};
constexpr int kMaxDevices = 64;
DeviceGate g_gates[kMaxDevices];
struct SharedGate {
  DeviceGate* g;
  explicit SharedGate(int dev) : g(dev >= 0 && dev < kMaxDevices ? &g_gates[dev] : nullptr) {
    if (g) g->lock_shared();
  }
  ~SharedGate() { release(); }
  void release() {
    if (g) g->unlock_shared();
    g = nullptr;
  }
};
struct ExclusiveGate {
  DeviceGate* g;
  explicit ExclusiveGate(int dev) : g(dev >= 0 && dev < kMaxDevices ? &g_gates[dev] : nullptr) {
    if (g) g->lock();
  }
  ~ExclusiveGate() {
    if (g) g->unlock();
  }
};

// How host threads wait on the device (CE_HOST_SYNC=spin|yield|blocking; unset
// keeps the driver default, which spins while a process has one context). One
// process per GPU with several slot threads each spinning in
// cudaEventSynchronize can oversubscribe the host cores at N GPUs; blocking
// sync parks the waiting threads instead. Applied once per device.
static void apply_host_sync(int d) {
  static std::atomic<unsigned long long> done{0};
  if (d < 0 || d >= 64 || (done.load() >> d) & 1ull) return;
  done.fetch_or(1ull << d);
  const char* e = getenv("CE_HOST_SYNC");
  if (!e || !e[0]) return;
  unsigned flag = !strcmp(e, "blocking") ? cudaDeviceScheduleBlockingSync
                  : !strcmp(e, "yield")  ? cudaDeviceScheduleYield
                  : !strcmp(e, "spin")   ? cudaDeviceScheduleSpin
                                         : cudaDeviceScheduleAuto;
  unsigned cur = 0;
  cudaGetDeviceFlags(&cur);
  cudaSetDeviceFlags((cur & ~cudaDeviceScheduleMask) | flag);
  cudaGetLastError();
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
    apply_host_sync(d);
  }
  ~DevGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline size_t act_bytes(const ce_net* net) { return net->prec == CE_PREC_FP32 ? 4 : 2; }

// Two pinned ints per ce_train call for the non-finite flag snapshots, carved
// from one process-wide pinned block (cudaHostAlloc per net costs milliseconds).
int* pinned_flag_slots() {
  static std::atomic<unsigned> next{0};
  static int* block = nullptr;
  static std::atomic<int> ready{0};
  constexpr unsigned kSlots = 4096;
  if (!ready.load()) {
    static std::atomic_flag lock = ATOMIC_FLAG_INIT;
    while (lock.test_and_set()) {
    }
    if (!ready.load()) {
      if (cudaHostAlloc((void**)&block, kSlots * 2 * sizeof(int), cudaHostAllocPortable) != cudaSuccess) block = nullptr;
      ready.store(1);
    }
    lock.clear();
  }
  if (!block) return nullptr;
  return block + 2 * (next.fetch_add(1) % kSlots);
}

// The stream-ordered pool returns freed memory to the OS at every sync by
// default; candidates come and go every few ms, so keep it cached instead.
void keep_pool_memory(int device) {
  static std::atomic<unsigned> done{0};
  if (device < 0 || device >= 32 || (done.fetch_or(1u << device) & (1u << device))) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

// CE_PROF_NVTX=1: the profiling pass runs eagerly and each class bracket is also
// an NVTX push/pop range named after the class, so `ncu --nvtx --nvtx-include
// dense_bwd/` measures DRAM bytes on exactly the launches the events time.
static bool prof_nvtx() {
  static const bool on = [] { const char* e = getenv("CE_PROF_NVTX"); return e && e[0] == '1'; }();
  return on;
}

struct Prof {
  ce_net* net;
  int cls;
  double flops, bytes;
  int kernels, layer;
  cudaEvent_t a = nullptr;
  Prof(ce_net* n, int c, double f, double b, int k = 1)
      : net(n), cls(c), flops(f), bytes(b), kernels(k), layer(n->prof_layer_cur) {
    net->acc += k;
    if (net->prof_on) {
      cudaEventCreate(&a);
      cudaEventRecordWithFlags(a, net->st, net->prof_capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
      if (prof_nvtx() && net->prof_in_train) nvtxRangePushA(kProfNames[cls]);
    }
  }
  ~Prof() {
    if (net->prof_on) {
      cudaEvent_t b;
      cudaEventCreate(&b);
      cudaEventRecordWithFlags(b, net->st, net->prof_capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
      net->prof_pending.push_back(ProfEvent{cls, layer, flops, bytes, a, b});
      if (prof_nvtx() && net->prof_in_train) nvtxRangePop();
    }
  }
};

void prof_release(ce_net* net) {
  for (auto& e : net->prof_pending) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  net->prof_pending.clear();
}

// Accumulate the bracketed launches. keep: the events belong to a captured step
// graph and are re-recorded by its next replay (read after every replay).
void prof_collect(ce_net* net, bool keep = false) {
  for (auto& e : net->prof_pending) {
    float ms = 0.f;
    cudaEventSynchronize(e.b);
    cudaEventElapsedTime(&ms, e.a, e.b);
    const double ideal = 1e3 * std::max(e.flops / g_peak_flops, e.bytes / g_peak_bytes);
    for (ProfTotals* t : {&net->prof[e.cls], &net->prof_layers[{e.layer, e.cls}]}) {
      t->launches += 1;
      t->ms += ms;
      t->flops += e.flops;
      t->bytes += e.bytes;
      t->ideal_ms += ideal;
    }
  }
  if (!keep) prof_release(net);
}

// CE_POOL_FUSION: 0 = never fuse max-pool into the conv epilogue, 1 = only where
// the conv runs the gather loader anyway (packed first layer, C % 64 != 0; default),
// 2 = every non-overlapping pool after a conv. The window-major row order needs the
// gather loader, which is slower than the TMA im2col loader on C % 64 == 0 layers:
// with mode 2 VGG16STYLE inference (three such pools) fell from 126k to 79k patches/s.
int pool_fusion_mode() {
  static const int mode = [] {
    const char* e = getenv("CE_POOL_FUSION");
    return e ? atoi(e) : 1;
  }();
  return mode;
}

PoolMap layer_pool_map(const ce_net* net, size_t conv_li, int n) {
  const Layer& cv = net->L[conv_li];
  const Layer& pl = net->L[conv_li + 1];
  return make_pool_map(n, cv.g.oh, cv.g.ow, pl.g.k, pl.g.s);
}

int pick_splits(long long blocks_per_split, long long K, long long min_chunk, int num_sms, int waves = 2,
                int max_splits = 64) {
  long long want = ((long long)waves * num_sms + blocks_per_split - 1) / blocks_per_split;
  long long cap = K / min_chunk;
  if (want > cap) want = cap;
  if (want > max_splits) want = max_splits;
  if (want < 1) want = 1;
  return (int)want;
}

// ----------------------------------------------------------------------------- forward
// loss = true (training): a fused head also computes the loss and dL/dlogits
// into gbuf[0] and sets *loss_fused.
template <class T>
int enqueue_forward(ce_net* net, int n, bool loss = false, bool* loss_fused = nullptr) {
  bool fused_dummy = false;
  if (!loss_fused) loss_fused = &fused_dummy;
  cudaStream_t st = net->st;
  const void* in = net->x0;
  bool in_act = true;
  for (size_t li = 0; li < net->L.size(); ++li) {
    Layer& l = net->L[li];
    net->prof_layer_cur = (int)li;
    if (l.kind == CE_LAYER_CONV && l.pool_fused) {  // conv + max-pool in one GEMM epilogue
      ConvGeom g = l.g;
      g.n = n;
      Layer& pl = net->L[li + 1];
      const PoolMap pm = layer_pool_map(net, li, n);
      const int K = g.k * g.k * g.c;
      const double ab = (double)act_bytes(net), pooled = (double)pm.windows * g.co;
      Prof pf(net, P_CONV_FWD, 2.0 * pm.windows * pm.KK * g.co * g.k * g.k * l.c_real,
              ab * ((double)n * g.h * g.w * g.c + pooled + (double)g.co * K) + pooled + 4.0 * g.co, l.packed ? 2 : 1);
      if (l.packed) {  // implicit packed operand: no im2col matrix in HBM
        int s = conv_fwd_packed_implicit(g, (const bf16*)in, l.c_real, l.Kp, l.Wp, l.b, l.relu, &pm, (bf16*)pl.out,
                                         pl.arg, net->num_sms, st);
        if (s != CE_OK) return s;
      } else {
        int s = conv_fwd_tc_pool(g, (const bf16*)in, l.Wbf, l.b, l.relu, pl.g.k, pl.g.s, (bf16*)pl.out, pl.arg,
                                 net->num_sms, st, net->ws, net->ws_bytes);
        if (s != CE_OK) return s;
      }
      CE_CHECK_LAUNCH();
      in = pl.out;
      in_act = true;
      ++li;  // the pool layer is done
      continue;
    }
    if (l.kind == CE_LAYER_CONV) {
      ConvGeom g = l.g;
      g.n = n;
      const int M = n * g.oh * g.ow, K = g.k * g.k * g.c;
      const double ab = (double)act_bytes(net);
      Prof pf(net, P_CONV_FWD, 2.0 * M * g.co * g.k * g.k * l.c_real,
              ab * ((double)n * g.h * g.w * g.c + (double)M * g.co + (double)g.co * K) + 4.0 * g.co);
      if (l.packed) {
        if (net->use_tc) {  // implicit packed operand: no im2col matrix in HBM
          int s = conv_fwd_packed_implicit(g, (const bf16*)in, l.c_real, l.Kp, l.Wp, l.b, l.relu, nullptr,
                                           (bf16*)l.out, nullptr, net->num_sms, st);
          if (s != CE_OK) return s;
        } else {  // fp32 check mode: explicit im2col + CUDA-core GEMM
          launch_im2col_packed((const T*)in, g, l.c_real, l.Kp, (T*)l.xcol, st);
          CE_CHECK_LAUNCH();
          conv_fwd_packed_simt(g, (const float*)l.xcol, l.Kp, l.Wpf, l.b, l.relu, (float*)l.out, st);
        }
      } else if (net->use_tc) {
        int s = conv_fwd_tc(g, (const bf16*)in, l.Wbf, l.b, l.relu, (bf16*)l.out, net->num_sms, st, net->ws,
                            net->ws_bytes);
        if (s != CE_OK) return s;
      } else {
        simt_gemm(make_fwd_a((const T*)in, g), FwdB{l.W, K}, FwdEpi<T>{(T*)l.out, l.b, g.co, l.relu != 0}, M, g.co, K,
                  1, st);
      }
    } else if (l.kind == CE_LAYER_POOL) {
      ConvGeom g = l.g;
      g.n = n;
      size_t total = (size_t)n * g.oh * g.ow * g.c;
      Prof pf(net, P_POOL, 0.0, (double)act_bytes(net) * ((double)n * g.h * g.w * g.c + total) + total);
      if (int e = launch_maxpool_fwd<T>((const T*)in, g, (T*)l.out, l.arg, l.mask_in, st)) return e;
      CE_CHECK_LAUNCH();
    } else {
      const int B = n, K = l.in_units, O = l.out_units;
      if (l.head) {  // logits (+ loss and dL/dlogits when training) in one kernel
        const bool with_loss = loss && B <= kHeadMaxBatch;
        Prof pf(net, P_DENSE_FWD, 2.0 * B * K * O, 4.0 * K * O + (in_act ? act_bytes(net) : 4.0) * B * K, 1);
        unsigned* ticket = (unsigned*)(net->d_step + 2);
        const int32_t* lab = with_loss ? net->ybatch : nullptr;
        int s = in_act ? launch_head_fwd((const T*)in, K, l.W, l.b, B, K, O, net->ws, ticket, (float*)l.out, lab,
                                         (float*)net->gbuf[0], net->d_losses, net->d_step, net->d_step + 1,
                                         net->num_sms, st)
                       : launch_head_fwd((const float*)in, K, l.W, l.b, B, K, O, net->ws, ticket, (float*)l.out, lab,
                                         (float*)net->gbuf[0], net->d_losses, net->d_step, net->d_step + 1,
                                         net->num_sms, st);
        if (s != CE_OK) return s;
        if (with_loss) *loss_fused = true;
        CE_CHECK_LAUNCH();
        in = l.out;
        in_act = false;
        continue;
      }
      long long bps = simt_tiles(B, O);
      int splits = simt_splits(K, pick_splits(bps, K, 256, net->num_sms, 8, 256));
      while (splits > 1 && (size_t)splits * B * O * 4 > net->ws_bytes) splits = simt_splits(K, splits - 1);
      // weights are read once in the operand type: the bf16 mirror on the tensor-core path, fp32 otherwise
      Prof pf(net, P_DENSE_FWD, 2.0 * B * K * O, (net->use_tc ? 2.0 : 4.0) * K * O + (in_act ? act_bytes(net) : 4.0) * B * K, 2);
      if (net->use_tc) {
        const bf16* x16 = (const bf16*)in;
        if (!in_act) {
          f32_to_bf16_pad_kernel<<<grid_for((size_t)B * l.in_pad), 256, 0, st>>>((const float*)in, B, K, l.in_pad,
                                                                                   l.x16);
          x16 = l.x16;
          net->acc += 1;
        }
        int s = dense_fwd_tc(x16, l.in_pad, l.Wbp, K, l.in_pad, O, B, net->ws, &splits, net->num_sms, st);
        if (s != CE_OK) return s;
      } else if (dense_split3_enabled(B, (long long)K * O)) {  // fp32 check mode on the tensor cores
        int s = dense_fwd_split3((const float*)in, K, l.W, K, O, B, net->ws, &splits, net->num_sms, st);
        if (s != CE_OK) return s;
      } else if (dense_stream_enabled(B, K, (long long)K * O) &&
                 (size_t)dense_fwd_stream_splits(B, K, O, net->num_sms) * B * O * 4 <= net->ws_bytes) {
        splits = dense_fwd_stream((const float*)in, l.W, B, K, O, dense_fwd_stream_splits(B, K, O, net->num_sms),
                                  net->ws, st);
      } else if (dense_fwd_simt_enabled()) {
        splits = dense_fwd_simt_splits(B, K, O, net->num_sms);
        while (splits > 1 && (size_t)splits * B * O * 4 > net->ws_bytes) --splits;
        splits = in_act ? dense_fwd_simt((const T*)in, l.W, B, K, O, splits, net->ws, st)
                        : dense_fwd_simt((const float*)in, l.W, B, K, O, splits, net->ws, st);
      } else {
        PartialEpi pe{net->ws, B, O};
        if (in_act)
          simt_gemm(DenseXA<T>{(const T*)in, K}, DenseWB{l.W, K}, pe, B, O, K, splits, st);
        else
          simt_gemm(DenseXA<float>{(const float*)in, K}, DenseWB{l.W, K}, pe, B, O, K, splits, st);
      }
      launch_dense_reduce(net->ws, splits, B, O, l.b, (float*)l.out, st);
    }
    CE_CHECK_LAUNCH();
    in = l.out;
    in_act = l.kind != CE_LAYER_DENSE;
  }
  return CE_OK;
}

template <class TO, class TM>
struct DenseDxEpi {
  TO* dx;
  const TM* mask;
  int in;
  __device__ void operator()(int b, int i, int, float v) const {
    size_t off = (size_t)b * in + i;
    if (mask && !(ldf(mask, off) > 0.f)) v = 0.f;
    stf(dx, off, v);
  }
};

// ----------------------------------------------------------------------------- backward + SGD
template <class T>
int enqueue_backward(ce_net* net, int n, float lr, float mu) {
  cudaStream_t st = net->st;
  int cur = 0;  // gbuf[cur] holds dL/d(output of layer li) (pre-ReLU for conv)
  const bool keep = net->keep_grads;
  for (int li = (int)net->L.size() - 1; li >= 0; --li) {
    Layer& l = net->L[li];
    net->prof_layer_cur = li;
    const void* x = li == 0 ? net->x0 : net->L[li - 1].out;
    const void* gin = net->gbuf[cur];
    void* gout = net->gbuf[cur ^ 1];
    const T* mask = (l.mask_in && li > 0) ? (const T*)net->L[li - 1].out : nullptr;
    if (l.kind == CE_LAYER_DENSE && l.head) {
      const int B = n, K = l.in_units, O = l.out_units;
      const float* g = (const float*)gin;
      // algorithmic bytes: fused momentum SGD reads W, V and writes W, V (16 B/param, fp32 master);
      // dX reuses the same W pass; x is read and dX written once
      Prof pf(net, P_DENSE_BWD, (l.need_dx ? 4.0 : 2.0) * B * K * O,
              16.0 * K * O + (l.need_dx ? 2.0 : 1.0) * (l.in_is_act ? act_bytes(net) : 4.0) * B * K, 1);
      int s = l.in_is_act
                  ? launch_head_bwd((const T*)x, K, g, B, K, O, l.W, l.VW, keep ? l.GW : nullptr,
                                    l.need_dx ? (T*)gout : (T*)nullptr, mask, l.b, l.Vb, keep ? l.Gb : nullptr, lr, mu,
                                    st)
                  : launch_head_bwd((const float*)x, K, g, B, K, O, l.W, l.VW, keep ? l.GW : nullptr,
                                    l.need_dx ? (float*)gout : (float*)nullptr, (const float*)nullptr, l.b, l.Vb,
                                    keep ? l.Gb : nullptr, lr, mu, st);
      if (s != CE_OK) return s;
      CE_CHECK_LAUNCH();
    } else if (l.kind == CE_LAYER_DENSE) {
      const int B = n, K = l.in_units, O = l.out_units;
      const float* g = (const float*)gin;
      // algorithmic bytes: SGD over the fp32 master (W, V read + written: 16 B/param) plus, on the tensor-core
      // path, the bf16 mirror rewrite (2) and the dX pass over that mirror (2); fp32 mode reads fp32 W for dX (4)
      const double per_param = net->use_tc ? 18.0 + (l.need_dx ? 2.0 : 0.0) : 16.0 + (l.need_dx ? 4.0 : 0.0);
      Prof pf(net, P_DENSE_BWD, (l.need_dx ? 4.0 : 2.0) * B * K * O,
              per_param * K * O + (l.need_dx ? 2.0 : 1.0) * (l.in_is_act ? act_bytes(net) : 4.0) * B * K,
              l.need_dx ? 4 : 3);
      if (net->use_tc) {
        const bool dw_simt = dense_dw_simt_enabled(B);
        if (l.need_dx || !dw_simt) {
          f32_to_bf16_pad_kernel<<<grid_for((size_t)B * l.out_pad), 256, 0, st>>>(g, B, O, l.out_pad, net->gbf);
          CE_CHECK_LAUNCH();
        }
        if (l.need_dx) {
          int s = l.in_is_act ? dense_dx_tc(l.Wbp, net->gbf, K, l.in_pad, O, l.out_pad, B, mask, (T*)gout,
                                            net->num_sms, st)
                              : dense_dx_tc(l.Wbp, net->gbf, K, l.in_pad, O, l.out_pad, B, (const float*)nullptr,
                                            (float*)gout, net->num_sms, st);
          if (s != CE_OK) return s;
        }
        const bf16* xb = l.in_is_act ? (const bf16*)x : l.x16;
        if (dw_simt) {
          dense_dw_sgd_simt(xb, l.in_pad, g, B, K, O, l.W, l.VW, keep ? l.GW : nullptr, l.Wbp, l.in_pad, lr, mu, st);
          CE_CHECK_LAUNCH();
        } else {
          int s = dense_dw_sgd_tc(xb, l.in_pad, net->gbf, K, l.in_pad, O, l.out_pad, B, l.W, l.VW,
                                  keep ? l.GW : nullptr, l.Wbp, lr, mu, net->num_sms, st);
          if (s != CE_OK) return s;
        }
      } else {
      const bool small = B <= kDenseSimtMaxBatch;
      if (l.need_dx) {
        if constexpr (std::is_same<T, float>::value) {
          if (dense_split3_enabled(B, (long long)K * O)) {  // fp32 check mode on the tensor cores
            int s = l.in_is_act ? dense_dx_split3(g, l.W, B, K, O, mask, (float*)gout, net->num_sms, st)
                                : dense_dx_split3(g, l.W, B, K, O, (const float*)nullptr, (float*)gout,
                                                  net->num_sms, st);
            if (s != CE_OK) return s;
            goto dx_done;
          }
          if (dense_stream_enabled(B, K, (long long)K * O)) {  // streaming-W FFMA
            if (l.in_is_act)
              dense_dx_stream(g, l.W, B, K, O, mask, (float*)gout, st);
            else
              dense_dx_stream(g, l.W, B, K, O, (const float*)nullptr, (float*)gout, st);
            goto dx_done;
          }
        }
        if (small) {
          if (l.in_is_act)
            dense_dx_simt(g, l.W, B, K, O, mask, (T*)gout, st);
          else
            dense_dx_simt(g, l.W, B, K, O, (const float*)nullptr, (float*)gout, st);
        } else if (l.in_is_act) {
          simt_gemm(DenseGA{g, O}, DenseWN{l.W, K}, DenseDxEpi<T, T>{(T*)gout, mask, K}, B, K, O, 1, st);
        } else {
          simt_gemm(DenseGA{g, O}, DenseWN{l.W, K}, DenseDxEpi<float, float>{(float*)gout, nullptr, K}, B, K, O, 1,
                    st);
        }
      dx_done:
        CE_CHECK_LAUNCH();
      }
      if (small) {
        if (l.in_is_act)
          dense_dw_sgd_simt((const T*)x, K, g, B, K, O, l.W, l.VW, keep ? l.GW : nullptr, (bf16*)nullptr, 0, lr, mu,
                            st);
        else
          dense_dw_sgd_simt((const float*)x, K, g, B, K, O, l.W, l.VW, keep ? l.GW : nullptr, (bf16*)nullptr, 0, lr,
                            mu, st);
      } else {
        DenseSgdEpi se{l.W, l.VW, keep ? l.GW : nullptr, nullptr, K, lr, mu};
        if (l.in_is_act)
          simt_gemm(DenseGT{g, O}, DenseXN<T>{(const T*)x, K}, se, O, K, B, 1, st);
        else
          simt_gemm(DenseGT{g, O}, DenseXN<float>{(const float*)x, K}, se, O, K, B, 1, st);
      }
      CE_CHECK_LAUNCH();
      }
      float* bpart = net->ws;
      int bs = colsum(g, B, O, bpart, st);
      launch_bias_sgd(bpart, bs, O, l.b, l.Vb, keep ? l.Gb : nullptr, lr, mu, st);
      CE_CHECK_LAUNCH();
    } else if (l.kind == CE_LAYER_CONV) {
      ConvGeom g = l.g;
      g.n = n;
      const T* dy = (const T*)gin;
      const int Mo = n * g.oh * g.ow, K = g.k * g.k * g.c;
      const double ab = (double)act_bytes(net);
      const double useful = 2.0 * Mo * g.co * g.k * g.k * l.c_real;
      if (l.need_dx) {
        Prof pf(net, P_CONV_DGRAD, useful,
                ab * ((double)Mo * g.co + (double)g.co * K + 2.0 * n * g.h * g.w * g.c));
        if (net->use_tc) {
          int s = l.col2im ? conv_dgrad_col2im(g, (const bf16*)dy, l.Wbf, (const bf16*)mask, (bf16*)gout, net->zbuf,
                                             net->num_sms, st)
                         : conv_dgrad_tc(g, (const bf16*)dy, l.Wtbf, (const bf16*)mask, (bf16*)gout, net->num_sms, st);
          if (s != CE_OK) return s;
        } else {
          simt_gemm(make_dgrad_a(dy, g), DgradB{l.W, g}, DgradEpi<T>{(T*)gout, mask, g.c}, n * g.h * g.w, g.c,
                    g.k * g.k * g.co, 1, st);
        }
        CE_CHECK_LAUNCH();
      }
      int splits;
      {
      Prof pf(net, P_CONV_WGRAD, useful, ab * ((double)Mo * g.co + (double)n * g.h * g.w * g.c));
      if (l.packed && !net->use_tc) {
        const long long Mo_ = (long long)n * g.oh * g.ow;
        splits = simt_splits((int)Mo_, pick_splits(simt_tiles(g.co, l.Kp), Mo_, 512, net->num_sms));
        while (splits > 1 && (size_t)splits * g.co * l.Kp * 4 > net->ws_bytes) splits = simt_splits((int)Mo_, splits - 1);
        conv_wgrad_packed_simt(g, (const float*)l.xcol, l.Kp, (const float*)dy, net->ws, splits, st);
      } else if (l.packed) {
        const PoolMap pm = l.pool_fused ? layer_pool_map(net, li, n) : PoolMap{};
        const int rows = l.pool_fused ? pool_rows(pm) : Mo;
        int s = conv_wgrad_packed_implicit(g, (const bf16*)x, l.c_real, l.Kp, (const bf16*)dy,
                                           l.pool_fused ? &pm : nullptr, net->ws, &splits, net->num_sms, st);
        if (s != CE_OK) return s;
        pf.bytes = ab * ((double)rows * g.co + (double)n * g.h * g.w * g.c) + 4.0 * splits * g.co * l.Kp;
      } else if (net->use_tc) {
        int s = conv_wgrad_tc(g, (const bf16*)x, (const bf16*)dy, net->ws, &splits, net->num_sms, st);
        if (s != CE_OK) return s;
        pf.bytes += 4.0 * splits * g.co * K;
      } else {
        long long bps = simt_tiles(g.co, K);
        splits = simt_splits(Mo, pick_splits(bps, Mo, 512, net->num_sms));
        while (splits > 1 && (size_t)splits * g.co * K * 4 > net->ws_bytes) splits = simt_splits(Mo, splits - 1);
        simt_gemm(WgradA<T>{dy, g.co}, WgradB<T>{make_fwd_a((const T*)x, g)}, PartialEpi{net->ws, g.co, K}, g.co, K, Mo,
                  splits, st);
      }
      CE_CHECK_LAUNCH();
      }
      if (l.packed) {  // bias gradient = row Kr of the packed wgrad: no column-sum pass
        Prof pf(net, P_CONV_SGD, 0.0, 4.0 * splits * g.co * l.Kp + 20.0 * g.co * (packed_kr(g, l.c_real) + 1));
        if (l.Wpf)
          launch_conv_sgd_packed(net->ws, splits, g, l.c_real, l.Kp, l.W, l.VW, keep ? l.GW : nullptr, l.Wpf, l.b,
                                 l.Vb, keep ? l.Gb : nullptr, lr, mu, st);
        else
          launch_conv_sgd_packed(net->ws, splits, g, l.c_real, l.Kp, l.W, l.VW, keep ? l.GW : nullptr, l.Wp, l.b,
                                 l.Vb, keep ? l.Gb : nullptr, lr, mu, st);
        CE_CHECK_LAUNCH();
        if (!l.need_dx) break;
        cur ^= 1;
        continue;
      }
      float* bpart = net->ws + (size_t)splits * g.co * K;
      Prof pf(net, P_CONV_SGD, 0.0, ab * Mo * g.co + 4.0 * splits * g.co * K + 20.0 * g.co * K, 3);
      int bsplits = colsum(dy, Mo, g.co, bpart, st);
      launch_conv_sgd(net->ws, splits, g.co, K, g.c, g.k, g.s, l.W, l.VW, keep ? l.GW : nullptr, l.Wbf, l.Wtbf, bpart,
                      bsplits, l.b, l.Vb, keep ? l.Gb : nullptr, lr, mu, st);
      CE_CHECK_LAUNCH();
    } else {  // pool
      if (l.need_dx && l.fused && net->L[li - 1].packed) {
        // dY of the packed conv in its window-major xcol row order (no raster pass)
        const PoolMap pm = layer_pool_map(net, li - 1, n);
        Prof pf(net, P_POOL, 0.0, (double)act_bytes(net) * ((double)pool_rows(pm) + pm.windows) * l.g.c +
                                      (double)pm.windows * l.g.c);
        launch_pool_expand_rows((const T*)gin, l.arg, pm, l.g.c, (T*)gout, st);
        CE_CHECK_LAUNCH();
      } else if (l.need_dx) {
        ConvGeom g = l.g;
        g.n = n;
        size_t total = (size_t)n * g.h * g.w * g.c;
        // algorithmic bytes: dy + dx in the activation type, argmax 1 B per pooled element; the ReLU
        // mask of the input is folded into the argmax by the forward (kPoolDead)
        Prof pf(net, P_POOL, 0.0, (double)act_bytes(net) * ((double)n * g.oh * g.ow * g.c + total) +
                                      (double)n * g.oh * g.ow * g.c);
        if (int e = launch_maxpool_bwd<T, T>((const T*)gin, l.arg, g, (const T*)nullptr, (T*)gout, st)) return e;
        CE_CHECK_LAUNCH();
      }
    }
    if (!l.need_dx) break;  // nothing below needs gradients
    cur ^= 1;
  }
  return CE_OK;
}

template <class T>
int enqueue_step(ce_net* net, int n, float lr, float mu) {
  bool loss_fused = false;
  int s = enqueue_forward<T>(net, n, true, &loss_fused);
  if (s != CE_OK) return s;
  const Layer& last = net->L.back();
  net->prof_layer_cur = -1;
  if (!loss_fused) {
    Prof pf(net, P_LOSS, 0.0, 16.0 * n * net->classes);
    xent_kernel<int32_t><<<1, 1024, 0, net->st>>>((const float*)last.out, net->ybatch, n, net->classes,
                                          (float*)net->gbuf[0], net->d_losses, net->d_step, net->d_step + 1);
    CE_CHECK_LAUNCH();
  }
  return enqueue_backward<T>(net, n, lr, mu);
}

int forward_any(ce_net* net, int n) {
  return net->prec == CE_PREC_FP32 ? enqueue_forward<float>(net, n) : enqueue_forward<bf16>(net, n);
}
int step_any(ce_net* net, int n, float lr, float mu) {
  return net->prec == CE_PREC_FP32 ? enqueue_step<float>(net, n, lr, mu) : enqueue_step<bf16>(net, n, lr, mu);
}

int gather_any(ce_net* net, const ce_dataset* ds, const int32_t* perm, int n_perm, int spe, int base, int B,
               bool labels) {
  dim3 grid = gather_grid(ds->h * ds->w, B);
  int HW = ds->h * ds->w;
  net->prof_layer_cur = -1;
  Prof pf(net, P_GATHER, 0.0, (double)B * HW * (ds->c + net->in_cp * act_bytes(net)));
  if (net->prec == CE_PREC_FP32)
    gather_u8_kernel<float><<<grid, 256, 0, net->st>>>(ds->pix, ds->lab, perm, net->d_step, n_perm, spe, base, B,
                                                       ds->c, net->in_cp, HW, (float*)net->x0,
                                                       labels ? net->ybatch : nullptr);
  else
    gather_u8_kernel<bf16><<<grid, 256, 0, net->st>>>(ds->pix, ds->lab, perm, net->d_step, n_perm, spe, base, B,
                                                      ds->c, net->in_cp, HW, (bf16*)net->x0,
                                                      labels ? net->ybatch : nullptr);
  CE_CHECK_LAUNCH();
  return CE_OK;
}

int upload_host_batch(ce_net* net, const float* x, int n) {
  size_t elems = (size_t)n * net->in_c * net->in_h * net->in_w;
  if (elems > net->xhost_cap) {
    if (net->d_xhost) {
      cudaFreeAsync(net->d_xhost, net->st);
      net->allocs.erase(std::find(net->allocs.begin(), net->allocs.end(), (void*)net->d_xhost));
    }
    ALLOC(net->d_xhost, elems * 4);
    net->xhost_cap = elems;
  }
  CE_CUDA(cudaMemcpyAsync(net->d_xhost, x, elems * 4, cudaMemcpyHostToDevice, net->st));
  int HW = net->in_h * net->in_w;
  size_t total = (size_t)n * HW;
  net->acc += 1;
  if (net->prec == CE_PREC_FP32)
    nchw_to_nhwc_kernel<float><<<grid_for(total), 256, 0, net->st>>>(net->d_xhost, n, net->in_c, net->in_cp, HW,
                                                                      (float*)net->x0);
  else
    nchw_to_nhwc_kernel<bf16><<<grid_for(total), 256, 0, net->st>>>(net->d_xhost, n, net->in_c, net->in_cp, HW,
                                                                     (bf16*)net->x0);
  CE_CHECK_LAUNCH();
  return CE_OK;
}

int check_net(const ce_net* net) {
  if (!net) return fail(CE_EINVAL, "null net");
  return CE_OK;
}

// RAII for ce_train's graph exec and events: every return path (including a
// failed launch inside the replay loop) drains the stream and releases them
struct TrainRes {
  cudaGraphExec_t exec = nullptr;
  cudaEvent_t ev[4] = {};
  cudaStream_t owner = nullptr;
  ~TrainRes() {
    if (owner) cudaStreamSynchronize(owner);
    if (exec) cudaGraphExecDestroy(exec);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  }
};

}  // namespace

// =============================================================================== C ABI
extern "C" {

int ce_version(void) { return 1; }
long long ce_launch_count(void) { return g_launches.load(); }
int ce_prof_num_classes(void) { return P_NCLASS; }

int ce_net_set_profiling(ce_net* net, int on) {
  if (!net) return fail(CE_EINVAL, "null net");
  net->prof_on = on != 0;
  if (on) {
    for (auto& t : net->prof) t = ProfTotals();
    net->prof_layers.clear();
  }
  return CE_OK;
}

int ce_net_prof_layer(ce_net* net, int layer, int cls, long long* launches, double* ms, double* flops, double* bytes,
                      double* ideal_ms) {
  if (!net || cls < 0 || cls >= P_NCLASS) return fail(CE_EINVAL, "bad profile class %d", cls);
  auto it = net->prof_layers.find({layer, cls});
  const ProfTotals t = it == net->prof_layers.end() ? ProfTotals() : it->second;
  if (launches) *launches = t.launches;
  if (ms) *ms = t.ms;
  if (flops) *flops = t.flops;
  if (bytes) *bytes = t.bytes;
  if (ideal_ms) *ideal_ms = t.ideal_ms;
  return CE_OK;
}

int ce_net_prof_read(ce_net* net, int cls, const char** name, long long* launches, double* ms, double* flops,
                     double* bytes) {
  if (!net || cls < 0 || cls >= P_NCLASS) return fail(CE_EINVAL, "bad profile class %d", cls);
  const ProfTotals& t = net->prof[cls];
  if (name) *name = kProfNames[cls];
  if (launches) *launches = t.launches;
  if (ms) *ms = t.ms;
  if (flops) *flops = t.flops;
  if (bytes) *bytes = t.bytes;
  return CE_OK;
}
int ce_prof_set_peaks(double flops_per_s, double bytes_per_s) {
  if (!(flops_per_s > 0) || !(bytes_per_s > 0)) return fail(CE_EINVAL, "peaks must be positive");
  g_peak_flops = flops_per_s;
  g_peak_bytes = bytes_per_s;
  return CE_OK;
}

int ce_net_prof_ideal(ce_net* net, int cls, double* ideal_ms) {
  if (!net || cls < 0 || cls >= P_NCLASS || !ideal_ms) return fail(CE_EINVAL, "bad profile class %d", cls);
  *ideal_ms = net->prof[cls].ideal_ms;
  return CE_OK;
}

const char* ce_last_error(void) { return g_err; }

int ce_device_count(int* count) {
  CE_CUDA(cudaGetDeviceCount(count));
  return CE_OK;
}

int ce_dataset_create(int device, const uint8_t* pixels, const uint8_t* labels, int n, int c, int h, int w,
                      ce_dataset** out) {
  if (!pixels || !labels || !out || n <= 0 || c <= 0 || h <= 0 || w <= 0)
    return fail(CE_EINVAL, "ce_dataset_create: bad arguments");
  DevGuard dg(device);
  ce_dataset* ds = new ce_dataset();
  ds->device = device;
  ds->n = n;
  ds->c = c;
  ds->h = h;
  ds->w = w;
  size_t bytes = (size_t)n * c * h * w;
  cudaError_t e1 = cudaMalloc(&ds->pix, bytes);
  cudaError_t e2 = cudaMalloc(&ds->lab, n);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    cudaGetLastError();
    if (ds->pix) cudaFree(ds->pix);
    if (ds->lab) cudaFree(ds->lab);
    delete ds;
    return fail(CE_ENOMEM, "dataset allocation of %zu bytes failed", bytes);
  }
  CE_CUDA(cudaMemcpy(ds->pix, pixels, bytes, cudaMemcpyHostToDevice));
  CE_CUDA(cudaMemcpy(ds->lab, labels, n, cudaMemcpyHostToDevice));
  *out = ds;
  return CE_OK;
}

int ce_dataset_destroy(ce_dataset* ds) {
  if (!ds) return CE_OK;
  DevGuard dg(ds->device);
  cudaFree(ds->pix);
  cudaFree(ds->lab);
  delete ds;
  return CE_OK;
}

int ce_net_destroy(ce_net* net) {
  if (!net) return CE_OK;
  DevGuard dg(net->device);
  cudaStreamSynchronize(net->st);
  for (void* p : net->allocs) cudaFreeAsync(p, net->st);
  cudaStreamSynchronize(net->st);
  cudaStreamDestroy(net->st);
  delete net;
  return CE_OK;
}

int ce_net_create(const ce_net_desc* d, int device, int precision, ce_net** out) {
  if (!d || !out || d->n_layers < 1 || !d->layers) return fail(CE_EINVAL, "ce_net_create: bad descriptor");
  if (precision != CE_PREC_BF16 && precision != CE_PREC_FP32) return fail(CE_EINVAL, "bad precision %d", precision);
  if (d->max_batch < 1 || d->max_batch > 1024) return fail(CE_EINVAL, "max_batch %d out of range", d->max_batch);
  DevGuard dg(device);
  ce_net* net = new ce_net();
  net->device = device;
  net->prec = precision;
  net->in_c = d->in_c;
  net->in_cp = (d->in_c + 7) / 8 * 8;
  net->in_h = d->in_h;
  net->in_w = d->in_w;
  net->max_batch = d->max_batch;
  cudaDeviceGetAttribute(&net->num_sms, cudaDevAttrMultiProcessorCount, device);
  keep_pool_memory(device);
  if (cudaStreamCreateWithFlags(&net->st, cudaStreamNonBlocking) != cudaSuccess) {
    delete net;
    return fail(CE_ECUDA, "stream creation failed");
  }
  net->use_tc = precision == CE_PREC_BF16 && conv_tc_enabled();
  int rc = CE_OK;
  auto bail = [&](int s) {
    ce_net_destroy(net);
    return s;
  };
  // ---- shapes
  int c = d->in_c, cs = net->in_cp, h = d->in_h, w = d->in_w;
  bool features_done = false, seen_param = false;
  int prev_kind = 0, prev_relu = 0;
  int units = 0;
  for (int i = 0; i < d->n_layers; ++i) {
    const ce_layer_desc& ld = d->layers[i];
    Layer l;
    l.kind = ld.kind;
    if (ld.kind == CE_LAYER_CONV || ld.kind == CE_LAYER_POOL) {
      if (features_done) return bail(fail(CE_EINVAL, "layer %d: feature layer after dense", i));
      int k = ld.kernel, s = ld.stride;
      if (k < 1 || s < 1) return bail(fail(CE_EINVAL, "layer %d: kernel and stride must be >= 1", i));
      if (h < k || w < k) return bail(fail(CE_EINVAL, "layer %d: window %d exceeds input %dx%d", i, k, h, w));
      l.g.c = cs;
      l.g.h = h;
      l.g.w = w;
      l.g.k = k;
      l.g.s = s;
      l.g.oh = (h - k) / s + 1;
      l.g.ow = (w - k) / s + 1;
      l.c_real = c;
      if (ld.kind == CE_LAYER_CONV) {
        if (ld.out_channels < 1 || ld.out_channels % 8) return bail(fail(CE_EINVAL, "layer %d: out_channels %d not a multiple of 8", i, ld.out_channels));
        l.g.co = ld.out_channels;
        l.relu = ld.relu;
        l.out_c_store = l.out_c_real = ld.out_channels;
      } else {
        l.g.co = cs;
        l.out_c_store = cs;
        l.out_c_real = c;
      }
      l.need_dx = seen_param;
      l.mask_in = prev_kind == CE_LAYER_CONV && prev_relu;
      l.out_per_sample = (size_t)l.g.oh * l.g.ow * l.out_c_store;
      if (ld.kind == CE_LAYER_CONV) {
        seen_param = true;
        c = cs = l.g.co;
      }
      h = l.g.oh;
      w = l.g.ow;
    } else if (ld.kind == CE_LAYER_DENSE) {
      if (ld.units < 1) return bail(fail(CE_EINVAL, "layer %d: dense units must be >= 1", i));
      if (!features_done) {
        l.in_units = h * w * cs;
        l.hw_in = h * w;
        l.c_real = c;
        l.in_is_act = true;
        features_done = true;
      } else {
        l.in_units = units;
        l.hw_in = 0;
        l.c_real = units;
        l.in_is_act = false;
      }
      l.out_units = ld.units;
      l.need_dx = seen_param;
      l.mask_in = prev_kind == CE_LAYER_CONV && prev_relu;
      l.out_per_sample = ld.units;
      seen_param = true;
      units = ld.units;
    } else {
      return bail(fail(CE_EINVAL, "layer %d: unknown kind %d", i, ld.kind));
    }
    prev_kind = ld.kind;
    prev_relu = ld.relu;
    net->L.push_back(l);
  }
  if (net->L.back().kind != CE_LAYER_DENSE) return bail(fail(CE_EINVAL, "network must end in a Dense layer"));
  net->classes = net->L.back().out_units;
  // ---- packed first layers and conv + max-pool fusion
  for (size_t i = 0; i < net->L.size(); ++i) {
    Layer& l = net->L[i];
    if (l.kind != CE_LAYER_CONV) continue;
    const long long Mo = (long long)d->max_batch * l.g.oh * l.g.ow;
    l.packed = (net->use_tc || precision == CE_PREC_FP32) && l.c_real < l.g.c && !l.need_dx && !packed_disabled() &&
               packable(l.g, l.c_real) &&
               packed_kp(l.g, l.c_real) <= kPackedMaxKp && Mo * packed_kp(l.g, l.c_real) / 8 < (1ll << 32);
    if (i + 1 < net->L.size() && net->L[i + 1].kind == CE_LAYER_POOL && net->use_tc &&
        pool_fusable(net->L[i + 1].g.k, net->L[i + 1].g.s) && pool_fusion_mode() > 0 &&
        (pool_fusion_mode() >= 2 || l.packed || (l.g.c % 64 != 0 && !im2col32_ok(l.g)))) {
      l.pool_fused = true;
      net->L[i + 1].fused = true;
    }
  }
  // ---- allocations
  const size_t B = d->max_batch, ab = act_bytes(net);
  size_t total_params = 0;
  for (auto& l : net->L) {
    if (l.kind == CE_LAYER_CONV) total_params += (size_t)l.g.co * l.g.k * l.g.k * l.g.c;
    if (l.kind == CE_LAYER_DENSE) total_params += (size_t)l.out_units * l.in_units;
  }
  net->keep_grads = false;  // opt-in (ce_net_keep_grads): storing dW costs 4 B/param/step
  size_t max_g = (size_t)B * net->in_cp * net->in_h * net->in_w * ab, ws = 0, gbf_elems = 0, zbytes = 0;
  for (size_t i = 0; i < net->L.size(); ++i) {
    Layer& l = net->L[i];
    if (l.kind == CE_LAYER_DENSE) {
      ALLOC(l.out, B * l.out_units * 4);
      max_g = std::max(max_g, B * l.out_units * 4);
      max_g = std::max(max_g, B * (size_t)l.in_units * (l.in_is_act ? ab : 4));
      l.wn = (size_t)l.out_units * l.in_units;
      l.bn = l.out_units;
      l.in_pad = (l.in_units + 7) / 8 * 8;
      l.out_pad = (l.out_units + 7) / 8 * 8;
      l.head = i + 1 == net->L.size() && l.out_units <= kHeadMaxOut && !head_disabled();
      if (l.head) {  // partial logits of the forward CTAs
        ws = std::max(ws, (size_t)head_fwd_grid(l.in_units, net->num_sms, 1) * B * l.out_units * 4);
      } else if (net->use_tc) {
        if (l.in_is_act && l.in_pad != l.in_units) return bail(fail(CE_EINVAL, "feature width not a multiple of 8"));
        ALLOC(l.Wbp, (size_t)l.out_units * l.in_pad * 2);
        if (!l.in_is_act) ALLOC(l.x16, B * (size_t)l.in_pad * 2);
        gbf_elems = std::max(gbf_elems, B * (size_t)l.out_pad);
        int spt = dense_fwd_splits(l.out_units, l.in_units, net->num_sms);
        ws = std::max(ws, (size_t)spt * B * l.out_units * 4);
      }
      if (precision == CE_PREC_FP32 && dense_stream_enabled(1, l.in_units, (long long)l.in_units * l.out_units))
        for (int bq : {(int)B, std::min((int)B, 64), std::min((int)B, 32), std::min((int)B, 16)})
          ws = std::max(ws, (size_t)dense_fwd_stream_splits(bq, l.in_units, l.out_units, net->num_sms) * bq *
                                l.out_units * 4);
      if (precision == CE_PREC_FP32 && dense_split3_enabled(1, (long long)l.in_units * l.out_units))
        ws = std::max(ws, (size_t)dense_fwd_split3_splits(l.out_units, l.in_units, net->num_sms) * B * l.out_units * 4);
      long long bps = simt_tiles((int)B, l.out_units);
      int sp = simt_splits(l.in_units, pick_splits(bps, l.in_units, 256, net->num_sms, 8, 256));
      ws = std::max(ws, (size_t)sp * B * l.out_units * 4);
      ws = std::max(ws, (size_t)dense_fwd_simt_splits((int)B, l.in_units, l.out_units, net->num_sms) * B *
                            l.out_units * 4);
      ws = std::max(ws, (size_t)(kColsumMaxSplits + 64) * l.out_units * 4);
    } else {
      if (!l.pool_fused) ALLOC(l.out, B * l.out_per_sample * ab);  // fused: only the pooled map exists
      max_g = std::max(max_g, B * l.out_per_sample * ab);
      if (l.kind == CE_LAYER_POOL) ALLOC(l.arg, B * l.out_per_sample);
      if (l.kind == CE_LAYER_CONV) {
        const int K = l.g.k * l.g.k * l.g.c;
        l.wn = (size_t)l.g.co * K;
        l.bn = l.g.co;
        long long Mo = (long long)B * l.g.oh * l.g.ow;
        long long bps = simt_tiles(l.g.co, K);
        int sp = simt_splits((int)Mo, pick_splits(bps, Mo, 512, net->num_sms));
        sp = std::max(sp, conv_wgrad_tc_max_splits(l.g, (int)B, net->num_sms));
        ws = std::max(ws, (size_t)sp * l.g.co * K * 4 + (size_t)(kColsumMaxSplits + 64) * l.g.co * 4);
        if (net->use_tc) {  // split-K partials of a sub-wave forward, for any batch the net may run
          ConvGeom gb = l.g;
          const Layer* pool = i + 1 < net->L.size() && net->L[i + 1].fused ? &net->L[i + 1] : nullptr;
          for (gb.n = 1; gb.n <= (int)B; ++gb.n)
            ws = std::max(ws, pool ? conv_pool_ws_bytes(gb, pool->g.k, pool->g.s, net->num_sms)
                                   : conv_fwd_ws_bytes(gb, net->num_sms));
        }
        l.col2im = net->use_tc && l.need_dx && col2im_dgrad_eligible(l.g);
        if (l.col2im) zbytes = std::max(zbytes, col2im_dgrad_zbytes(l.g, (int)B));
        if (l.packed) {
          l.Kp = packed_kp(l.g, l.c_real);
          // rows of the packed GEMMs: pixels, or the window-major pooled order (padding rows included)
          const long long rows = l.pool_fused ? pool_rows(layer_pool_map(net, i, (int)B)) : Mo;
          const int psp = conv_wgrad_packed_splits(l.Kp, (int)rows, net->num_sms);
          ws = std::max(ws, (size_t)psp * l.g.co * l.Kp * 4);
          max_g = std::max(max_g, (size_t)rows * l.g.co * ab);  // window-major dY of the fused pool
          if (precision == CE_PREC_FP32) ALLOC(l.xcol, (size_t)rows * l.Kp * ab);  // bf16: implicit operand
          if (precision == CE_PREC_FP32) {
            ALLOC(l.Wpf, (size_t)l.g.co * l.Kp * 4);
            ws = std::max(ws, (size_t)simt_splits((int)Mo, pick_splits(simt_tiles(l.g.co, l.Kp), Mo, 512,
                                                                         net->num_sms)) * l.g.co * l.Kp * 4);
          }
        }
      }
    }
    if (l.wn) {
      l.pidx = (int)net->params.size();
      net->params.push_back((int)i);
      ALLOC(l.W, l.wn * 4);
      ALLOC(l.VW, l.wn * 4);
      ALLOC(l.b, l.bn * 4);
      ALLOC(l.Vb, l.bn * 4);

      if (precision == CE_PREC_BF16 && l.kind == CE_LAYER_CONV) {
        if (l.packed) {
          ALLOC(l.Wp, (size_t)l.g.co * l.Kp * 2);
        } else {
          ALLOC(l.Wbf, l.wn * 2);
          if (!l.col2im) ALLOC(l.Wtbf, l.wn * 2);  // col2im dgrad reads the forward mirror
        }
      }
      cudaMemsetAsync(l.W, 0, l.wn * 4, net->st);
      cudaMemsetAsync(l.VW, 0, l.wn * 4, net->st);
      cudaMemsetAsync(l.b, 0, l.bn * 4, net->st);
      cudaMemsetAsync(l.Vb, 0, l.bn * 4, net->st);
    }
  }
  ALLOC(net->x0, B * net->in_cp * net->in_h * net->in_w * ab);
  ALLOC(net->ybatch, B * 4);
  ALLOC(net->gbuf[0], max_g);
  ALLOC(net->gbuf[1], max_g);
  net->gbytes = max_g;
  ALLOC(net->ws, ws);
  net->ws_bytes = ws;
  if (zbytes) ALLOC(net->zbuf, zbytes);
  if (gbf_elems) ALLOC(net->gbf, gbf_elems * 2);
  ALLOC(net->d_step, 16);  // [0] step, [1] non-finite flag, [2] head ticket
  cudaMemsetAsync(net->d_step, 0, 16, net->st);
  net->losses_cap = 4096;
  ALLOC(net->d_losses, net->losses_cap * 4);
  cudaError_t e = cudaStreamSynchronize(net->st);
  if (e != cudaSuccess) return bail(fail(CE_ECUDA, "net create: %s", cudaGetErrorString(e)));
  (void)rc;
  *out = net;
  return CE_OK;
}

// Stream priority of the net (> 0: the device's highest, else default). The
// scheduler raises it for the slot that runs the longest candidates, so their
// kernels win the SM arbitration against the short candidates packed beside them.
int ce_net_set_priority(ce_net* net, int priority) {
  if (check_net(net)) return CE_EINVAL;
  DevGuard dg(net->device);
  int least = 0, greatest = 0;
  CE_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  cudaStream_t s = nullptr;
  CE_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority > 0 ? greatest : least));
  CE_CUDA(cudaStreamSynchronize(net->st));  // allocations made on the old stream are complete
  cudaStreamDestroy(net->st);
  net->st = s;
  return CE_OK;
}

int ce_net_device_bytes(const ce_net* net, size_t* bytes) {
  if (check_net(net)) return CE_EINVAL;
  *bytes = net->bytes;
  return CE_OK;
}

int ce_net_num_param_layers(const ce_net* net, int* count) {
  if (check_net(net)) return CE_EINVAL;
  *count = (int)net->params.size();
  return CE_OK;
}

static int param_layer(ce_net* net, int p, Layer** out) {
  if (!net || p < 0 || p >= (int)net->params.size()) return fail(CE_EINVAL, "param layer %d out of range", p);
  *out = &net->L[net->params[p]];
  return CE_OK;
}

static size_t host_w_count(const Layer& l) {
  if (l.kind == CE_LAYER_CONV) return (size_t)l.g.co * l.c_real * l.g.k * l.g.k;
  if (l.in_is_act) return (size_t)l.out_units * l.hw_in * l.c_real;
  return (size_t)l.out_units * l.in_units;
}

int ce_net_set_params(ce_net* net, int p, const float* w, const float* b) {
  Layer* lp;
  if (int s = param_layer(net, p, &lp)) return s;
  Layer& l = *lp;
  DevGuard dg(net->device);
  SharedGate gate(net->device);
  cudaStream_t st = net->st;
  size_t hn = host_w_count(l);
  // stage through a temporary in chunks of rows to bound memory for giant heads
  size_t rows = l.kind == CE_LAYER_CONV ? (size_t)l.g.co : (size_t)l.out_units;
  size_t hrow = hn / rows, drow = l.wn / rows;
  size_t chunk_rows = std::max<size_t>(1, std::min(rows, (size_t)(256u << 20) / (hrow * 4)));
  float* tmp = nullptr;
  CE_CUDA(cudaMallocAsync(&tmp, chunk_rows * hrow * 4, st));
  for (size_t r0 = 0; r0 < rows; r0 += chunk_rows) {
    size_t nr = std::min(chunk_rows, rows - r0);
    CE_CUDA(cudaMemcpyAsync(tmp, w + r0 * hrow, nr * hrow * 4, cudaMemcpyHostToDevice, st));
    float* dst = l.W + r0 * drow;
    if (l.kind == CE_LAYER_CONV)
      conv_w_to_dev_kernel<<<grid_for(nr * drow), 256, 0, st>>>(tmp, (int)nr, l.c_real, l.g.c, l.g.k, dst);
    else if (l.in_is_act)
      dense_w_to_dev_kernel<<<grid_for(nr * drow), 256, 0, st>>>(tmp, nr, l.c_real, l.in_units / l.hw_in, l.hw_in,
                                                                   dst);
    else
      CE_CUDA(cudaMemcpyAsync(dst, tmp, nr * drow * 4, cudaMemcpyDeviceToDevice, st));
    CE_CHECK_LAUNCH();
  }
  CE_CUDA(cudaFreeAsync(tmp, st));
  if (b) CE_CUDA(cudaMemcpyAsync(l.b, b, l.bn * 4, cudaMemcpyHostToDevice, st));
  else CE_CUDA(cudaMemsetAsync(l.b, 0, l.bn * 4, st));
  CE_CUDA(cudaMemsetAsync(l.VW, 0, l.wn * 4, st));
  CE_CUDA(cudaMemsetAsync(l.Vb, 0, l.bn * 4, st));
  if (l.Wbf) f32_to_bf16_kernel<<<grid_for(l.wn), 256, 0, st>>>(l.W, l.wn, l.Wbf);
  if (l.Wbp)
    f32_to_bf16_pad_kernel<<<grid_for((size_t)l.out_units * l.in_pad), 256, 0, st>>>(l.W, l.out_units, l.in_units,
                                                                                      l.in_pad, l.Wbp);
  if (l.Wtbf) conv_wt_kernel<<<grid_for(l.wn), 256, 0, st>>>(l.W, l.g.co, l.g.k, l.g.s, l.g.c, l.Wtbf);
  if (l.Wp)
    pack_first_w_kernel<<<grid_for((size_t)l.g.co * l.Kp), 256, 0, st>>>(l.W, l.g.co, l.g.k, l.g.c, l.c_real, l.Kp,
                                                                         l.Wp);
  if (l.Wpf)
    pack_first_w_kernel<<<grid_for((size_t)l.g.co * l.Kp), 256, 0, st>>>(l.W, l.g.co, l.g.k, l.g.c, l.c_real, l.Kp,
                                                                         l.Wpf);
  CE_CHECK_LAUNCH();
  CE_CUDA(cudaStreamSynchronize(st));
  return CE_OK;
}

// Seeded Kaiming-uniform init on the device (init.cuh), bit-exact to the host draw.
int ce_net_init_uniform(ce_net* net, int p, uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                        double limit) {
  Layer* lp;
  if (int s = param_layer(net, p, &lp)) return s;
  Layer& l = *lp;
  DevGuard dg(net->device);
  SharedGate gate(net->device);
  cudaStream_t st = net->st;
  InitLayout L{};
  size_t count = host_w_count(l);
  if (l.kind == CE_LAYER_CONV) {
    L.kind = 1;
    L.co = l.g.co;
    L.cin = l.c_real;
    L.k = l.g.k;
    L.cp = l.g.c;
  } else if (l.in_is_act) {
    L.kind = 2;
    L.cp = l.in_units / l.hw_in;
    L.hw = l.hw_in;
    L.in_ref = (long long)l.hw_in * l.c_real;
    L.in_dev = l.in_units;
  }
  CE_CUDA(cudaMemsetAsync(l.W, 0, l.wn * 4, st));
  const size_t nchunks = (count + kInitChunk - 1) / kInitChunk;
  kaiming_uniform_kernel<<<grid_for(nchunks, 128), 128, 0, st>>>(st_hi, st_lo, inc_hi, inc_lo, 0ull, count,
                                                                  -limit, 2.0 * limit, L, l.W);
  CE_CHECK_LAUNCH();
  CE_CUDA(cudaMemsetAsync(l.b, 0, l.bn * 4, st));
  CE_CUDA(cudaMemsetAsync(l.VW, 0, l.wn * 4, st));
  CE_CUDA(cudaMemsetAsync(l.Vb, 0, l.bn * 4, st));
  if (l.Wbf) f32_to_bf16_kernel<<<grid_for(l.wn), 256, 0, st>>>(l.W, l.wn, l.Wbf);
  if (l.Wtbf) conv_wt_kernel<<<grid_for(l.wn), 256, 0, st>>>(l.W, l.g.co, l.g.k, l.g.s, l.g.c, l.Wtbf);
  if (l.Wbp)
    f32_to_bf16_pad_kernel<<<grid_for((size_t)l.out_units * l.in_pad), 256, 0, st>>>(l.W, l.out_units, l.in_units,
                                                                                      l.in_pad, l.Wbp);
  if (l.Wp)
    pack_first_w_kernel<<<grid_for((size_t)l.g.co * l.Kp), 256, 0, st>>>(l.W, l.g.co, l.g.k, l.g.c, l.c_real, l.Kp,
                                                                         l.Wp);
  if (l.Wpf)
    pack_first_w_kernel<<<grid_for((size_t)l.g.co * l.Kp), 256, 0, st>>>(l.W, l.g.co, l.g.k, l.g.c, l.c_real, l.Kp,
                                                                         l.Wpf);
  CE_CHECK_LAUNCH();
  // no host buffers involved: the draws stay stream-ordered before the net's next
  // work (training / forward on the same stream), so no synchronisation here
  return CE_OK;
}

static int download_w(ce_net* net, const Layer& l, const float* dsrc, float* hdst) {
  cudaStream_t st = net->st;
  size_t hn = host_w_count(l);
  if (l.kind == CE_LAYER_DENSE && !l.in_is_act) {
    CE_CUDA(cudaMemcpyAsync(hdst, dsrc, hn * 4, cudaMemcpyDeviceToHost, st));
    return CE_OK;
  }
  float* tmp = nullptr;
  CE_CUDA(cudaMallocAsync(&tmp, hn * 4, st));
  if (l.kind == CE_LAYER_CONV)
    conv_w_to_host_kernel<<<grid_for(hn), 256, 0, st>>>(dsrc, l.g.co, l.c_real, l.g.c, l.g.k, tmp);
  else
    dense_w_to_host_kernel<<<grid_for(hn), 256, 0, st>>>(dsrc, l.out_units, l.c_real, l.in_units / l.hw_in, l.hw_in,
                                                          tmp);
  CE_CHECK_LAUNCH();
  CE_CUDA(cudaMemcpyAsync(hdst, tmp, hn * 4, cudaMemcpyDeviceToHost, st));
  CE_CUDA(cudaFreeAsync(tmp, st));
  return CE_OK;
}

int ce_net_get_params(ce_net* net, int p, float* w, float* b, float* vw, float* vb) {
  Layer* lp;
  if (int s = param_layer(net, p, &lp)) return s;
  DevGuard dg(net->device);
  if (w) if (int s = download_w(net, *lp, lp->W, w)) return s;
  if (vw) if (int s = download_w(net, *lp, lp->VW, vw)) return s;
  if (b) CE_CUDA(cudaMemcpyAsync(b, lp->b, lp->bn * 4, cudaMemcpyDeviceToHost, net->st));
  if (vb) CE_CUDA(cudaMemcpyAsync(vb, lp->Vb, lp->bn * 4, cudaMemcpyDeviceToHost, net->st));
  CE_CUDA(cudaStreamSynchronize(net->st));
  return CE_OK;
}

int ce_net_keep_grads(ce_net* net, int on) {
  if (check_net(net)) return CE_EINVAL;
  DevGuard dg(net->device);
  if (on)
    for (int p : net->params) {
      Layer& l = net->L[p];
      if (!l.GW) ALLOC(l.GW, l.wn * 4);
      if (!l.Gb) ALLOC(l.Gb, l.bn * 4);
    }
  net->keep_grads = on != 0;
  CE_CUDA(cudaStreamSynchronize(net->st));
  return CE_OK;
}

int ce_net_get_grads(ce_net* net, int p, float* gw, float* gb) {
  Layer* lp;
  if (int s = param_layer(net, p, &lp)) return s;
  if (!lp->GW) return fail(CE_EINVAL, "gradients are not retained; call ce_net_keep_grads first");
  DevGuard dg(net->device);
  if (gw) if (int s = download_w(net, *lp, lp->GW, gw)) return s;
  if (gb) CE_CUDA(cudaMemcpyAsync(gb, lp->Gb, lp->bn * 4, cudaMemcpyDeviceToHost, net->st));
  CE_CUDA(cudaStreamSynchronize(net->st));
  return CE_OK;
}

int ce_net_forward_host(ce_net* net, const float* x, int n, float* logits) {
  if (check_net(net)) return CE_EINVAL;
  if (n < 1 || n > net->max_batch) return fail(CE_EINVAL, "batch %d outside [1, %d]", n, net->max_batch);
  DevGuard dg(net->device);
  SharedGate gate(net->device);
  net->acc = 0;
  if (int s = upload_host_batch(net, x, n)) return s;
  if (int s = forward_any(net, n)) return s;
  g_launches += net->acc;
  if (logits)
    CE_CUDA(cudaMemcpyAsync(logits, net->L.back().out, (size_t)n * net->classes * 4, cudaMemcpyDeviceToHost, net->st));
  CE_CUDA(cudaStreamSynchronize(net->st));
  return CE_OK;
}

int ce_net_layer_materialized(const ce_net* net, int layer, int* yes) {
  if (check_net(net)) return CE_EINVAL;
  if (layer < 0 || layer >= (int)net->L.size() || !yes) return fail(CE_EINVAL, "layer %d out of range", layer);
  *yes = net->L[layer].pool_fused ? 0 : 1;
  return CE_OK;
}

int ce_net_get_activation(ce_net* net, int layer, int n, float* out) {
  if (check_net(net)) return CE_EINVAL;
  if (layer < 0 || layer >= (int)net->L.size()) return fail(CE_EINVAL, "layer %d out of range", layer);
  if (n < 1 || n > net->max_batch) return fail(CE_EINVAL, "bad n");
  DevGuard dg(net->device);
  Layer& l = net->L[layer];
  if (l.pool_fused)
    return fail(CE_EINVAL, "layer %d runs fused with the next max-pool; its output is not materialised", layer);
  cudaStream_t st = net->st;
  if (l.kind == CE_LAYER_DENSE) {
    CE_CUDA(cudaMemcpyAsync(out, l.out, (size_t)n * l.out_units * 4, cudaMemcpyDeviceToHost, st));
  } else {
    int HW = l.g.oh * l.g.ow;
    size_t total = (size_t)n * l.out_c_real * HW;
    float* tmp;
    CE_CUDA(cudaMallocAsync(&tmp, total * 4, st));
    if (net->prec == CE_PREC_FP32)
      nhwc_to_nchw_kernel<float><<<grid_for(total), 256, 0, st>>>((const float*)l.out, n, l.out_c_real, l.out_c_store,
                                                                  HW, tmp);
    else
      nhwc_to_nchw_kernel<bf16><<<grid_for(total), 256, 0, st>>>((const bf16*)l.out, n, l.out_c_real, l.out_c_store,
                                                                 HW, tmp);
    CE_CHECK_LAUNCH();
    CE_CUDA(cudaMemcpyAsync(out, tmp, total * 4, cudaMemcpyDeviceToHost, st));
    CE_CUDA(cudaFreeAsync(tmp, st));
  }
  CE_CUDA(cudaStreamSynchronize(st));
  return CE_OK;
}

int ce_net_train_batch_host(ce_net* net, const float* x, const int64_t* labels, int n, float lr, float momentum,
                            float* loss) {
  if (check_net(net)) return CE_EINVAL;
  if (n < 1 || n > net->max_batch) return fail(CE_EINVAL, "batch %d outside [1, %d]", n, net->max_batch);
  DevGuard dg(net->device);
  SharedGate gate(net->device);
  std::vector<int32_t> y(n);
  for (int i = 0; i < n; ++i) {
    if (labels[i] < 0 || labels[i] >= net->classes) return fail(CE_EINVAL, "labels must lie in [0, %d]", net->classes - 1);
    y[i] = (int32_t)labels[i];
  }
  if (int s = upload_host_batch(net, x, n)) return s;
  CE_CUDA(cudaMemcpyAsync(net->ybatch, y.data(), n * 4, cudaMemcpyHostToDevice, net->st));
  CE_CUDA(cudaMemsetAsync(net->d_step, 0, 4, net->st));
  net->acc = 0;
  if (int s = step_any(net, n, lr, momentum)) return s;
  g_launches += net->acc;
  CE_CUDA(cudaMemcpyAsync(loss, net->d_losses, 4, cudaMemcpyDeviceToHost, net->st));
  CE_CUDA(cudaStreamSynchronize(net->st));
  return CE_OK;
}

int ce_train(ce_net* net, const ce_dataset* ds, const int32_t* perm, int n_perm, int epochs, int steps_per_epoch,
               int batch, float lr, float momentum, float* losses, double* device_ms) {
  if (check_net(net)) return CE_EINVAL;
  if (!ds || !perm || epochs < 1 || steps_per_epoch < 1 || batch < 1 || batch > net->max_batch)
    return fail(CE_EINVAL, "ce_train: bad arguments");
  if (ds->c != net->in_c || ds->h != net->in_h || ds->w != net->in_w)
    return fail(CE_EINVAL, "dataset shape does not match the network input");
  if ((long long)steps_per_epoch * batch > n_perm) return fail(CE_EINVAL, "steps_per_epoch * batch exceeds n");
  DevGuard dg(net->device);
  cudaStream_t st = net->st;
  const int steps = epochs * steps_per_epoch;
  if (steps > net->losses_cap) {
    release_alloc(net, net->d_losses);
    ALLOC(net->d_losses, (size_t)steps * 4);
    net->losses_cap = steps;
  }
  size_t pn = (size_t)epochs * n_perm;
  if (pn > net->perm_cap) {
    release_alloc(net, net->d_perm);
    ALLOC(net->d_perm, pn * 4);
    net->perm_cap = pn;
  }
  CE_CUDA(cudaMemcpyAsync(net->d_perm, perm, pn * 4, cudaMemcpyHostToDevice, st));
  CE_CUDA(cudaMemsetAsync(net->d_step, 0, 8, st));
  CE_CUDA(cudaMemsetAsync(net->d_losses, 0, (size_t)steps * 4, st));
  if (!net->h_flags) {
    net->h_flags = pinned_flag_slots();
    if (!net->h_flags) return fail(CE_ENOMEM, "pinned flag pool allocation failed");
  }
  // capture one step; when profiling, every kernel class is bracketed by
  // event-record nodes inside the graph, so the per-class times are the graph's
  // own device times (no host launch gaps), read after every replay
  TrainRes r;  // graph exec + events: released on every return path
  bool graphed = false;
  net->acc = 0;
  long long per_step = 0;
  SharedGate capture_gate(net->device);  // no exclusive latency window (device sync) during a capture
  if (net->prof_on) prof_release(net);
  if (!(net->prof_on && prof_nvtx()) && cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
    cudaGraph_t graph = nullptr;
    net->prof_capturing = net->prof_on;
    int s = gather_any(net, ds, net->d_perm, n_perm, steps_per_epoch, 0, batch, true);
    if (s == CE_OK) s = step_any(net, batch, lr, momentum);
    net->prof_capturing = false;
    cudaError_t ce = cudaStreamEndCapture(st, &graph);
    if (s != CE_OK) {
      if (graph) cudaGraphDestroy(graph);
      prof_release(net);
      return s;
    }
    if (ce == cudaSuccess && cudaGraphInstantiate(&r.exec, graph, 0) == cudaSuccess) graphed = true;
    if (graph) cudaGraphDestroy(graph);
    per_step = net->acc;
  }
  capture_gate.release();
  cudaGetLastError();
  if (net->prof_on && getenv("CE_PROF_DEBUG"))
    fprintf(stderr, "[ce_train profile] graphed=%d bracketed launches per step=%zu\n", (int)graphed,
            net->prof_pending.size());
  if (!graphed) prof_release(net);  // eager fallback: fresh events per launch
  net->acc = 0;
  CE_CUDA(cudaEventCreate(&r.ev[0]));
  CE_CUDA(cudaEventCreate(&r.ev[1]));
  CE_CUDA(cudaEventCreateWithFlags(&r.ev[2], cudaEventDisableTiming));
  CE_CUDA(cudaEventCreateWithFlags(&r.ev[3], cudaEventDisableTiming));
  cudaEvent_t e0 = r.ev[0], e1 = r.ev[1], *chunk_ev = r.ev + 2;
  r.owner = st;
  CE_CUDA(cudaEventRecord(e0, st));
  // Replay in chunks; after each chunk snapshot the device non-finite flag. With
  // one chunk in flight ahead, a diverged candidate stops within two chunks
  // (the reference stops at the first non-finite loss, evaluator.py:168-170).
  const int chunk = 16;
  int launched = 0, nchunk = 0;
  struct InTrain {  // NVTX class ranges of the eager profiling pass: this loop's steps only
    ce_net* n;
    explicit InTrain(ce_net* x) : n(x) { n->prof_in_train = true; }
    ~InTrain() { n->prof_in_train = false; }
  } in_train(net);
  while (launched < steps) {
    const int todo = std::min(chunk, steps - launched);
    {
      SharedGate gate(net->device);  // enqueue under the gate; ce_latency drains in-flight chunks
      for (int i = 0; i < todo; ++i) {
        if (graphed) {
          CE_CUDA(cudaGraphLaunch(r.exec, st));
          if (net->prof_on && !net->prof_pending.empty()) {  // read this replay's event nodes
            CE_CUDA(cudaStreamSynchronize(st));
            prof_collect(net, true);
          }
        } else {
          if (int s = gather_any(net, ds, net->d_perm, n_perm, steps_per_epoch, 0, batch, true)) return s;
          if (int s = step_any(net, batch, lr, momentum)) return s;
        }
      }
    }
    launched += todo;
    const int slot = nchunk & 1;
    CE_CUDA(cudaMemcpyAsync(net->h_flags + slot, net->d_step + 1, 4, cudaMemcpyDeviceToHost, st));
    CE_CUDA(cudaEventRecord(chunk_ev[slot], st));
    if (nchunk >= 1) {
      CE_CUDA(cudaEventSynchronize(chunk_ev[slot ^ 1]));
      if (net->h_flags[slot ^ 1]) break;
    }
    ++nchunk;
  }
  g_launches += graphed ? per_step * launched : net->acc;
  CE_CUDA(cudaEventRecord(e1, st));
  CE_CUDA(cudaMemcpyAsync(losses, net->d_losses, (size_t)steps * 4, cudaMemcpyDeviceToHost, st));
  cudaError_t se = cudaStreamSynchronize(st);
  if (net->prof_on) {
    if (graphed) {  // every replay was collected already; the graph goes before its events
      cudaGraphExecDestroy(r.exec);
      r.exec = nullptr;
      prof_release(net);
    } else {
      prof_collect(net);
    }
  }
  if (se != cudaSuccess) return fail(CE_ECUDA, "train loop: %s", cudaGetErrorString(se));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (device_ms) *device_ms = ms;
  return CE_OK;
}

int ce_predict(ce_net* net, const ce_dataset* ds, int batch, double* scores, int64_t* preds) {
  if (check_net(net)) return CE_EINVAL;
  if (!ds || batch < 1 || batch > net->max_batch) return fail(CE_EINVAL, "ce_predict: bad arguments");
  DevGuard dg(net->device);
  SharedGate gate(net->device);
  cudaStream_t st = net->st;
  if ((size_t)ds->n > net->pred_cap) {
    release_alloc(net, net->d_scores);
    release_alloc(net, net->d_preds);
    ALLOC(net->d_scores, (size_t)ds->n * 8);
    ALLOC(net->d_preds, (size_t)ds->n * 8);
    net->pred_cap = ds->n;
  }
  net->acc = 0;
  for (int start = 0; start < ds->n; start += batch) {
    int nb = std::min(batch, ds->n - start);
    if (int s = gather_any(net, ds, nullptr, 0, 1, start, nb, false)) return s;
    if (int s = forward_any(net, nb)) return s;
    net->acc += 1;
    predict_head_kernel<<<cdiv(nb, 128), 128, 0, st>>>((const float*)net->L.back().out, nb, net->classes, start,
                                                        net->d_scores, net->d_preds);
    CE_CHECK_LAUNCH();
  }
  g_launches += net->acc;
  CE_CUDA(cudaMemcpyAsync(scores, net->d_scores, (size_t)ds->n * 8, cudaMemcpyDeviceToHost, st));
  CE_CUDA(cudaMemcpyAsync(preds, net->d_preds, (size_t)ds->n * 8, cudaMemcpyDeviceToHost, st));
  CE_CUDA(cudaStreamSynchronize(st));
  return CE_OK;
}

namespace {
// RAII for the streaming resources of ce_predict_stream
struct StreamRes {
  cudaStream_t cs = nullptr;
  cudaEvent_t ev[6] = {};
  uint8_t* stage[2] = {};
  cudaStream_t owner = nullptr;
  const void* registered = nullptr;
  ~StreamRes() {
    if (owner) {
      cudaStreamSynchronize(owner);
      for (auto* p : stage)
        if (p) cudaFreeAsync(p, owner);
    }
    if (cs) {
      cudaStreamSynchronize(cs);
      cudaStreamDestroy(cs);
    }
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (registered) cudaHostUnregister(const_cast<void*>(registered));
  }
};
}  // namespace

int ce_predict_stream(ce_net* net, const uint8_t* pixels, long long count, int batch, double* scores, int64_t* preds,
                      double* seconds) {
  if (check_net(net)) return CE_EINVAL;
  if (!pixels || count < 1 || batch < 1 || batch > net->max_batch || !scores || !preds)
    return fail(CE_EINVAL, "ce_predict_stream: bad arguments");
  DevGuard dg(net->device);
  SharedGate gate(net->device);
  cudaStream_t st = net->st;
  const int HW = net->in_h * net->in_w;
  const size_t img = (size_t)net->in_c * HW;
  const size_t total_bytes = img * (size_t)count;
  if ((size_t)count > net->pred_cap) {
    release_alloc(net, net->d_scores);
    release_alloc(net, net->d_preds);
    ALLOC(net->d_scores, (size_t)count * 8);
    ALLOC(net->d_preds, (size_t)count * 8);
    net->pred_cap = count;
  }
  StreamRes r;
  // pageable input is page-locked for the duration so the copies are truly async
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, pixels) != cudaSuccess || attr.type == cudaMemoryTypeUnregistered) {
    cudaGetLastError();
    CE_CUDA(cudaHostRegister(const_cast<uint8_t*>(pixels), total_bytes, cudaHostRegisterReadOnly));
    r.registered = pixels;
  }
  CE_CUDA(cudaStreamCreateWithFlags(&r.cs, cudaStreamNonBlocking));
  for (auto& e : r.ev) CE_CUDA(cudaEventCreate(&e));
  cudaEvent_t *copied = r.ev, *consumed = r.ev + 2, t0 = r.ev[4], t1 = r.ev[5];
  r.owner = st;
  for (auto& p : r.stage) CE_CUDA(cudaMallocAsync((void**)&p, img * batch, st));
  CE_CUDA(cudaEventRecord(t0, st));
  CE_CUDA(cudaStreamWaitEvent(r.cs, t0, 0));  // staging exists, timing starts
  net->acc = 0;
  const long long chunks = (count + batch - 1) / batch;
  for (long long i = 0; i < chunks; ++i) {
    const int b = (int)(i & 1);
    const long long start = i * batch;
    const int nb = (int)std::min<long long>(batch, count - start);
    if (i >= 2) CE_CUDA(cudaStreamWaitEvent(r.cs, consumed[b], 0));  // gather of chunk i-2 done
    CE_CUDA(cudaMemcpyAsync(r.stage[b], pixels + (size_t)start * img, img * nb, cudaMemcpyHostToDevice, r.cs));
    CE_CUDA(cudaEventRecord(copied[b], r.cs));
    CE_CUDA(cudaStreamWaitEvent(st, copied[b], 0));
    dim3 grid = gather_grid(HW, nb);
    if (net->prec == CE_PREC_FP32)
      gather_u8_kernel<float><<<grid, 256, 0, st>>>(r.stage[b], nullptr, nullptr, nullptr, 0, 0, 0, nb, net->in_c,
                                                    net->in_cp, HW, (float*)net->x0, nullptr);
    else
      gather_u8_kernel<bf16><<<grid, 256, 0, st>>>(r.stage[b], nullptr, nullptr, nullptr, 0, 0, 0, nb, net->in_c,
                                                   net->in_cp, HW, (bf16*)net->x0, nullptr);
    CE_CHECK_LAUNCH();
    CE_CUDA(cudaEventRecord(consumed[b], st));  // the copy of chunk i+2 may now overwrite this buffer
    if (int s = forward_any(net, nb)) return s;
    predict_head_kernel<<<cdiv(nb, 128), 128, 0, st>>>((const float*)net->L.back().out, nb, net->classes, (int)start,
                                                        net->d_scores, net->d_preds);
    CE_CHECK_LAUNCH();
    net->acc += 2;
  }
  g_launches += net->acc;
  CE_CUDA(cudaMemcpyAsync(scores, net->d_scores, (size_t)count * 8, cudaMemcpyDeviceToHost, st));
  CE_CUDA(cudaMemcpyAsync(preds, net->d_preds, (size_t)count * 8, cudaMemcpyDeviceToHost, st));
  CE_CUDA(cudaEventRecord(t1, st));
  CE_CUDA(cudaEventSynchronize(t1));
  float ms = 0.f;
  CE_CUDA(cudaEventElapsedTime(&ms, t0, t1));
  if (seconds) *seconds = ms * 1e-3;
  return CE_OK;
}

int ce_latency(ce_net* net, const float* x, int n, int warmup, int reps, double* seconds) {
  if (check_net(net)) return CE_EINVAL;
  if (n < 1 || n > net->max_batch || warmup < 0 || reps < 1) return fail(CE_EINVAL, "ce_latency: bad arguments");
  DevGuard dg(net->device);
  // exclusive per-GPU window: no other slot enqueues while we hold the gate, and
  // what they already enqueued drains before the first timed forward
  static const bool shared_window = [] {  // CE_LATENCY_SHARED=1: no exclusive window (comparison only)
    const char* e = getenv("CE_LATENCY_SHARED");
    return e && e[0] == '1';
  }();
  ExclusiveGate gate(shared_window ? -1 : net->device);
  if (!shared_window) CE_CUDA(cudaDeviceSynchronize());
  cudaStream_t st = net->st;
  net->acc = 0;
  if (int s = upload_host_batch(net, x, n)) return s;
  for (int i = 0; i < warmup; ++i)
    if (int s = forward_any(net, n)) return s;
  std::vector<cudaEvent_t> ev(2 * reps);
  for (auto& e : ev) CE_CUDA(cudaEventCreate(&e));
  for (int r = 0; r < reps; ++r) {
    CE_CUDA(cudaEventRecord(ev[2 * r], st));
    if (int s = forward_any(net, n)) return s;
    CE_CUDA(cudaEventRecord(ev[2 * r + 1], st));
  }
  g_launches += net->acc;
  CE_CUDA(cudaStreamSynchronize(st));
  for (int r = 0; r < reps; ++r) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[2 * r], ev[2 * r + 1]);
    seconds[r] = ms * 1e-3;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return CE_OK;
}

}  // extern "C"
