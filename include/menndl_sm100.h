/*
 * menndl_sm100.h — C ABI of libmenndl_sm100.so, the B200 (sm_100a) candidate
 * evaluation library behind paper_1909_12291_b200.
 *
 * The reference (convevo, pure Python + numpy) has no native boundary; the
 * surfaces this ABI replaces are its Python operator / candidate interfaces:
 *
 *   ce_net_create + ce_net_set_params   <- genome.instantiate        (genome.py:309-335)
 *                                          + nn._kaiming_uniform init (nn.py:44-46)
 *   ce_train                            <- evaluator.train_short     (evaluator.py:145-171)
 *                                          looping nn.train_batch    (nn.py:325-331)
 *   ce_net_train_batch_host             <- nn.train_batch            (nn.py:325-331)
 *   ce_net_forward_host                 <- nn.Network.forward        (nn.py:264-272)
 *   ce_net_get_activation               <- per-layer outputs of Conv2d/ReLU/MaxPool/Dense.forward
 *                                          (nn.py:82-94, 140-150, 178-180, 225-231)
 *   ce_net_get_grads                    <- Layer.grads after Network.backward (nn.py:96-116, 233-240)
 *   ce_net_get_params                   <- Layer.params / Layer._vel after sgd_step (nn.py:306-322)
 *   ce_predict                          <- evaluator.predict_scores  (evaluator.py:174-186)
 *   ce_latency                          <- evaluator.measure_latency (evaluator.py:189-210)
 *   ce_predict_stream                   <- predict_scores over a streamed slide + metrics.slide_seconds
 *                                          (evaluator.py:174-186, metrics.py:77-81)
 *   ce_dataset_create                   <- data.PatchSet.as_float    (data.py:65-66), uploaded once
 *
 * Kernel level (operator drop-in, paper_1909_12291_b200/nn.py):
 *   ce_conv_fwd / ce_conv_wgrad / ce_conv_dgrad  <- Conv2d.forward / backward (nn.py:82-116)
 *   ce_maxpool_fwd / ce_maxpool_bwd              <- MaxPool.forward / backward (nn.py:140-167)
 *   ce_dense_fwd / ce_dense_bwd                  <- Dense.forward / backward   (nn.py:225-240)
 *   ce_relu_fwd / ce_relu_bwd                    <- ReLU.forward / backward    (nn.py:170-183)
 *   ce_softmax_xent                              <- softmax_cross_entropy      (nn.py:287-303)
 *   ce_sgd_momentum                              <- sgd_step, per tensor       (nn.py:306-322)
 *   ce_pcg64_uniform                             <- _kaiming_uniform draws     (nn.py:44-46)
 *   ce_gather_u8_normalize                       <- PatchSet.as_float + x[idx] (data.py:65-66, evaluator.py:166)
 *   ce_permute_flatten_weights                   <- Flatten column order       (nn.py:186-202)
 *
 * Conventions
 *   - Every entry point returns a status (CE_OK ... CE_ECUDA); the message of
 *     the last failure on the calling thread is available from ce_last_error().
 *     Python maps CE_EINVAL -> ShapeError/ValueError, everything else ->
 *     EvalFailure (errors.py:4-26), so no exception escapes evaluate().
 *   - Host pointers are never retained after a call returns. A ce_net owns its
 *     device buffers; one ce_net is used by one thread at a time; distinct nets
 *     may be driven concurrently from different threads (different streams).
 *   - Host-side tensors use the reference layouts: activations NCHW float32,
 *     conv weights (out, in, kh, kw), dense weights (out, in) with the flatten
 *     order (c, h, w) of nn.Flatten (nn.py:197-199). Device layouts are NHWC
 *     and are converted inside the library.
 */
#ifndef MENNDL_SM100_H
#define MENNDL_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define CE_OK 0
#define CE_EINVAL 1     /* bad argument / shape            -> ShapeError / ValueError */
#define CE_ENONFINITE 2 /* non-finite loss                 -> EvalFailure             */
#define CE_ENOMEM 3     /* device allocation failed        -> EvalFailure             */
#define CE_ECUDA 4      /* CUDA launch / runtime failure   -> EvalFailure (+ GPU unhealthy if sticky) */

/* precision of activations and conv/dense operands */
#define CE_PREC_BF16 0 /* bf16 operands, fp32 accumulate, fp32 master weights (tcgen05 path) */
#define CE_PREC_FP32 1 /* fp32 check mode (CUDA-core FFMA)                                   */

/* layer kinds of a network descriptor (ReLU is a flag on conv, Flatten is implicit) */
#define CE_LAYER_CONV 1
#define CE_LAYER_POOL 2
#define CE_LAYER_DENSE 3

typedef struct ce_layer_desc {
  int kind;         /* CE_LAYER_*                                    */
  int out_channels; /* conv                                          */
  int kernel;       /* conv kernel / pool window                     */
  int stride;       /* conv / pool stride                            */
  int relu;         /* conv: ReLU follows (genome.py:322-323)        */
  int units;        /* dense output units                            */
} ce_layer_desc;

typedef struct ce_net_desc {
  int in_c, in_h, in_w;        /* per-sample input shape (3, 100, 100)          */
  int n_layers;                /* feature layers, then dense layers (last = classes) */
  const ce_layer_desc* layers;
  int max_batch;               /* largest batch the net will see               */
} ce_net_desc;

typedef struct ce_net ce_net;
typedef struct ce_dataset ce_dataset;

int ce_version(void);
const char* ce_last_error(void);
int ce_device_count(int* count);

/* ---- datasets: u8 NCHW pixels + u8 labels, uploaded once per device ------ */
int ce_dataset_create(int device, const uint8_t* pixels, const uint8_t* labels, int n, int c, int h, int w,
                      ce_dataset** out);
int ce_dataset_destroy(ce_dataset* ds);

/* ---- networks ------------------------------------------------------------- */
int ce_net_create(const ce_net_desc* desc, int device, int precision, ce_net** out);
int ce_net_destroy(ce_net* net);
/* bytes of device memory the net holds (parameters + activations + workspace) */
int ce_net_device_bytes(const ce_net* net, size_t* bytes);
/* stream priority of the net's work: > 0 the device's highest, otherwise default */
int ce_net_set_priority(ce_net* net, int priority);
/* number of parameterised layers (conv + dense), in layer order */
int ce_net_num_param_layers(const ce_net* net, int* count);
/* param layer p: weights in reference layout (conv (o,c,kh,kw), dense (o,in)), bias (o) */
int ce_net_set_params(ce_net* net, int p, const float* w, const float* b);
int ce_net_get_params(ce_net* net, int p, float* w, float* b, float* vel_w, float* vel_b);
/* param layer p: Kaiming-uniform U(-limit, limit) weights drawn on the device from the
 * numpy PCG64 stream whose 128-bit state / increment are given (the state the
 * reference's default_rng(seed) has when it reaches this layer, genome.py:313,
 * nn.py:44-46); bit-exact to the host draw. Zero bias and velocities.           */
int ce_net_init_uniform(ce_net* net, int p, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                        uint64_t inc_lo, double limit);
/* retain raw parameter gradients of the next steps for ce_net_get_grads (off by default) */
int ce_net_keep_grads(ce_net* net, int on);
int ce_net_get_grads(ce_net* net, int p, float* gw, float* gb);

/* inference forward of n samples (float32 NCHW host) -> logits (n, classes) */
int ce_net_forward_host(ce_net* net, const float* x, int n, float* logits);
/* output of layer `layer` (descriptor index) from the last forward, NCHW / (n, units) float32;
 * CE_EINVAL for a conv whose max-pool runs in its epilogue (not materialised) */
int ce_net_get_activation(ce_net* net, int layer, int n, float* out);
/* *yes = 0 when layer `layer` is a conv fused with the following max-pool (bf16, non-overlapping window) */
int ce_net_layer_materialized(const ce_net* net, int layer, int* yes);
/* one SGD step on a host batch; writes the pre-step mean loss */
int ce_net_train_batch_host(ce_net* net, const float* x, const int64_t* labels, int n, float lr, float momentum,
                            float* loss);

/* train_short: `epochs` x `steps_per_epoch` steps of `batch` samples; perm is
 * epochs x n_perm int32 (one numpy permutation of the n_perm training patches
 * per epoch, evaluator.py:161); step b of an epoch uses perm[b*batch:(b+1)*batch]
 * (evaluator.py:139-142). losses receives one pre-step loss per step (the
 * caller raises EvalFailure at the first non-finite one, evaluator.py:168-170);
 * device_ms receives the device time of the loop.                            */
int ce_train(ce_net* net, const ce_dataset* train, const int32_t* perm, int n_perm, int epochs,
             int steps_per_epoch, int batch, float lr, float momentum, float* losses, double* device_ms);
/* predict_scores: softmax p[:,1] and argmax over the whole set in chunks of `batch` */
int ce_predict(ce_net* net, const ce_dataset* set, int batch, double* scores, int64_t* preds);
/* Streamed whole-slide inference: predict_scores (evaluator.py:174-186) over
 * `count` u8 NCHW patches in HOST memory (pinned for full overlap; pageable
 * input is page-locked for the call), copied in chunks of `batch` on a copy
 * stream double-buffered against gather + forward + softmax head. scores
 * (p[:,1]) / preds (argmax) go to host arrays of `count`; *seconds = device
 * time from the first copy to the results on the host side of the last D2H
 * (the prediction rate of metrics.py:77-81 is count / seconds).             */
int ce_predict_stream(ce_net* net, const uint8_t* pixels, long long count, int batch, double* scores, int64_t* preds,
                      double* seconds);
/* measure_latency: warmup + reps device-timed forwards of a host batch (float32 NCHW) */
int ce_latency(ce_net* net, const float* x, int n, int warmup, int reps, double* seconds);

/* ---- kernel level: single passes on caller-owned device tensors (NHWC) ------
 * Replaces Conv2d.forward / Conv2d.backward / MaxPool.forward / MaxPool.backward
 * (nn.py:82-116, 140-167) for one layer. bf16: x/y/dy/dx/w are bf16, conv
 * weights [c_out][kh][kw][c] (tensor-core path); fp32: all float32 (FFMA path).
 * Gradients dw/db are always float32. `stream` is a cudaStream_t (may be 0).  */
typedef struct ce_conv_desc {
  int n, c, h, w;   /* input batch and NHWC geometry (c = stored channels)    */
  int c_out;        /* conv output channels (ignored by pool)                 */
  int kernel;       /* conv kernel / pool window                              */
  int stride;
  int precision;    /* CE_PREC_*                                              */
} ce_conv_desc;

size_t ce_conv_workspace_bytes(const ce_conv_desc* d);
/* y = conv(x, w) + bias, ReLU if relu (nn.py:82-94, 178-180).
 * pool_k > 0: max-pool epilogue (MaxPool.forward, nn.py:140-150) for a
 * non-overlapping window (pool_k in {2, 3}, pool_s >= pool_k; bf16 only): y is
 * the POOLED map [n][ph][pw][c_out] and arg its u8 argmax (row-major first
 * max; 0xFF = dead window when relu), the pre-pool map is never written.      */
int ce_conv_fwd(const ce_conv_desc* d, const void* x, const void* w, const float* bias, int relu, int pool_k,
                int pool_s, void* y, uint8_t* arg, void* stream);
/* dx = conv^T(dy, w), optionally gated by (mask > 0) -- the ReLU backward of the
 * layer that produced the conv input (nn.py:182-183)                          */
int ce_conv_dgrad(const ce_conv_desc* d, const void* dy, const void* w, const void* mask, void* dx, void* workspace,
                  size_t ws_bytes, void* stream);
int ce_conv_wgrad(const ce_conv_desc* d, const void* x, const void* dy, float* dw, float* db, void* workspace,
                  size_t ws_bytes, void* stream);
int ce_maxpool_fwd(const ce_conv_desc* d, const void* x, void* y, uint8_t* arg, void* stream);
int ce_maxpool_bwd(const ce_conv_desc* d, const void* dy, const uint8_t* arg, const void* mask, void* dx,
                   void* stream);

/* Batch gather + normalise (data.py:65-66 as_float, evaluator.py:166 x[idx]):
 * out[b] = pixels[idx[b]] / 255 for b < n. pixels: device u8 NCHW (count, c, h, w);
 * idx: device int32; out: NHWC with channels zero-padded to c_store (>= c),
 * bf16 or float32 by `precision`.                                               */
int ce_gather_u8_normalize(const uint8_t* pixels, int c, int h, int w, const int32_t* idx, int n, int c_store,
                           int precision, void* out, void* stream);

/* Dense layer passes (replaces Dense.forward / Dense.backward, nn.py:225-240).
 * fp32: x [n][in] float32, w [out][in] float32 master (the FFMA path).
 * bf16: x [n][in_pad] bf16 and w16 [out][in_pad] bf16 mirror of w, in_pad = in
 *       rounded up to 8 with zero columns (tensor-core path); w is still the
 *       float32 master (read by the fused SGD).
 * y / dy / dw / db are float32. dx and mask have the activation type (bf16 in
 * bf16 mode, laid out [n][in] -- no padding -- ; float32 otherwise).          */
typedef struct ce_dense_desc {
  int n;          /* batch rows (bf16: <= 256)                                 */
  int in, out;    /* units                                                    */
  int precision;  /* CE_PREC_*                                                */
} ce_dense_desc;

/* Momentum SGD fused into a gradient pass (sgd_step, nn.py:306-322):
 * v <- momentum*v - lr*g ; w <- w + v, in fp32 without contraction.          */
typedef struct ce_sgd_args {
  float lr, momentum;
  float* vel_w;  /* velocity of w (same layout as w), updated in place          */
  float* vel_b;  /* velocity of b                                               */
} ce_sgd_args;

size_t ce_dense_workspace_bytes(const ce_dense_desc* d);
/* y = x @ w^T + b                                                              */
int ce_dense_fwd(const ce_dense_desc* d, const void* x, const float* w, const void* w16, const float* b, float* y,
                 void* workspace, size_t ws_bytes, void* stream);
/* dx = dy @ w (pre-update weights; optional, skipped when dx is NULL), gated by
 * (mask > 0) when mask is given; dw = dy^T x and db = sum_n dy (each optional).
 * With sgd != NULL, w / b (and w16 in bf16 mode) are updated in place after dx. */
int ce_dense_bwd(const ce_dense_desc* d, const void* x, const float* dy, float* w, void* w16, float* b, void* dx,
                 const void* mask, float* dw, float* db, const ce_sgd_args* sgd, void* workspace, size_t ws_bytes,
                 void* stream);

/* softmax_cross_entropy (nn.py:287-303) on device float32 logits [n][k], int64
 * labels: *loss (device float) = -mean(logp[label]), grad = (softmax - onehot)/n.
 * n <= 1024. Labels outside [0, k) make the loss NaN (the host mirror raises
 * ValueError before calling, as the reference does).                           */
int ce_softmax_xent(const float* logits, const int64_t* labels, int n, int k, float* loss, float* grad, void* stream);

/* sgd_step on one parameter tensor (nn.py:306-322), bit-exact fp32:
 * vel <- momentum*vel - lr*g ; w <- w + vel. lr > 0 and 0 <= momentum < 1
 * (nn.py:308-311) else CE_EINVAL.                                              */
int ce_sgd_momentum(float* w, float* vel, const float* g, size_t count, float lr, float momentum, void* stream);

/* ReLU (nn.py:170-183) on `count` contiguous elements (bf16 or float32 by precision):
 * y = x > 0 ? x : 0, mask[i] = (x[i] > 0) as u8 (mask may be NULL); backward
 * dx = mask ? dy : 0. Pointers 16-byte aligned.                                */
int ce_relu_fwd(const void* x, size_t count, int precision, void* y, uint8_t* mask, void* stream);
int ce_relu_bwd(const void* dy, const uint8_t* mask, size_t count, int precision, void* dx, void* stream);

/* numpy Generator(PCG64(state, inc)) advanced by `skip` draws, then
 * .uniform(low, high, size=count).astype(float32) (nn.py:44-46), bit-exact.    */
int ce_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, uint64_t skip,
                     double low, double high, float* out, size_t count, void* stream);

/* Dense columns between the reference flatten order (c, h, w) (nn.py:186-202)
 * and the device NHWC order (h, w, c_store), padded channels zero.
 * direction 0: src [rows][c*hw] -> dst [rows][hw*c_store]; 1: the inverse.     */
int ce_permute_flatten_weights(const float* src, size_t rows, int c, int c_store, int hw, int direction, float* dst,
                               void* stream);

/* ---- instrumentation (bench.py) ------------------------------------------- */
/* kernels this process has launched through the library (graph replays count every node) */
long long ce_launch_count(void);
/* per-kernel-class CUDA-event timing of ce_train (steps run un-graphed while enabled) */
int ce_prof_num_classes(void);
int ce_net_set_profiling(ce_net* net, int on);
int ce_net_prof_read(ce_net* net, int cls, const char** name, long long* launches, double* ms, double* flops,
                     double* bytes);
/* roofline time of a class: sum over its launches of max(flops / P, bytes / BW), P and BW set process-wide by
 * ce_prof_set_peaks (bench.py passes MEASURED_PEAKS.json's sustained bf16 FLOP/s and HBM bytes/s) */
int ce_prof_set_peaks(double flops_per_s, double bytes_per_s);
int ce_net_prof_ideal(ce_net* net, int cls, double* ideal_ms);
/* the same totals for one layer (descriptor index; -1 = batch gather and stand-alone loss) */
int ce_net_prof_layer(ce_net* net, int layer, int cls, long long* launches, double* ms, double* flops, double* bytes,
                      double* ideal_ms);

#ifdef __cplusplus
}
#endif
#endif /* MENNDL_SM100_H */
