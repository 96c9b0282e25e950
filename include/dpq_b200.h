/* dpq_b200 — C-ABI of the B200-native DP-LLM decode hot path.
 *
 * The reference (`dpq`, /root/reference/pkg/src/dpq) is pure Python + numpy;
 * its operator boundary for this path is the Python API listed next to each
 * entry point ("replaces ..."). The Python package `paper_2508_06041_b200`
 * binds these symbols with ctypes (see INTEGRATION.md for the stub a `dpq`
 * maintainer would add). Plain pointers and sizes only; every function
 * returns 0 on success or a negative status, with the message available from
 * dpq_last_error() (thread-local). Nothing throws across the ABI.
 *
 * Pointers suffixed _dev are device pointers on the handle's device; _host
 * are host pointers. `stream` is a cudaStream_t passed as void* (0 = legacy
 * default stream).
 */
#ifndef DPQ_B200_H
#define DPQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPQ_OK 0
#define DPQ_ERR_ARG -1      /* bad argument (QuantError / ValueError class)   */
#define DPQ_ERR_CUDA -2     /* CUDA runtime error                             */
#define DPQ_ERR_STATE -3    /* handle misuse (e.g. sequence cap exceeded)     */
#define DPQ_ERR_RANGE -4    /* engine fixed-point accumulator range exceeded  */

typedef struct dpq_store dpq_store;
typedef struct dpq_plan dpq_plan;
typedef struct dpq_session dpq_session;

/* One quantized layer (reference QuantizedLayer, quant.py:27-40). Codes are
 * row-major rows*cols, uint16 (code_bytes=2) or uint8 (code_bytes=1), each
 * < 2^n_bits, or (code_bytes=0) the .dpqs file's packed code stream as it lies
 * on disk: code-major, LSB-first, n_bits per code, ceil(rows*cols*n_bits/8)
 * bytes (reference pack_codes, quant.py:123-126) -- repacked into bitplanes on
 * the device, never unpacked on the host. codes_on_device selects host or
 * device memory for `codes`. */
typedef struct {
  int32_t rows, cols, n_bits, b_min;
  int32_t code_bytes;
  int32_t codes_on_device;
  const void* codes;
  const float* lo;        /* host, [rows] */
  const float* hi;        /* host, [rows] */
} dpq_layer_desc;

/* Selector parameters of one layer (reference PlanLayer + ErrorEstimator,
 * runtime.py:30-43, estimator.py:35-83). */
typedef struct {
  int32_t l, h, prefill_bit;
  int32_t est_kind;       /* 0 none, 1 linear, 2 projection, 3 exact          */
  int32_t prev_residual;  /* input_source == "previous_residual"              */
  int32_t k;              /* projection rank (rows of G)                      */
  int32_t g_dtype;        /* device copy of G: 0 f32, 1 f16, 2 e4m3+row scale */
  int32_t fx_bits_plus128; /* 0: fixed-point fraction bits of the engine's G.x
                             words derived from G; else 128 + those bits (tensor
                             parallel shards of G: the full layer's value)     */
  double T;               /* threshold; +/-INFINITY are the sentinels         */
  double slope, intercept;
  const double* G;        /* host, [k][cols] row-major (projection)           */
} dpq_sel_desc;

/* Model description for a decode session (reference ModelConfig +
 * ModelWeights embed/lm_head, model.py:45-110). Store layer index of
 * (block b, kind k in q,k,v,o,up,gate,down order) is 7*b + k. */
typedef struct {
  int32_t n_blocks, d_model, n_heads, n_kv_heads, d_ff, vocab, seq_cap;
  float norm_eps;
  const float* embed;     /* host, [vocab][d_model] */
  const float* lm_head;   /* host, [vocab][d_model] */
  int32_t track_exact;    /* DecodeEngine(track_exact=...)                    */
  int32_t async_prev_block; /* async_rule == "prev_block"                      */
  int32_t prime_from_prefill;
  int32_t use_graph;      /* capture the step into a CUDA graph               */
  int32_t use_pdl;        /* programmatic dependent launch between kernels    */
  int32_t use_persistent; /* one persistent step kernel (flag-linked stages)  */
} dpq_model_desc;

const char* dpq_last_error(void);
int dpq_version(void);
/* SM count and whether a usable sm_100 device is present. */
int dpq_device_info(int device, int* n_sm, int* cc_major, int* cc_minor);

/* ---- store: replaces quant.BitPlaneStore / QuantizedLayer (quant.py:27-40,
 *      102-110); codes are repacked into MSB-first device bitplanes. ------- */
int dpq_store_create(int device, int n_layers, const dpq_layer_desc* layers, dpq_store** out);
int dpq_store_destroy(dpq_store* s);
/* Streaming build of a large store: dpq_store_create with n_layers = 0, then
 * layers appended in canonical order (each repacked on the device as it
 * arrives, so the caller can free its codes before the next layer). */
int dpq_store_append(dpq_store* s, int n_layers, const dpq_layer_desc* layers);
/* Algorithmic bytes of the selected planes + (lo, span) for one GEMV at b. */
int dpq_store_layer_bytes(const dpq_store* s, int layer, int b, int64_t* bytes);

/* quant.quantize_layer (quant.py:43-64) on the device, float64 semantics:
 * W_dev float32 [rows][cols] -> codes_dev uint16, lo_dev/hi_dev float32. */
int dpq_quantize_device(int device, const float* W_dev, int rows, int cols, int n_bits,
                        uint16_t* codes_dev, float* lo_dev, float* hi_dev, void* stream);

/* quant.gemv (quant.py:95-99): y = W_b x, reading only planes 0..b-1.
 * Calls on one store share its scratch (tile counters, window partials,
 * estimator sums): issue them on one stream (or order the streams). The
 * launch uses programmatic dependent launch: the next call on the stream may
 * start streaming its weights while this one drains. */
int dpq_gemv(dpq_store* s, int layer, int b, const float* x_dev, float* y_dev, void* stream);
/* quant.dequantize (quant.py:67-80): float64 [rows][cols]. */
int dpq_dequantize(dpq_store* s, int layer, int b, double* out_dev, void* stream);

/* ---- plan: replaces runtime.PrecisionPlan selector state ---------------- */
int dpq_plan_create(dpq_store* s, int n_layers, const dpq_sel_desc* sels, dpq_plan** out);
int dpq_plan_destroy(dpq_plan* p);

/* runtime.select_precision (runtime.py:184-193) fused into the GEMV prologue:
 * the estimate, the threshold compare and the selected-bit GEMV run in one
 * kernel; bit_out_dev (int32) / est_out_dev (float32, NaN if none) receive the
 * decision. est_in_dev: estimator input when it differs from x (async), or
 * NULL. exact_out_dev (nullable): ||(W_h - W_l) x|| (track_exact). Same
 * stream rule as dpq_gemv (the plan's store scratch). */
int dpq_select_gemv(dpq_plan* p, int layer, const float* x_dev, const float* est_in_dev,
                    float* y_dev, int32_t* bit_out_dev, float* est_out_dev,
                    float* exact_out_dev, void* stream);

/* ErrorEstimator.estimate (estimator.py:82-83) for linear / projection
 * estimators on the device: est_out_host = slope*||x||+b or ||G x||. */
typedef struct dpq_estimator dpq_estimator;
int dpq_estimator_create(int device, const dpq_sel_desc* sel, int cols, dpq_estimator** out);
int dpq_estimator_eval(dpq_estimator* e, const float* x_dev, double* est_out_host, void* stream);
int dpq_estimator_destroy(dpq_estimator* e);
/* estimator.exact_error (estimator.py:30-32): ||(W_h - W_l) x|| from the
 * shared plane sums (one pass over h planes). */
int dpq_exact_error(dpq_store* s, int layer, int l, int h, const float* x_dev, double* out_host,
                    void* stream);

/* ---- session: replaces runtime.DecodeEngine (runtime.py:245-390) -------- */
int dpq_session_create(dpq_store* s, dpq_plan* p, const dpq_model_desc* m, dpq_session** out);
int dpq_session_destroy(dpq_session* ss);
int dpq_session_reset(dpq_session* ss);
/* One DecodeEngine.step(token, dynamic). logits_host (nullable) receives
 * float32 [vocab] (synchronises). forced_bits (nullable, int8 [n_layers])
 * replays recorded decisions (parity after a threshold tie). */
int dpq_session_step(dpq_session* ss, int token, int dynamic, const int8_t* forced_bits,
                     float* logits_host);
/* Greedy decode on the device: n_new dynamic steps starting from the argmax
 * of the last logits; tokens_host receives the generated tokens. No host
 * round trip per token. */
int dpq_session_decode(dpq_session* ss, int n_new, int32_t* tokens_host);
/* Enqueue `n` greedy dynamic steps without synchronising (benchmarking). */
int dpq_session_launch_steps(dpq_session* ss, int n, void* stream);
/* Trace of the dynamic steps so far: bits int8 / estimates f32 (NaN = none) /
 * exact errors f32, each [n_steps][n_layers]. */
int dpq_session_trace(dpq_session* ss, int* n_steps, int8_t* bits, float* est, float* exact);
int dpq_session_position(dpq_session* ss, int* pos);
/* 1 if the session runs the persistent step kernel, 0 for the multi-kernel graph. */
int dpq_session_is_persistent(dpq_session* ss);
/* Diagnostics: run one step eagerly (no graph) with CUDA events around every
 * fused selector+GEMV op launch; op_ms receives the per-launch device time
 * in schedule order (4 ops per block: qkv, o, up|gate, down). */
int dpq_session_profile_ops(dpq_session* ss, int token, int dynamic, float* op_ms, int max_ops,
                            int* n_ops);
/* Persistent engine stage list (kind: 0 begin, 1 op, 2 attention, 3 head,
 * 4 emit; idx: op index in schedule order / block). n_stages = 0 when the
 * session runs the multi-kernel path (exact / track_exact plans). */
int dpq_session_engine_stages(dpq_session* ss, int* n_stages, int32_t* kinds, int32_t* idx);
int dpq_session_logits_dev(dpq_session* ss, float** logits_dev);
/* Diagnostics (env DPQ_DEBUG_TIMES=1 at session creation): per-CTA phase
 * timestamps (globaltimer ns) of every op of the last step, [op][per_op]. */
int dpq_session_debug_times(dpq_session* ss, uint64_t* out, int64_t n, int* per_op);
/* Wait for the session's enqueued work (dpq_session_step with logits_host =
 * NULL, dpq_session_launch_steps) and check the engine's error flags;
 * dpq_session_logits copies the last step's float32 [vocab] logits. */
int dpq_session_sync(dpq_session* ss);
int dpq_session_logits(dpq_session* ss, float* logits_host);

/* ---- tensor parallelism (north star (4); runtime.py:348-369 sharded by
 * output rows, replaces the reference's single-process matvec loop) ------
 * One session per rank, each on its row shard of every linear layer: store
 * layer i holds rows [rank R_i / N, (rank + 1) R_i / N) (q/k/v: the rank's
 * heads, o/down: d/N rows, up/gate: d_ff/N rows); plan layer i holds the
 * rank's rows [rank k / N, ...) of the full layer's projection G and the
 * full layer's threshold. The persistent engine of each rank publishes its
 * output rows, attention states, estimator partials and stage arrivals into
 * every rank's exchange arena (peer stores over NVLink / same-device
 * memory), so ranks take identical decisions and identical tokens. */
typedef struct {
  int32_t tp_rank, tp_size;   /* 1..8 ranks                                   */
  int32_t grid;               /* CTAs of this rank's engine (0: every SM)     */
  int32_t pad_;
} dpq_tp_desc;
int dpq_session_create_tp(dpq_store* s, dpq_plan* p, const dpq_model_desc* m, const dpq_tp_desc* tp,
                          dpq_session** out);
/* The rank's exchange arena (device pointer, bytes) and its CUDA IPC handle
 * (64 bytes, cudaIpcMemHandle_t) for ranks in other processes. */
int dpq_session_tp_arena(dpq_session* ss, void** base, int64_t* bytes);
int dpq_session_tp_ipc_handle(dpq_session* ss, void* handle_out);
int dpq_tp_ipc_open(int device, const void* handle, void** base);
int dpq_tp_ipc_close(int device, void* base);
/* peer_bases[q]: rank q's arena as mapped in this process (own arena at
 * tp_rank). Call on every rank before the first step. */
int dpq_session_tp_connect(dpq_session* ss, void* const* peer_bases);

/* Host-side reference of the device plane layout (test infrastructure for the
 * repack; the product path repacks on the device). */
int dpq_repack_host(const uint16_t* codes, int rows, int cols, int n_bits, uint8_t* planes,
                    int64_t planes_bytes);
int64_t dpq_planes_bytes(int rows, int cols, int n_bits);

#ifdef __cplusplus
}
#endif
#endif
