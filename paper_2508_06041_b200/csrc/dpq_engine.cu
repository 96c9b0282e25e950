// Persistent decode-step engine for sm_100a (the fast path of dpq_session).
//
// One cooperative kernel runs whole decode steps (reference DecodeEngine.step,
// runtime.py:330-381) on one CTA per SM. A step is the stage list
//   BEGIN | per block: QKV  O  UPGATE  DOWN | HEAD
// with NO grid barrier between stages: every vector a stage publishes (the
// residual stream, q|k|v, the attention chunk states, SiLU(gate)*up) and every
// cross-window partial sum is a 64-bit word {float value, u32 epoch} (single-
// copy atomic, so no fence), and a reader waits only for the words it reads,
// tagged with the epoch of the stage that produces them. A relaxed arrival
// counter (one arrival per CTA and stage, in stage order) bounds the skew: a
// stage writes its double-buffered state only after every CTA has finished
// stage E - 2.
//
// Warp roles of a CTA (NCW consumer warps, one reducer warp, one TMA producer
// warp), all walking the same stage list:
//  * producer: streams the CTA's bitplane items (one (tile, plane) = 2 KB,
//    cp.async.bulk into a ring of 2 KB slots, mbarrier full/empty) for every op
//    as far ahead as the ring allows: base planes [0, nb) of the CTA's tasks,
//    then - once the op's precision decisions are taken from the estimator
//    accumulators (runtime.py:184-193, estimator.py:35-60) - the extra planes
//    [nb, h) of the layers that decided high;
//  * consumers: per op, the input window (512 columns) -> shared memory, the
//    estimator feeds of that window (G[w] . x[w] rows, fixed point, into the
//    layer accumulators) and the window's byte LUT (257 x 64 fp32), then the
//    CTA's tasks: task k (one 32-row tile of one layer) goes to warp k mod NCW,
//    Horner over its planes (S_{p+1} = 2 S_p + P_p, quant.py:74), 64 conflict-
//    free byte-LUT lookups per 2 KB item; the base sum and the extra-plane sum
//    of a (tile, window) are published as separate tagged words (no parking);
//  * reducer: unit u of an op (a tile, or an up|gate tile pair) belongs to CTA
//    u mod G; the warp waits for its units' window partials as they arrive
//    (concurrently with the consumers), S = 2^(h - nb) S_base + S_extra in fixed
//    window order, the affine epilogue y = s_in (lo sum x + span 2^-b (S +
//    sum x / 2)) (an exact restatement of quant.py:74-78 @ x), the residual add
//    / SiLU(gate)*up (runtime.py:364-370), and publishes the output tile.
// Per (op, CTA) the work is static (host-built): the CTA's window w (CTAs are
// split into window-aligned sets) and its tasks, every m-th tile of the op
// (m = CTAs of the window), so each layer of the op is spread evenly whatever
// bits it selects. Attention (runtime.py:351-362) runs in the o op's prologue
// on (head, 64-position chunk) units; o's input windows merge the chunk states.
#include "dpq_common.cuh"

// Consumer-only CTA barrier (the producer and reducer warps never join).
#ifndef DPQ_ATTN_WARPS
#define DPQ_ATTN_WARPS 8           // warps per attention unit (kAttnChunk / this = positions per warp)
#endif
#ifndef DPQ_RING_SLOTS
#define DPQ_RING_SLOTS 64          // ring slots (2 KB): bytes in flight per SM = the queueing depth
#endif
#ifndef DPQ_PF_ITEMS
#define DPQ_PF_ITEMS 0             // (measured slower at 64-256) next op's first base items prefetched into L2 per CTA
#endif
#ifndef DPQ_SEQ_SLEEP
#define DPQ_SEQ_SLEEP 100          // ns of back-off while a ring item is not yet issued (measured: -1.2%)
#endif
#ifndef DPQ_CONS_SLEEP
#define DPQ_CONS_SLEEP 0           // reducer: back-off while the consumers finish the stage
#endif
#ifndef DPQ_STAGE_SLEEP
#define DPQ_STAGE_SLEEP 0          // consumers: back-off on the stage counter (skew bound)
#endif
#ifndef DPQ_PSLOT_SLEEP
#define DPQ_PSLOT_SLEEP 100        // producer: back-off while its ring slot is still in use (-0.4%)
#endif
#ifndef DPQ_DEC_SLEEP
#define DPQ_DEC_SLEEP 0            // consumers: back-off while the op's decision is pending
#endif
#ifndef DPQ_SLOT_SLEEP
#define DPQ_SLOT_SLEEP 0           // ns of back-off while a ring item is in flight
#endif
#ifndef DPQ_FEEDS_FIRST
#define DPQ_FEEDS_FIRST 1          // estimator feeds + statistics before the window LUT (1 all ops, 2 q|k|v and o; measured 1 best)
#endif
#ifndef DPQ_LUT_PAIR
#define DPQ_LUT_PAIR 1             // LUT build jobs of two (1) or four (2) row blocks sharing the low-nibble sums (1: -0.6%, 2: +0.4%)
#endif
#ifndef DPQ_REL_ARRIVE
#define DPQ_REL_ARRIVE 1           // release / acq_rel atomics instead of fence + atomic (stage arrival, head)
#endif
#ifndef DPQ_EXTRA_PREFETCH
#define DPQ_EXTRA_PREFETCH 0       // extra planes of deciding layers prefetched into L2 while the decision is pending
#endif
#define CSYNC() asm volatile("bar.sync 1, %0;" :: "n"(dpq::eng::NT) : "memory")

namespace dpq {
namespace eng {

#ifndef DPQ_NCW
#define DPQ_NCW 10
#endif
constexpr int NCW = DPQ_NCW;       // consumer warps (12 warps per CTA: 3 per SMSP -> 168 registers)
constexpr int NW = NCW;
constexpr int NT = NCW * 32;       // consumer threads
constexpr int kRedWarp = NCW;      // reducer warp
constexpr int kProdWarp = NCW + 1; // TMA producer warp
constexpr int NTB = NT + 64;
constexpr int kItemBytes = 2048;   // one (tile, plane) item = kTileBytes
constexpr int kMaxSlots = DPQ_RING_SLOTS;      // ring slots (2 KB); the host checks they fit
constexpr int kDecRing = 4;        // op decision entries in flight
constexpr int kDbgRec = 28;        // debug stamps per (stage, CTA)
constexpr unsigned kPrevTag = 0x80000000u;   // previous-step sum x^2 words: tag = kPrevTag | rotation
constexpr int kCurSlots = 4;       // estimator-set slots of the current step (step % 4)
constexpr int kPrevSlots = 4;      // previous-step slots (rotation % 4)
constexpr int kSetSlots = kCurSlots + kPrevSlots;
// Packed G.x words: each window adds (1 << 56) + (v + 2^47), v = G_r[w] . x[w]
// at 2^fb with |v| < 2^47, so one relaxed red.add carries value and count
// (no release fence, no second atomic): count = word >> 56 (<= 255 windows).
constexpr int kCntShift = 56;
constexpr long long kFxBias = 1ll << 47;
constexpr uint32_t kLut = 0x20000;        // the window LUT (absolute shared address)

enum { ST_BEGIN = 0, ST_OP = 1, ST_HEAD = 3, ST_OUT = 4 };
enum { SRC_IMM = 0, SRC_PREV_STEP = 1, SRC_PREV_BLOCK = 2 };
enum { FEED_CUR = 0, FEED_CURFB = 1, FEED_PREV = 2 };
enum { ERR_RANGE = 1 };

typedef unsigned long long u64;

struct Layer {
  const uint4* planes;
  long long pstride;       // uint4 per plane
  const float* lo;
  const float* span;
  int rows, n_tiles, tile_off, out_off;
  int l, h, prefill_bit;
  int sentinel;            // 0 estimate, 1 low (T = +inf), 2 high (T = -inf)
  int xread;               // dual: all h planes streamed in dynamic steps (exact estimator / track_exact):
                           // y_l and y_h from the shared planes, ||y_h - y_l|| into exact set xset
  int xset, xcnt;          // exact set index; CTAs contributing to it (units of this layer)
  int est;                 // EST_NONE / EST_LINEAR / EST_PROJECTION
  int src;                 // SRC_*
  int k;                   // projection rank (0: linear)
  double fbscale;          // 2^-fb of the packed G.x words
  int set;                 // estimator set in each Prog.fpart slot: [k packed G.x words][n_win sum x^2 words]
  int feed_stage;          // stage (index in the step) whose consumers write the set
  int trace;               // trace column
  double T, slope, intercept;
};

// Static work of one CTA in one op (host-built): window w (CTA j of the m
// sharing it), tasks [task0, task0 + n_tasks) of Prog.tasks, and the CTA's
// task count per layer.
struct alignas(16) CtaWork {
  int task0;
  short n_tasks, w, j, m;
  short cnt[kMaxOpLayers];
  short pad;
};
static_assert(sizeof(CtaWork) == 32, "CtaWork is 32 bytes");

struct alignas(16) Op {
  Layer L[kMaxOpLayers];
  int n_layers;
  int cols, n_win, n_tiles;
  int rms;                 // input RMS-normalised (runtime.py:383-384)
  int pair;                // up|gate SiLU pair epilogue
  int add;                 // residual add: out = res_in + y
  int attn_in;             // input = attention of the q|k|v op (out of stage in_stage)
  int push;                // output published to every tensor-parallel rank (row-shard all-gather)
  int plain_io;            // single-op programs: input = plain floats at Prog.embed, output = plain floats at Prog.y_out
  int in_stage;            // stage (index in the step) publishing `in`
  int res_stage;           // stage publishing res_in
  int inst;                // input instance: statistics + estimator feeds
  int block;
  int feed_rows;           // projection rows of the input's feeds (split over the window's CTAs)
  int n_units;             // reduce units (tiles, or up|gate pairs)
  const u64* in;           // tagged input (attn_in: the q|k|v op's output)
  const u64* res_in;       // tagged residual input (add)
  u64* out;                // tagged output
  const CtaWork* work;     // [G]
  long long pad2;
};
static_assert(sizeof(Op) % 16 == 0, "Op is copied to shared memory in 16-byte words");

// Estimator feed of one input instance: G [n_win][k][512] (f32 / f16 / e4m3 +
// per-row scale) applied to each window, into the accumulator set `acc`.
struct Feed {
  const void* G;
  const float* gscale;
  int dtype, k, row0;      // row0: first row of this feed in the instance's row list
  int set;                 // the layer's set in Prog.fpart
  int set_r0;              // first set row of this rank's G rows (tensor parallel: G sharded by k)
  int kset;                // G rows of the set (all ranks'); its sum x^2 words follow them
  int kind;                // FEED_*
  double fxscale;          // 2^fb of the packed G.x words
};

struct ECtl {
  int mode;                // MODE_PREFILL / MODE_DYNAMIC            (host-written)
  int token;               //                                        (host-written)
  int force;               // decisions replaced by forced_bits      (host-written)
  int pos;
  int trace_step;
  int has_prev;
  int prime;
  int async_prev_block;
  int n_steps_done;        // steps since reset: publish word of the step control
  int rot;                 // previous-step slot rotations
  const signed char* forced_bits;
};

struct Prog {
  int n_stages;
  const int2* stages;      // (kind, op index)
  const Op* ops;
  const uint2* tasks;      // (tile | layer << 16, per-layer task counts before it: 10 bits each)
  const int* feed_begin;   // [n_inst + 1]
  const Feed* feeds;
  int n_inst;
  int d, H, KV, hd, dkv, f, vocab, seq_cap, n_blocks;   // H, KV, dkv: this rank's heads (tensor parallel)
  int dq;                  // this rank's q width (H hd)
  int hg0;                 // global index of this rank's first head
  // tensor parallelism (row shards): peer_off[q] = byte offset from this
  // rank's exchange arena to rank q's, mapped in this address space (peer
  // memory over NVLink; q = tp_rank: 0); pushed words go to every rank
  int tp_size, tp_rank;
  long long peer_off[8];
  float eps;
  const float* embed;
  const float* lm;
  const float* cosv;
  const float* sinv;
  u64* xe;                 // tagged x = embed[token]
  const u64* xfinal;       // tagged residual after the last block
  int final_stage;
  float* logits;
  // single-op programs (dpq_gemv / dpq_select_gemv): BEGIN reads the plain
  // input from `embed` (token 0), ST_OUT writes the op's output rows as plain
  // floats to y_out and the decision / estimate to bit_out / est_out
  float* y_out;
  int32_t* bit_out;
  float* est_out;
  int out_rows, out_op_stage;
  int gemv_mode;           // > 0: single-op program; the step runs in this mode (MODE_*)
  int gemv_force;          // 1: the op's bit is gemv_bit (dpq_gemv); 0: the selector decides
  int gemv_bit;
  float* const* kc;        // [n_blocks] -> [seq_cap][dkv]
  float* const* vc;
  u64* slot;               // [2 (stage parity)][slot_half]: per op row (hi, lo) packed fixed-point
                           // sums of the windows' base partials (see add_partial)
  u64* slotx;              // [2][slot_half] the same for the extra-plane partials
  long long slot_half;
  u64* fpart;              // estimator sets [kSetSlots][set_stride]: per estimating layer k packed
                           // G.x words (kCntShift) + n_win tagged sum x[w]^2 words; slots
                           // step % 4 (current step), kCurSlots + rot % 4 (previous-step feeds)
  long long set_stride;
  u64* istat;              // [n_inst][istat_win][2] tagged window sums (sum x, sum x^2)
  int istat_win;
  u64* bar;                // stage arrivals (one per CTA and stage)
  unsigned* head_cnt;
  unsigned* err;           // sticky error flags (ERR_RANGE: fixed-point range exceeded)
  signed char* tr_bits;
  float* tr_est;
  float* tr_exact;         // [max_steps][n_trace] exact errors (dual layers)
  u64* xerr;               // [kCurSlots][n_xsets][2] packed (hi, lo) sums of (y_h - y_l)^2
  const int2* xsets;       // [n_xsets] (trace column, contributing CTAs)
  int n_xsets;
  int n_trace, max_steps;
  int* tok_log;
  ECtl* ctl;
  int smem_dyn;
  u64* dbg;                // optional [n_stages][G][kDbgRec] %globaltimer stamps
  u64* attn_part;          // [H][attn_maxch][hd + 2] tagged chunk partials (o[hd], m, l)
  int attn_maxch;
};

__device__ __forceinline__ void st_tag_all(const Prog& P, u64* p, float v, unsigned e) {
  const u64 w = ((u64)e << 32) | __float_as_uint(v);
  if (P.tp_size == 1) {
    __stcg(p, w);
    return;
  }
  for (int q = 0; q < P.tp_size; ++q)
    __stcg(reinterpret_cast<u64*>(reinterpret_cast<char*>(p) + P.peer_off[q]), w);
}
__device__ __forceinline__ void red_all(const Prog& P, u64* p, u64 v) {
  if (P.tp_size == 1) {      // single GPU: gpu scope
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
    return;
  }
  for (int q = 0; q < P.tp_size; ++q)
    asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" :: "l"(reinterpret_cast<char*>(p) + P.peer_off[q]), "l"(v)
                 : "memory");
}

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 ld_relaxed64(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 ld_acq64(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_acq_s64(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acq_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_add64(long long* p, long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_rel_add64(long long* p, long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_rel_addu64(u64* p, u64 v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
// tagged word {float v, u32 epoch}: one 64-bit store, single-copy atomic
__device__ __forceinline__ void st_tag(u64* p, float v, unsigned e) {
  __stcg(p, ((u64)e << 32) | __float_as_uint(v));
}
// A tagged word published to every tensor-parallel rank (p in the exchange arena).
__device__ __forceinline__ void st_tag_all(const struct Prog& P, u64* p, float v, unsigned e);
__device__ __forceinline__ void red_all(const struct Prog& P, u64* p, u64 v);
__device__ __forceinline__ uint4 ld_tag2(const u64* p) {   // two tagged words (16-byte aligned)
  uint4 r;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ u64 gclock() {
  u64 t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Spin-wait watchdog: a wait beyond its limit records (line, block, thread, a,
// b) in mapped host memory (dpq_engine_diag) and traps: a launch error, not a
// hang. No call, so nothing is spilled around the polling loops.
__device__ u64* g_diag = nullptr;
#define hang(what, a, b)                                                                   \
  do {                                                                                     \
    if (g_diag) {                                                                          \
      volatile u64* d_ = g_diag;                                                           \
      d_[1] = (u64)__LINE__; d_[2] = blockIdx.x; d_[3] = threadIdx.x;                      \
      d_[4] = (u64)(long long)(a); d_[5] = (u64)(long long)(b);                            \
      __threadfence_system(); d_[0] = 1ull; __threadfence_system();                        \
    }                                                                                      \
    __trap();                                                                              \
  } while (0)
#define SPIN_UNTIL_NS(cond, what, a, b, NS)                                                \
  do {                                                                                     \
    unsigned n_ = 0;                                                                       \
    u64 t0_ = 0;                                                                           \
    while (!(cond)) {                                                                      \
      if ((++n_ & 1023u) == 0) {                                                           \
        const u64 t_ = gclock();                                                           \
        if (t0_ == 0) t0_ = t_;                                                            \
        else if (t_ - t0_ > (NS)) hang(what, a, b);                                        \
      }                                                                                    \
    }                                                                                      \
  } while (0)
#define SPIN_UNTIL(cond, what, a, b) SPIN_UNTIL_NS(cond, what, a, b, 4000000000ull)

template <typename T>
__device__ __forceinline__ T wsum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// 1/sqrt(x) in double without library slow paths (MUFU seed + two Newton steps).
__device__ __forceinline__ double rsqrt_d(double x) {
  double r = (double)rsqrtf((float)x);
  r = r * (1.5 - 0.5 * x * r * r);
  r = r * (1.5 - 0.5 * x * r * r);
  return r;
}

// ---------------------------------------------------------------------------
// LUT lookups: lane l, byte s of its 64-byte plane segment -> LUT row e, slot
// (l + s) mod 64 (layout in dpq_common.cuh); address formed by one PRMT.
// ---------------------------------------------------------------------------
#define ENG_LDS(dst, addr, IMM) asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(dst) : "r"(addr), "n"(IMM))

__device__ __forceinline__ float plane_sum(const uint4 d0, const uint4 d1, const uint4 d2, const uint4 d3,
                                           uint32_t lanereg) {
#ifdef DPQ_NO_LOOKUP   // timing experiment only: the data path without the LUT lookups
  return __uint_as_float((d0.x ^ d1.y ^ d2.z ^ d3.w) & 0x007fffffu);
#endif
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#define ENG_WORD(W, S0)                                                 \
  {                                                                     \
    float v0, v1, v2, v3;                                               \
    ENG_LDS(v0, __byte_perm((W), lanereg, 0x7604u), 4 * (S0 + 0));      \
    ENG_LDS(v1, __byte_perm((W), lanereg, 0x7614u), 4 * (S0 + 1));      \
    ENG_LDS(v2, __byte_perm((W), lanereg, 0x7624u), 4 * (S0 + 2));      \
    ENG_LDS(v3, __byte_perm((W), lanereg, 0x7634u), 4 * (S0 + 3));      \
    a0 += v0; a1 += v1; a2 += v2; a3 += v3;                             \
  }
  ENG_WORD(d0.x, 0) ENG_WORD(d0.y, 4) ENG_WORD(d0.z, 8) ENG_WORD(d0.w, 12)
  ENG_WORD(d1.x, 16) ENG_WORD(d1.y, 20) ENG_WORD(d1.z, 24) ENG_WORD(d1.w, 28)
  ENG_WORD(d2.x, 32) ENG_WORD(d2.y, 36) ENG_WORD(d2.z, 40) ENG_WORD(d2.w, 44)
  ENG_WORD(d3.x, 48) ENG_WORD(d3.y, 52) ENG_WORD(d3.z, 56) ENG_WORD(d3.w, 60)
#undef ENG_WORD
  return (a0 + a1) + (a2 + a3);
}

// Byte LUT of one 512-column window from the staged window xw: row e, slot g =
// sum_{t: bit t of e} x[8g + t]; row 256 = 0 (target of the wrapped "e - 1"
// encoding for e = 0). Job q = (group g, 16-row block m) writes rows
// [16 m, 16 m + 16) of slot g (low nibble subset sums + the high nibble's);
// the 1024 jobs are spread over all consumer threads (conflict-free stores).
__device__ __forceinline__ void lut_build(float* lut, const float* xw) {
#if DPQ_LUT_PAIR
  // job q = (slot g, row blocks 2 mm and 2 mm + 1): the low-nibble subset sums
  // once for both (512 jobs, at most 2 per thread)
  constexpr int kMB = DPQ_LUT_PAIR == 2 ? 4 : 2;      // row blocks per job
  for (int q = threadIdx.x; q < 1024 / kMB; q += NT) {
    const int g = q & 63, mm = q >> 6;
    const float4 xa = *reinterpret_cast<const float4*>(xw + 8 * g);
    const float4 xb = *reinterpret_cast<const float4*>(xw + 8 * g + 4);
    float L[16];
    L[0] = 0.f;
#pragma unroll
    for (int n = 1; n < 16; ++n) {
      const int low = n & (-n);
      L[n] = L[n ^ low] + (low == 1 ? xa.x : low == 2 ? xa.y : low == 4 ? xa.z : xa.w);
    }
#pragma unroll
    for (int h = 0; h < kMB; ++h) {
      const int m = kMB * mm + h;
      float H = 0.f;
      if (m & 1) H += xb.x;
      if (m & 2) H += xb.y;
      if (m & 4) H += xb.z;
      if (m & 8) H += xb.w;
#pragma unroll
      for (int i = 0; i < 16; ++i) lut[(16 * m + i) * kGroups + g] = L[i] + H;
    }
  }
  if (threadIdx.x < 64) lut[256 * kGroups + threadIdx.x] = 0.f;
  return;
#endif
  for (int q = threadIdx.x; q < 1024; q += NT) {
    const int g = q & 63, m = q >> 6;
    const float4 xa = *reinterpret_cast<const float4*>(xw + 8 * g);
    const float4 xb = *reinterpret_cast<const float4*>(xw + 8 * g + 4);
    float L[16];
    L[0] = 0.f;
#pragma unroll
    for (int n = 1; n < 16; ++n) {
      const int low = n & (-n);
      L[n] = L[n ^ low] + (low == 1 ? xa.x : low == 2 ? xa.y : low == 4 ? xa.z : xa.w);
    }
    float H = 0.f;
    if (m & 1) H += xb.x;
    if (m & 2) H += xb.y;
    if (m & 4) H += xb.z;
    if (m & 8) H += xb.w;
#pragma unroll
    for (int i = 0; i < 16; ++i) lut[(16 * m + i) * kGroups + g] = L[i] + H;
  }
  if (threadIdx.x < 64) lut[256 * kGroups + threadIdx.x] = 0.f;
}

constexpr int kMaxTasks = 256;     // tasks (tiles) per CTA and op

struct Smem {
  Prog prog;
  ECtl ctl[2];                       // control block of the step, by step parity
  Op cop[2];                         // consumer: current / next op (by op parity)
  CtaWork cw[2];
  Op pop;                            // producer copy
  CtaWork pw;
  Op rop[2];                         // reducer copies (current / prefetched next, by op parity)
  unsigned long long full[kMaxSlots], empty[kMaxSlots];   // ring mbarriers
  volatile int seq[kMaxSlots];       // FIFO index armed in each slot (phase disambiguation)
  unsigned slot_off[kMaxSlots];
  volatile int dec_op;               // decisions of ops < dec_op are published
  int dec_fin[kDecRing][kMaxOpLayers];
  float dec_est[kDecRing];           // first layer's estimate of the op (single-op programs)
  float4 xraw[8][32];                // dual ops: per unit and lane (S_base, S_extra) of up to two tiles
  volatile int cons_ops;             // ops finished by the consumers
  volatile unsigned cons_gs;         // consumer stages finished (global stage number + 1)
  volatile int step_ready;           // steps whose control block is in ctl[]
  int head_last;
  float head_v[NW];
  int head_i[NW];
  double red[32];
  alignas(16) double dred[kMaxOpLayers][2][32];  // reducer: per-lane estimator partials (decide_op)
  double dest[kMaxOpLayers];         // reducer: the op's estimates, real and streaming bits
  int dbit[kMaxOpLayers], dfin[kMaxOpLayers];
  alignas(16) float attn_q[128];     // RoPE'd q of the current attention unit
  alignas(16) float attn_m[DPQ_ATTN_WARPS][132];  // per-warp (o[hd], m, l) of the unit
  alignas(16) float xw[kWinCols];    // the op's input window
  signed char gemv_bits[4];          // single-op programs: the forced bit (ECtl.forced_bits -> here)
  uint2 ctask[2][kMaxTasks];         // consumer task lists (by op parity)
  uint2 ptask[kMaxTasks];            // producer task list
  const uint4* psrc[kMaxTasks];      // producer: plane-0 address of each task's tile
};

__device__ __forceinline__ int layer_of(const Op& O, int t) {
  int li = 0;
  while (li + 1 < O.n_layers && t >= O.L[li + 1].tile_off) ++li;
  return li;
}

// Per-layer integers of an op (<= 3 layers) in registers: indexed by select,
// never by a local-memory array.
struct I3 {
  int v0, v1, v2;
  __device__ __forceinline__ int operator[](int i) const { return i == 0 ? v0 : (i == 1 ? v1 : v2); }
  __device__ __forceinline__ void set(int i, int x) {
    if (i == 0) v0 = x;
    else if (i == 1) v1 = x;
    else v2 = x;
  }
};

// Base planes per layer for the step mode (known before the decision).
__device__ __forceinline__ int base_bit(const Layer& L, const ECtl& C) {
  if (C.mode == MODE_PREFILL) return L.prefill_bit;
  if (L.xread) return L.l;              // dual: base l planes, then the h - l extras regardless of the decision
  if (C.force && L.trace >= 0) return C.forced_bits[L.trace];
  if (L.sentinel == 2) return L.h;
  return L.l;
}

// Task k of a CTA's list: op tile, layer, and per-layer counts of the tasks before it.
__device__ __forceinline__ int task_tile(uint2 t) { return (int)(t.x & 0xffffu); }
__device__ __forceinline__ int task_layer(uint2 t) { return (int)(t.x >> 16); }
__device__ __forceinline__ int task_before(uint2 t, const I3& per_layer) {
  return (int)(t.y & 1023u) * per_layer.v0 + (int)((t.y >> 10) & 1023u) * per_layer.v1 +
         (int)((t.y >> 20) & 1023u) * per_layer.v2;
}
__device__ __forceinline__ I3 base_bits(const Op& O, const ECtl& C) {
  I3 r{0, 0, 0};
  r.v0 = base_bit(O.L[0], C);
  if (O.n_layers > 1) r.v1 = base_bit(O.L[1], C);
  if (O.n_layers > 2) r.v2 = base_bit(O.L[2], C);
  return r;
}

// Asynchronous warp-parallel copy of an op descriptor (cp.async; complete
// after cp.async.wait_all of the issuing threads).
__device__ __forceinline__ void load_op_async(const Prog& P, int oi, Op* O) {
  const int lane = threadIdx.x & 31;
  const int nw4 = (int)(sizeof(Op) / 16);
  const char* src = reinterpret_cast<const char*>(P.ops + oi);
  for (int q = lane; q < nw4; q += 32)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"((uint32_t)__cvta_generic_to_shared(O) + 16u * q),
                 "l"(src + 16 * q) : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Warp-parallel copy of an op descriptor (+ this CTA's work and task list).
__device__ __forceinline__ void load_op(const Prog& P, int oi, int cta, Op* O, CtaWork* W, uint2* tasks) {
  const int lane = threadIdx.x & 31;
  const int nw4 = (int)(sizeof(Op) / 16);
  const int4* src = reinterpret_cast<const int4*>(P.ops + oi);
  int4* dst = reinterpret_cast<int4*>(O);
  for (int q = lane; q < nw4; q += 32) dst[q] = __ldg(src + q);
  __syncwarp();
  if (!W) return;
  const CtaWork* gw = O->work + cta;
  if (lane < 2) reinterpret_cast<int4*>(W)[lane] = __ldg(reinterpret_cast<const int4*>(gw) + lane);
  __syncwarp();
  const int n = W->n_tasks, t0 = W->task0;
  for (int k = lane; k < n; k += 32) tasks[k] = __ldg(P.tasks + t0 + k);
  __syncwarp();
}

// ---------------------------------------------------------------------------
// TMA / mbarrier helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// Ring slot sl's offset in the dynamic shared memory (the layout the kernel
// prologue builds in sm.slot_off: below the LUT after Smem, then above its zero
// row), computed in registers: a shared-memory table read per item queues
// behind the consumers' LUT loads.
__device__ __forceinline__ uint32_t slot_offset(const void* smem0, int sl) {
  const uint32_t base = smem_u32(smem0);
  const uint32_t lo = (base + (uint32_t)sizeof(Smem) + 127u) & ~127u;
  const int n_lo = lo + kItemBytes <= kLut ? (int)((kLut - lo) / kItemBytes) : 0;
  return (sl < n_lo ? lo + (uint32_t)sl * kItemBytes : kLut + kLutBytes + (uint32_t)(sl - n_lo) * kItemBytes) - base;
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_n(unsigned long long* bar, unsigned n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t a, unsigned parity) {
  unsigned ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  return ok != 0;
}
// Bitplanes are streamed once per step (GBs >> L2): evict-first so they do not
// push the small, re-read state (vectors, partials, accumulators, G, KV rows)
// out of L2.
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ unsigned long long l2_evict_last_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float4 ld_keep(const float* p, unsigned long long policy) {
  float4 r;
  asm volatile("ld.global.cg.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(policy));
  return r;
}
__device__ __forceinline__ uint4 ld_nc16_half(const void* p) {   // 8 bytes (x, y)
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return make_uint4(r.x, r.y, 0u, 0u);
}
__device__ __forceinline__ unsigned ld_nc4(const void* p) {
  unsigned r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_nc16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                            unsigned long long policy) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}

// ---------------------------------------------------------------------------
// Estimator sets and input statistics: tagged per-window partials (plain
// 64-bit stores, no atomics, no fences); readers sum the windows in fixed
// order, so every CTA gets the same value.
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64* istat_words(const Prog& P, int inst, int w) {
  return P.istat + ((size_t)inst * P.istat_win + w) * 2;
}

// Feed rows of the op's input window (consumer prologue). Rows of all feeds
// of the instance are numbered 0..feed_rows-1; CTA j of the window's m takes
// rows j, j + m, ...; its i-th row goes to warp kFeedW0 + i % kFeedWarps.
// Row r of feed F: partial G_F[w][r] . x[w] in fp32 lanes + double warp sum,
// stored as the tagged float word (w, r) of the layer's set.
constexpr int kFeedW0 = 0, kFeedWarps = NCW - 1; // warps 0..NCW-2 (then the LUT build, all warps)
constexpr int kStatW = NCW - 1;                  // statistics warp

__device__ __forceinline__ bool feed_active(const Feed& F, const ECtl& C) {
  const bool dyn = C.mode == MODE_DYNAMIC;
  if (F.kind == FEED_PREV) return dyn || C.prime;
  if (F.kind == FEED_CURFB) return dyn && !C.has_prev;
  return dyn;
}
// Slot of a feed's words: previous-step feeds kCurSlots + rot % 4, current-step
// feeds step % 4 (zeroed two steps ahead in BEGIN); tag of its sum x^2 words:
// the rotation (previous step) or the stage epoch.
__device__ __forceinline__ u64* feed_words(const Prog& P, const ECtl& C, const Feed& F) {
  const int slot = F.kind == FEED_PREV ? kCurSlots + (C.rot & (kPrevSlots - 1)) : (C.n_steps_done & (kCurSlots - 1));
  return P.fpart + (size_t)slot * P.set_stride + F.set;
}
__device__ __forceinline__ unsigned feed_tag(const ECtl& C, const Feed& F, unsigned epoch) {
  return F.kind == FEED_PREV ? (kPrevTag | ((unsigned)C.rot & 0x7fffffffu)) : epoch;
}

// G row r of feed F in window w, lanes 16 columns each: raw data (f16: 2
// words, f32: 4, e4m3: 1 + the row scale), loaded ahead of the input window.
struct GRow {
  uint4 g[2];
  float scale;
};
// Lane l takes columns 4 l + 128 q + j (q, j < 4) of the window: the G loads
// are coalesced per q and the window reads (xw) are conflict-free LDS.128.
__device__ __forceinline__ void feed_row_load(const Feed& F, int w, int r, GRow& R) {
  const int lane = threadIdx.x & 31;
  const size_t base = ((size_t)w * F.k + r) * kWinCols + 4 * lane;
  R.scale = 1.f;
  if (F.dtype == G_F16) {
    const __half* g = reinterpret_cast<const __half*>(F.G) + base;
    uint2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 t = ld_nc16_half(g + 128 * q);
      v[q] = make_uint2(t.x, t.y);
    }
    R.g[0] = make_uint4(v[0].x, v[0].y, v[1].x, v[1].y);
    R.g[1] = make_uint4(v[2].x, v[2].y, v[3].x, v[3].y);
  } else if (F.dtype == G_F32) {
    // 16 floats per lane: loaded in feed_row_dot (not held across the input wait)
  } else {   // e4m3 with a per-row scale
    const unsigned char* g = reinterpret_cast<const unsigned char*>(F.G) + base;
    R.g[0] = make_uint4(ld_nc4(g), ld_nc4(g + 128), ld_nc4(g + 256), ld_nc4(g + 384));
    R.scale = __ldg(F.gscale + r);
  }
}
// Window partial G[w][r] . x[w] from the loaded row (fp32 lanes + double warp sum).
__device__ __forceinline__ double feed_row_dot(const Feed& F, int w, int r, const GRow& R, const float* xw) {
  const int lane = threadIdx.x & 31;
  float s = 0.f;
  float4 x[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) x[q] = *reinterpret_cast<const float4*>(xw + 4 * lane + 128 * q);
  if (F.dtype == G_F16) {
    const unsigned hw[8] = {R.g[0].x, R.g[0].y, R.g[0].z, R.g[0].w, R.g[1].x, R.g[1].y, R.g[1].z, R.g[1].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 u = __half22float2(*reinterpret_cast<const __half2*>(&hw[2 * q]));
      const float2 v = __half22float2(*reinterpret_cast<const __half2*>(&hw[2 * q + 1]));
      s = fmaf(u.x, x[q].x, s);
      s = fmaf(u.y, x[q].y, s);
      s = fmaf(v.x, x[q].z, s);
      s = fmaf(v.y, x[q].w, s);
    }
  } else if (F.dtype == G_F32) {
    const float* g = reinterpret_cast<const float*>(F.G) + ((size_t)w * F.k + r) * kWinCols + 4 * lane;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 a = ld_nc16(g + 128 * q);
      s = fmaf(__uint_as_float(a.x), x[q].x, s);
      s = fmaf(__uint_as_float(a.y), x[q].y, s);
      s = fmaf(__uint_as_float(a.z), x[q].z, s);
      s = fmaf(__uint_as_float(a.w), x[q].w, s);
    }
  } else {
    const unsigned wd[4] = {R.g[0].x, R.g[0].y, R.g[0].z, R.g[0].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float xv[4] = {x[q].x, x[q].y, x[q].z, x[q].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_fp8_e4m3 e;
        e.__x = (unsigned char)(wd[q] >> (8 * j));
        s = fmaf((float)e, xv[j], s);
      }
    }
    s *= R.scale;
  }
  return wsum((double)s);
}

// The feed row list: row q of the instance -> its feed (linear scan; <= a few feeds).
__device__ __forceinline__ const Feed* feed_of_row(const Prog& P, int inst, int q) {
  const int f0 = P.feed_begin[inst], f1 = P.feed_begin[inst + 1];
  const Feed* F = P.feeds + f0;
  for (int f = f0; f < f1; ++f) {
    const Feed* G = P.feeds + f;
    if (G->k > 0 && q >= G->row0 && q < G->row0 + G->k) return G;
  }
  return F;
}

// Feed rows of this CTA (rows j, j + m, ... of the instance's row list; its
// i-th row -> warp kFeedW0 + i % kFeedWarps). The first kFeedPre rows of a
// warp are loaded before the input window arrives (feed_prefetch) and
// finished once it is staged (feed_finish); further rows are loaded then.
#ifndef DPQ_FEED_PRE
#define DPQ_FEED_PRE 2
#endif
constexpr int kFeedPre = DPQ_FEED_PRE;
struct FeedPre {
  bool pre;                // the warp's first kFeedPre rows were prefetched
  const Feed* F[kFeedPre];
  int r[kFeedPre];
  GRow R[kFeedPre];
};

__device__ __forceinline__ void feed_prefetch(const Prog& P, const ECtl& C, const Op& O, const CtaWork& W,
                                              FeedPre& fp) {
  const int warp = threadIdx.x >> 5;
  fp.pre = true;
#pragma unroll
  for (int i = 0; i < kFeedPre; ++i) {
    fp.F[i] = nullptr;
    const int q = W.j + (warp - kFeedW0 + i * kFeedWarps) * W.m;
    if (warp < kFeedW0 || warp >= kFeedW0 + kFeedWarps || q >= O.feed_rows) continue;
    const Feed* F = feed_of_row(P, O.inst, q);
    if (!feed_active(*F, C)) continue;
    fp.F[i] = F;
    fp.r[i] = q - F->row0;
    feed_row_load(*F, W.w, fp.r[i], fp.R[i]);
  }
}

// Row partial -> packed fixed point (value + count) into word r of the set:
// one relaxed red.add; |v| 2^fb >= 2^47 raises the sticky range flag.
__device__ __forceinline__ void feed_add(const Prog& P, const ECtl& C, const Feed& F, int r, double v) {
  if ((threadIdx.x & 31) == 0) {
    const double s = v * F.fxscale;
    long long f = 0;
    if (fabs(s) < (double)kFxBias) f = llrint(s);
    else atomicOr(P.err, (unsigned)ERR_RANGE);
    red_all(P, feed_words(P, C, F) + F.set_r0 + r, (1ull << kCntShift) + (u64)(f + kFxBias));
  }
}

// Feeds + statistics of the op's input window, once it is staged in xw.
__device__ __forceinline__ void feed_finish(const Prog& P, const ECtl& C, const Op& O, const CtaWork& W,
                                            const FeedPre& fp, const float* xw, unsigned epoch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = W.j, m = W.m;
  if (warp >= kFeedW0 && warp < kFeedW0 + kFeedWarps) {
    if (fp.pre)
#pragma unroll
      for (int i = 0; i < kFeedPre; ++i)
        if (fp.F[i]) feed_add(P, C, *fp.F[i], fp.r[i], feed_row_dot(*fp.F[i], W.w, fp.r[i], fp.R[i], xw));
    for (int i = warp - kFeedW0 + (fp.pre ? kFeedPre * kFeedWarps : 0);; i += kFeedWarps) {
      const int q = j + i * m;
      if (q >= O.feed_rows) break;
      const Feed* F = feed_of_row(P, O.inst, q);
      if (!feed_active(*F, C)) continue;
      GRow R;
      feed_row_load(*F, W.w, q - F->row0, R);
      feed_add(P, C, *F, q - F->row0, feed_row_dot(*F, W.w, q - F->row0, R, xw));
    }
  } else if (warp == kStatW && j == 0) {
    // sum x, sum x^2 of the window: op statistics + the feeds' sum x^2 words
    double s = 0.0, q = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {          // columns 4 lane + 128 i .. + 3 (conflict-free LDS.128)
      const float4 v4 = *reinterpret_cast<const float4*>(xw + 4 * lane + 128 * i);
      const double vv[4] = {(double)v4.x, (double)v4.y, (double)v4.z, (double)v4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s += vv[j];
        q += vv[j] * vv[j];
      }
    }
    s = wsum(s);
    q = wsum(q);
    if (lane == 0) {
      u64* st = istat_words(P, O.inst, W.w);
      st_tag(st, (float)s, epoch);
      st_tag(st + 1, (float)q, epoch);
    }
    for (int f = P.feed_begin[O.inst] + lane; f < P.feed_begin[O.inst + 1]; f += 32) {
      const Feed& F = P.feeds[f];
      if (!feed_active(F, C)) continue;
      st_tag(feed_words(P, C, F) + F.kset + W.w, (float)q, feed_tag(C, F, epoch));
    }
  }
}

// ---------------------------------------------------------------------------
// Input window: the tagged vector's 512 values -> xw (threads < 128, 4 each),
// waiting for the producing stage's epoch.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void load_window(const u64* in, int cols, int w, unsigned epoch, float* xw) {
  const int t = threadIdx.x;
  if (t >= 128) return;
  const int c0 = w * kWinCols + 4 * t;
  float v[4] = {0.f, 0.f, 0.f, 0.f};
  if (c0 + 4 <= cols) {
    uint4 a, b;
    bool ok;
    SPIN_UNTIL((a = ld_tag2(in + c0), b = ld_tag2(in + c0 + 2),
                ok = a.y == epoch && a.w == epoch && b.y == epoch && b.w == epoch), "input window", c0, epoch);
    v[0] = __uint_as_float(a.x); v[1] = __uint_as_float(a.z);
    v[2] = __uint_as_float(b.x); v[3] = __uint_as_float(b.z);
  } else {
    for (int j = 0; j < 4; ++j)
      if (c0 + j < cols) {
        u64 x;
        SPIN_UNTIL((x = ld_relaxed64(in + c0 + j), (unsigned)(x >> 32) == epoch), "input window", c0 + j, epoch);
        v[j] = __uint_as_float((unsigned)x);
      }
  }
  *reinterpret_cast<float4*>(xw + 4 * t) = make_float4(v[0], v[1], v[2], v[3]);
}

// ---------------------------------------------------------------------------
// Attention for the o op's window (runtime.py:351-362): the 512 / head_dim
// heads whose outputs are columns of window w, computed by every CTA of the
// window (identical code and data, so identical results). Unit = (head, sub)
// takes positions sub, sub + nsub, ... with an online softmax in registers
// (lane = 4 consecutive dims); units are merged per head in fixed order. The
// window's first CTA appends k_t / v_t of the window's KV groups
// (runtime.py:355-356); position t itself is taken from registers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 tag4(const u64* p, unsigned epoch) {
  uint4 a, b;
  bool ok;
  SPIN_UNTIL((a = ld_tag2(p), b = ld_tag2(p + 2), ok = a.y == epoch && a.w == epoch && b.y == epoch && b.w == epoch),
             "q|k|v", 0, epoch);
  return make_float4(__uint_as_float(a.x), __uint_as_float(a.z), __uint_as_float(b.x), __uint_as_float(b.z));
}
// RoPE (half split, runtime.py:288-298) of dims [i0, i0 + 4) of a head vector.
__device__ __forceinline__ float4 rope4(const u64* v, int i0, int hd, float4 c, float4 s, unsigned e) {
  const int half = hd / 2;
  const bool lo = i0 < half;
  const float4 a = tag4(v + i0, e);
  const float4 b = tag4(v + (lo ? i0 + half : i0 - half), e);
  float4 r;
  if (lo) {   // x_i c_i - x_{i+half} s_i
    r.x = a.x * c.x - b.x * s.x; r.y = a.y * c.y - b.y * s.y;
    r.z = a.z * c.z - b.z * s.z; r.w = a.w * c.w - b.w * s.w;
  } else {    // x_{i-half} s_j + x_i c_j
    r.x = b.x * s.x + a.x * c.x; r.y = b.y * s.y + a.y * c.y;
    r.z = b.z * s.z + a.z * c.z; r.w = b.w * s.w + a.w * c.w;
  }
  return r;
}
__device__ __forceinline__ float dot4(float4 a, float4 b) { return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w; }

// Attention unit (head h, 64-position chunk ch), run in the o
// op's prologue (runtime.py:351-362), on kAttnWarps warps (kw) of this CTA;
// O is the o op (O.in = the q|k|v op's tagged output).
//  * The cached K / V rows of the chunk (positions < t; they do not depend on
//    this step) are copied into shared memory (kv: [64][hd] K | [64][hd] V)
//    with cp.async before the q / k / v tags are awaited.
//  * q, k_t, v_t: all tag loads of a poll are issued together (one L2 round
//    trip once published); RoPE (runtime.py:288-298). Position t (last chunk)
//    is this step's k / v; the first head of a KV group appends them to the
//    cache (runtime.py:355-356).
//  * Scores (runtime.py:358): warp kw takes rows 16 kw .. 16 kw + 15, two
//    lanes per row (half the dims each, columns rotated by lane so a quarter
//    warp hits distinct banks); per-warp softmax state (m, l) and o = sum_s
//    p_s V_s with lanes over dims; the warps' states are merged in fixed order
//    and published unnormalised as tagged words (epoch e). o's input load
//    merges the chunks of a head (attn_merge).
constexpr int kAttnChunk = 64;
constexpr int kAttnWarps = DPQ_ATTN_WARPS;           // warps per attention unit
constexpr int kRowsPerWarp = kAttnChunk / kAttnWarps;   // chunk rows (positions) per warp
constexpr int kLanesPerRow = 32 / kRowsPerWarp;         // lanes sharing a row's score

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void attn_unit(const Prog& P, const ECtl& C, const Op& O, Smem& sm, int h, int ch, int kw,
                                          float* kv, unsigned e, u64* dbg) {
  const int lane = threadIdx.x & 31, tix = kw * 32 + lane;
  const bool stamp = dbg && tix == 0;
  const long long ck0 = clock64();
  if (stamp) dbg[8] = gclock();
  const int hd = P.hd, qh = P.H / P.KV, g = h / qh, t = C.pos;
  const int s0 = kAttnChunk * ch, s1 = min(s0 + kAttnChunk, t + 1);
  const int nc = min(s1, t) - s0;                                       // cached rows of the chunk
  float* Ks = kv;
  float* Vs = kv + kAttnChunk * hd;
  float* kc = P.kc[O.block];
  float* vc = P.vc[O.block];
  const size_t goff = (size_t)g * hd;
  {
    const int q4 = hd / 4;
    for (int i = tix; i < nc * q4; i += 32 * kAttnWarps) {
      const int r = i / q4, c = 4 * (i - r * q4);
      cp_async16(Ks + r * hd + c, kc + (size_t)(s0 + r) * P.dkv + goff + c);
      cp_async16(Vs + r * hd + c, vc + (size_t)(s0 + r) * P.dkv + goff + c);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (stamp) dbg[12] = clock64() - ck0;
  const int half = hd / 2;
  const int i0 = 4 * lane;
  const bool act = i0 < hd;
  if (kw == 0) {
    const bool lo = i0 < half;
    const int ip = lo ? i0 + half : i0 - half;
    const int jj = lo ? i0 : i0 - half;
    const bool cur = t < s1;                                             // position t is in this chunk
    const u64* qv = O.in + (size_t)h * hd;
    const u64* kv_ = O.in + P.dq + goff;
    const u64* vv_ = O.in + P.dq + P.dkv + goff;
    float4 c4 = make_float4(0.f, 0.f, 0.f, 0.f), s4 = c4;
    if (act) {
      c4 = __ldg(reinterpret_cast<const float4*>(P.cosv + (size_t)t * half + jj));
      s4 = __ldg(reinterpret_cast<const float4*>(P.sinv + (size_t)t * half + jj));
    }
    uint4 w[10];
    bool ok;
    auto poll = [&]() {
      if (!act) return true;
      w[0] = ld_tag2(qv + i0); w[1] = ld_tag2(qv + i0 + 2);
      w[2] = ld_tag2(qv + ip); w[3] = ld_tag2(qv + ip + 2);
      bool r = true;
      if (cur) {
        w[4] = ld_tag2(kv_ + i0); w[5] = ld_tag2(kv_ + i0 + 2);
        w[6] = ld_tag2(kv_ + ip); w[7] = ld_tag2(kv_ + ip + 2);
        w[8] = ld_tag2(vv_ + i0); w[9] = ld_tag2(vv_ + i0 + 2);
#pragma unroll
        for (int j = 4; j < 10; ++j) r &= w[j].y == e && w[j].w == e;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) r &= w[j].y == e && w[j].w == e;
      return r;
    };
    SPIN_UNTIL((ok = poll()), "q|k|v", h, e);
    auto val4 = [&](int j) {
      return make_float4(__uint_as_float(w[j].x), __uint_as_float(w[j].z), __uint_as_float(w[j + 1].x),
                         __uint_as_float(w[j + 1].z));
    };
    auto rope = [&](float4 a, float4 b) {                              // runtime.py:288-298 (half split)
      float4 r;
      if (lo) {
        r.x = a.x * c4.x - b.x * s4.x; r.y = a.y * c4.y - b.y * s4.y;
        r.z = a.z * c4.z - b.z * s4.z; r.w = a.w * c4.w - b.w * s4.w;
      } else {
        r.x = b.x * s4.x + a.x * c4.x; r.y = b.y * s4.y + a.y * c4.y;
        r.z = b.z * s4.z + a.z * c4.z; r.w = b.w * s4.w + a.w * c4.w;
      }
      return r;
    };
    if (act) {
      *reinterpret_cast<float4*>(sm.attn_q + i0) = rope(val4(0), val4(2));
      if (cur) {
        const float4 k4 = rope(val4(4), val4(6)), v4 = val4(8);
        *reinterpret_cast<float4*>(Ks + (t - s0) * hd + i0) = k4;
        *reinterpret_cast<float4*>(Vs + (t - s0) * hd + i0) = v4;
        if (h % qh == 0) {                                               // KV append (runtime.py:355-356)
          *reinterpret_cast<float4*>(kc + (size_t)t * P.dkv + goff + i0) = k4;
          *reinterpret_cast<float4*>(vc + (size_t)t * P.dkv + goff + i0) = v4;
        }
      }
    }
  }
  if (stamp) { dbg[9] = gclock(); dbg[13] = clock64() - ck0; }
  asm volatile("cp.async.wait_all;" ::: "memory");
  asm volatile("bar.sync 2, %0;" :: "n"(32 * kAttnWarps) : "memory");
  if (stamp) { dbg[10] = gclock(); dbg[14] = clock64() - ck0; }
  // scores: row r of the chunk, slice part of its dims (kLanesPerRow lanes per
  // row); float4 chunks rotated by lane so a quarter warp hits 8 bank groups
  const float scale = 1.0f / sqrtf((float)hd);
  const int r = kRowsPerWarp * kw + lane / kLanesPerRow, part = lane % kLanesPerRow;
  const bool valid = s0 + r < s1;
  float a0 = 0.f, a1 = 0.f;
  {
    const int dpl = hd / kLanesPerRow;          // dims per lane (>= 4)
    const int nch = dpl / 4;                    // float4 chunks per lane
    const float* kr = Ks + r * hd + part * dpl;
    const float* qr = sm.attn_q + part * dpl;
    if (nch == 0) {                             // head_dim < 4 kLanesPerRow: scalar dims
      for (int i = 0; i < dpl; ++i) a0 += qr[i] * kr[i];
    } else {
      const int rot = lane % nch;
      for (int c = 0; c < nch; c += 2) {
        const int c0 = (c + rot) % nch, c1 = (c + 1 + rot) % nch;
        a0 += dot4(*reinterpret_cast<const float4*>(qr + 4 * c0), *reinterpret_cast<const float4*>(kr + 4 * c0));
        if (c + 1 < nch)
          a1 += dot4(*reinterpret_cast<const float4*>(qr + 4 * c1), *reinterpret_cast<const float4*>(kr + 4 * c1));
      }
    }
  }
  float a = a0 + a1;
#pragma unroll
  for (int off = 1; off < kLanesPerRow; off <<= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
  const float sc = valid ? a * scale : -CUDART_INF_F;
  float m = sc;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  const float p = valid ? expf(sc - m) : 0.f;                            // runtime.py:359-361
  const float l = wsum(part == 0 ? p : 0.f);
  if (stamp) dbg[15] = clock64() - ck0;
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
  const int n = max(0, min(kRowsPerWarp, s1 - s0 - kRowsPerWarp * kw));
#pragma unroll
  for (int j = 0; j < kRowsPerWarp; ++j) {
    if (j < n) {
      const float pj = __shfl_sync(0xffffffffu, p, kLanesPerRow * j);
      if (act) {
        const float4 vv = *reinterpret_cast<const float4*>(Vs + (kRowsPerWarp * kw + j) * hd + i0);
        o.x += pj * vv.x; o.y += pj * vv.y; o.z += pj * vv.z; o.w += pj * vv.w;
      }
    }
  }
  float* mw = sm.attn_m[kw];
  if (act) *reinterpret_cast<float4*>(mw + i0) = o;
  if (lane == 0) { mw[hd] = n > 0 ? m : -CUDART_INF_F; mw[hd + 1] = l; }
  asm volatile("bar.sync 2, %0;" :: "n"(32 * kAttnWarps) : "memory");
  if (kw == 0) {
    float M = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm.attn_m[w][hd]);
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) {
      const float mw_ = sm.attn_m[w][hd];
      const float ew = mw_ == -CUDART_INF_F ? 0.f : expf(mw_ - M);
      L += ew * sm.attn_m[w][hd + 1];
      if (act) {
        const float4 ow = *reinterpret_cast<const float4*>(sm.attn_m[w] + i0);
        acc.x += ew * ow.x; acc.y += ew * ow.y; acc.z += ew * ow.z; acc.w += ew * ow.w;
      }
    }
    // published to every rank (o's input windows span all heads)
    u64* dst = P.attn_part + ((size_t)(P.hg0 + h) * P.attn_maxch + ch) * (hd + 2);
    if (act) {
      st_tag_all(P, dst + i0, acc.x, e);
      st_tag_all(P, dst + i0 + 1, acc.y, e);
      st_tag_all(P, dst + i0 + 2, acc.z, e);
      st_tag_all(P, dst + i0 + 3, acc.w, e);
    }
    if (lane == 0) {
      st_tag_all(P, dst + hd, M, e);
      st_tag_all(P, dst + hd + 1, L, e);
    }
  }
  asm volatile("bar.sync 2, %0;" :: "n"(32 * kAttnWarps) : "memory");   // kv / attn_m reusable
  if (stamp) { dbg[11] = gclock(); dbg[6] = clock64() - ck0; }
}

// o's input window: the attention output of the window's heads, merged over
// the heads' chunk partials in fixed chunk order (runtime.py:359-362).
__device__ __forceinline__ void attn_merge(const Prog& P, const ECtl& C, int w, unsigned e, float* xw) {
  const int t = threadIdx.x;
  if (t >= 128) return;
  const int hd = P.hd;
  const int c0 = w * kWinCols + 4 * t;
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c0 < P.d) {
    const int h = c0 / hd, i = c0 - h * hd;
    const int nch = (C.pos + kAttnChunk) / kAttnChunk;
    const u64* base = P.attn_part + (size_t)h * P.attn_maxch * (hd + 2);
    float M = -CUDART_INF_F, L = 0.f;
    for (int ch = 0; ch < nch; ++ch) {                                   // online merge, fixed chunk order
      const u64* q = base + (size_t)ch * (hd + 2);
      uint4 a, b, s;
      bool ok;
      SPIN_UNTIL((a = ld_tag2(q + i), b = ld_tag2(q + i + 2), s = ld_tag2(q + hd),
                  ok = a.y == e && a.w == e && b.y == e && b.w == e && s.y == e && s.w == e), "attention partial", h, ch);
      const float mc = __uint_as_float(s.x);
      const float Mn = fmaxf(M, mc);
      const float ea = expf(M - Mn), eb = expf(mc - Mn);
      L = L * ea + __uint_as_float(s.z) * eb;
      r.x = r.x * ea + __uint_as_float(a.x) * eb;
      r.y = r.y * ea + __uint_as_float(a.z) * eb;
      r.z = r.z * ea + __uint_as_float(b.x) * eb;
      r.w = r.w * ea + __uint_as_float(b.z) * eb;
      M = Mn;
    }
    const float inv = 1.0f / L;                                          // runtime.py:362
    r.x *= inv; r.y *= inv; r.z *= inv; r.w *= inv;
  }
  *reinterpret_cast<float4*>(xw + 4 * t) = r;
}

// ---------------------------------------------------------------------------
// The stage counter. Global stage number gs = step * n_stages + si (steps
// since reset); epoch(gs) = gs + 1 tags everything stage gs publishes. Every
// CTA's reducer warp arrives once per stage, in order, after its consumers
// and itself are done with the stage; a stage writes its double-buffered
// state only after stage gs - 2 is done everywhere.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool stage_done(const Prog& P, unsigned gs) {
  if (gs < 2) return true;
  return ld_acq64(P.bar) >= (u64)(gs - 1) * gridDim.x * P.tp_size;
}

// ---------------------------------------------------------------------------
// Reduction + epilogue (reducer warp, lane = row of the tile)
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Cross-window partial sums (quant.py:74 @ x, one 512-column window per
// task): every window adds its row partial S_w to the row's two packed words
// (hi, lo) in one relaxed red.add each, no fence. v = round(S_w 2^30) (exact
// for fp32 S_w >= 2^-6) is split into hi = v >> 24 and lo = v mod 2^24; a
// word holds (count << 56) + sum of (part + 2^47), so the reader knows from
// the word itself when all n_win windows are in. Integer sums: the total is
// independent of the arrival order (deterministic). Range |S_w| < 2^33.
// ---------------------------------------------------------------------------
constexpr double kFxPart = 1073741824.0;   // 2^30
__device__ __forceinline__ void add_partial(u64* w, float S, unsigned* err) {
  long long v = 0;
  if (fabsf(S) < 8.0e9f) v = llrint((double)S * kFxPart);
  else atomicOr(err, (unsigned)ERR_RANGE);
  const long long hi = v >> 24, lo = v & 0xffffff;
  const u64 one = 1ull << kCntShift;
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(w), "l"(one + (u64)(hi + kFxBias)) : "memory");
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(w + 1), "l"(one + (u64)(lo + kFxBias)) : "memory");
}
__device__ __forceinline__ int packed_count(u64 w) { return (int)(w >> kCntShift); }
__device__ __forceinline__ long long packed_value(u64 w) {
  const long long c = (long long)(w >> kCntShift);
  return (long long)(w & ((1ull << kCntShift) - 1)) - c * kFxBias;
}
// the row's total from its (hi, lo) words
__device__ __forceinline__ double partial_total(uint4 q) {
  const u64 h = ((u64)q.y << 32) | q.x, l = ((u64)q.w << 32) | q.z;
  return (double)packed_value(h) * (1.0 / 64.0) + (double)packed_value(l) * (1.0 / kFxPart);
}

// Row totals of up to two op tiles (t1 = -1: none): base sums from slot,
// extra-plane sums from slotx when ex0 / ex1 > 0; every word of the poll is
// loaded at once (16 bytes per stream and lane), complete when each word
// counts n_win windows; S = 2^ex S_base + S_extra. The words are zeroed once
// read (this warp is their only reader; the stage parity reuses them two
// stages later).
__device__ __forceinline__ float2 tiles_S(const Prog& P, const Op& O, int t0, int ex0, int t1, int ex1,
                                         unsigned epoch, double* raw = nullptr) {
  const int lane = threadIdx.x & 31;
  const size_t par = (size_t)((epoch - 1u) & 1u) * P.slot_half;   // parity of the stage (epoch = gs + 1)
  u64* b0 = P.slot + par + ((size_t)t0 * 32 + lane) * 2;
  u64* x0 = P.slotx + par + ((size_t)t0 * 32 + lane) * 2;
  u64* b1 = P.slot + par + ((size_t)max(t1, 0) * 32 + lane) * 2;
  u64* x1 = P.slotx + par + ((size_t)max(t1, 0) * 32 + lane) * 2;
  const bool two = t1 >= 0, e0 = ex0 > 0, e1 = two && ex1 > 0;
  const unsigned nw = (unsigned)O.n_win;
  uint4 q0, q1, q2, q3;
  const uint4 full = make_uint4(0u, nw << 24, 0u, nw << 24);   // count n_win, value 0 (unused streams)
  bool ok;
  unsigned n_ = 0;
  u64 tt0 = 0;
  do {
    q0 = ld_tag2(b0);
    q1 = e0 ? ld_tag2(x0) : full;
    q2 = two ? ld_tag2(b1) : full;
    q3 = e1 ? ld_tag2(x1) : full;
    ok = (q0.y >> 24) == nw && (q0.w >> 24) == nw && (q1.y >> 24) == nw && (q1.w >> 24) == nw &&
         (q2.y >> 24) == nw && (q2.w >> 24) == nw && (q3.y >> 24) == nw && (q3.w >> 24) == nw;
    if ((++n_ & 1023u) == 0) {
      const u64 t_ = gclock();
      if (tt0 == 0) tt0 = t_;
      else if (t_ - tt0 > 4000000000ull) hang("window partials", t0, epoch);
    }
  } while (!__all_sync(0xffffffffu, ok));
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  *reinterpret_cast<uint4*>(b0) = z;
  if (e0) *reinterpret_cast<uint4*>(x0) = z;
  if (two) *reinterpret_cast<uint4*>(b1) = z;
  if (e1) *reinterpret_cast<uint4*>(x1) = z;
  if (raw) {       // (S_base, S_extra) of both tiles, uncombined (dual layers)
    raw[0] = partial_total(q0);
    raw[1] = e0 ? partial_total(q1) : 0.0;
    raw[2] = two ? partial_total(q2) : 0.0;
    raw[3] = e1 ? partial_total(q3) : 0.0;
  }
  const double s0 = e0 ? ldexp(partial_total(q0), ex0) + partial_total(q1) : partial_total(q0);
  const double s1 = e1 ? ldexp(partial_total(q2), ex1) + partial_total(q3) : partial_total(q2);
  return make_float2((float)s0, (float)s1);
}

struct Epi { float scale, sx; };

// op input statistics (sum x, sum x^2): the windows' tagged sums (lane =
// window), summed in a fixed shuffle tree (identical on every CTA).
__device__ __forceinline__ Epi op_epi(const Prog& P, const Op& O, unsigned epoch) {
  const int lane = threadIdx.x & 31;
  double s = 0.0, q = 0.0;
  for (int w0 = 0; w0 < O.n_win; w0 += 32) {
    const int w = w0 + lane;
    if (w < O.n_win) {
      uint4 v;
      SPIN_UNTIL((v = ld_tag2(istat_words(P, O.inst, w)), v.y == epoch && v.w == epoch), "statistics", O.inst, w);
      s += (double)__uint_as_float(v.x);
      q += (double)__uint_as_float(v.z);
    }
  }
  s = wsum(s);
  q = wsum(q);
  Epi e;
  e.sx = (float)s;
  e.scale = O.rms ? (float)rsqrt_d(q / (double)O.cols + (double)P.eps) : 1.f;
  return e;
}

// ---------------------------------------------------------------------------
// Precision decisions of an op (producer warp), runtime.py:184-193: from the
// estimator accumulators (identical integers on every CTA, so every CTA takes
// the same decisions without another exchange).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void decide_op(const Prog& P, const ECtl& C, const Op& O, Smem& sm, const I3& nb, I3& fin,
                                          int cta, unsigned step_base, u64* rdbg, float* est0, I3& real) {
  const int lane = threadIdx.x & 31;
  const bool dyn = C.mode == MODE_DYNAMIC;
  // every estimating layer's words in one poll: lane holds packed G.x words
  // r = lane + 32 q and the sum x^2 word of window lane (+ 32); complete when
  // every packed count is n_win and every sum x^2 word carries its tag.
  // The descriptor fields (shared memory) are read before the poll: after it
  // they would queue behind the consumer warps' LUT loads in the MIO pipe
  // (~1-2 us per op, measured).
  constexpr int NQ = kMaxK / 32;
  const int n_l = O.n_layers, n_win = O.n_win;
  const u64* base[kMaxOpLayers] = {nullptr, nullptr, nullptr};
  unsigned tag[kMaxOpLayers] = {0u, 0u, 0u};
  int kq[kMaxOpLayers] = {0, 0, 0};
  double fbs[kMaxOpLayers] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int li = 0; li < kMaxOpLayers; ++li) {
    if (li >= n_l) break;
    const Layer& L = O.L[li];
    kq[li] = L.k;
    fbs[li] = L.fbscale;
    if (!(dyn && L.sentinel == 0 && L.est != EST_NONE && L.est != EST_EXACT)) continue;
    const bool prev = L.src == SRC_PREV_STEP && C.has_prev;
    const int slot = prev ? kCurSlots + ((C.rot - 1) & (kPrevSlots - 1)) : (C.n_steps_done & (kCurSlots - 1));
    base[li] = P.fpart + (size_t)slot * P.set_stride + L.set;
    tag[li] = prev ? (kPrevTag | ((unsigned)(C.rot - 1) & 0x7fffffffu)) : step_base + (unsigned)L.feed_stage + 1u;
  }
  // lane li < n_l: layer li's decision parameters
  int d_est = 0, d_l = 0, d_h = 0, d_sent = 0, d_tr = -1, d_nb = 0, d_forced = 0;
  bool d_xr = false;
  double d_T = 0.0, d_slope = 0.0, d_icpt = 0.0;
  if (lane < n_l) {
    const Layer& L = O.L[lane];
    d_est = L.est;
    d_l = L.l;
    d_h = L.h;
    d_sent = L.sentinel;
    d_tr = L.trace;
    d_xr = L.xread != 0;
    d_T = L.T;
    d_slope = L.slope;
    d_icpt = L.intercept;
    d_nb = nb[lane];
    if (C.force && d_tr >= 0) d_forced = C.forced_bits[d_tr];
  }
  const bool force = C.force != 0, rms = O.rms != 0;
  const double inv_cols = 1.0 / (double)O.cols, eps = (double)P.eps;
  const bool trace_ok = dyn && cta == 0 && P.n_trace > 0 && C.trace_step < P.max_steps;
  signed char* const tr_bits = P.tr_bits + (size_t)C.trace_step * P.n_trace;
  float* const tr_est = P.tr_est + (size_t)C.trace_step * P.n_trace;
  u64 g[kMaxOpLayers][NQ], sw[kMaxOpLayers][2];
  u64 t_g = 0, t_s = 0;
  {
    bool ok;
    unsigned n_ = 0;
    u64 t0_ = 0;
    do {
      ok = true;
#pragma unroll
      for (int li = 0; li < kMaxOpLayers; ++li) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int r = q * 32 + lane;
          g[li][q] = (base[li] && r < kq[li]) ? ld_relaxed64(base[li] + r) : ((u64)n_win << kCntShift);
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int w = q * 32 + lane;
          sw[li][q] = (base[li] && w < n_win) ? ld_relaxed64(base[li] + kq[li] + w) : ((u64)tag[li] << 32);
        }
      }
      bool okg = true, oks = true;
#pragma unroll
      for (int li = 0; li < kMaxOpLayers; ++li) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) okg &= (int)(g[li][q] >> kCntShift) == n_win;
#pragma unroll
        for (int q = 0; q < 2; ++q) oks &= (unsigned)(sw[li][q] >> 32) == tag[li];
      }
      ok = okg && oks;
      if (rdbg) {
        const bool ag = __all_sync(0xffffffffu, okg), as = __all_sync(0xffffffffu, oks);
        if (ag && t_g == 0) t_g = gclock();
        if (as && t_s == 0) t_s = gclock();
      }
      if (rdbg && n_ == 0 && (threadIdx.x & 31) == 0) rdbg[22] = gclock();
      if ((++n_ & 1023u) == 0) {
        const u64 t_ = gclock();
        if (t0_ == 0) t0_ = t_;
        else if (t_ - t0_ > 4000000000ull) hang("estimator feeds", n_l, n_win);
      }
    } while (!__all_sync(0xffffffffu, ok));
    if (rdbg && (threadIdx.x & 31) == 0) {
      rdbg[23] = n_;
      rdbg[24] = t_g;
      rdbg[25] = t_s;
      rdbg[26] = gclock();
    }
  }
  // per-lane partials -> shared memory; lane li sums layer li's in lane order
  // and takes its decision (no shuffle chains)
#pragma unroll
  for (int li = 0; li < kMaxOpLayers; ++li) {
    if (base[li] == nullptr) continue;
    double q = 0.0, sq = 0.0;
#pragma unroll
    for (int qq = 0; qq < NQ; ++qq) {
      const int r = qq * 32 + lane;
      if (r < kq[li]) {
        const long long c = (long long)(g[li][qq] >> kCntShift);
        const long long v = (long long)(g[li][qq] & ((1ull << kCntShift) - 1)) - c * kFxBias;
        const double gv = (double)v * fbs[li];
        q += gv * gv;
      }
    }
#pragma unroll
    for (int qq = 0; qq < 2; ++qq)
      if (qq * 32 + lane < n_win) sq += (double)__uint_as_float((unsigned)sw[li][qq]);
    sm.dred[li][0][lane] = q;
    sm.dred[li][1][lane] = sq;
  }
  __syncwarp();
  if (lane < n_l) {
    const bool has = (lane == 0 ? base[0] : lane == 1 ? base[1] : base[2]) != nullptr;
    int bit = d_nb;
    double est = CUDART_NAN;
    if (d_xr && dyn) {         // dual: the real bit (the stream always reads h planes)
      if (force && d_tr >= 0) bit = d_forced;
      else if (d_sent == 1) bit = d_l;
      else if (d_sent == 2) bit = d_h;
      else if (d_est == EST_EXACT) bit = -1;                 // decided from ||y_h - y_l|| after the reduction
    }
    if (has) {
      double qa[4] = {0.0, 0.0, 0.0, 0.0}, sa[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const double2 a = *reinterpret_cast<const double2*>(&sm.dred[lane][0][i]);
        const double2 b = *reinterpret_cast<const double2*>(&sm.dred[lane][0][i + 2]);
        const double2 c = *reinterpret_cast<const double2*>(&sm.dred[lane][1][i]);
        const double2 d = *reinterpret_cast<const double2*>(&sm.dred[lane][1][i + 2]);
        qa[0] += a.x; qa[1] += a.y; qa[2] += b.x; qa[3] += b.y;
        sa[0] += c.x; sa[1] += c.y; sa[2] += d.x; sa[3] += d.y;
      }
      const double q = (qa[0] + qa[1]) + (qa[2] + qa[3]), sq = (sa[0] + sa[1]) + (sa[2] + sa[3]);
      const double sc = rms ? rsqrt_d(sq * inv_cols + eps) : 1.0;
      if (d_est == EST_PROJECTION) est = q > 0.0 ? sc * q * rsqrt_d(q) : 0.0;                  // estimator.py:56-57
      else est = d_slope * (sq > 0.0 ? sc * sq * rsqrt_d(sq) : 0.0) + d_icpt;                 // estimator.py:41-42
      if (!force) bit = est > d_T ? d_h : d_l;                                               // strict > (runtime.py:192)
    }
    sm.dbit[lane] = bit;
    sm.dfin[lane] = d_xr && dyn ? d_h : bit;              // the streaming bits (producer / consumers)
    sm.dest[lane] = has ? est : CUDART_NAN;
    if (bit >= 0 && trace_ok && d_tr >= 0) {
      tr_bits[d_tr] = (signed char)bit;
      tr_est[d_tr] = has ? (float)est : CUDART_NAN_F;
    }
  }
  __syncwarp();
#pragma unroll
  for (int li = 0; li < kMaxOpLayers; ++li)
    if (li < n_l) {
      real.set(li, sm.dbit[li]);
      fin.set(li, sm.dfin[li]);
    }
  *est0 = n_l > 0 ? (float)sm.dest[0] : CUDART_NAN_F;
  if (rdbg && lane == 0) rdbg[27] = gclock();
}

// ---------------------------------------------------------------------------
// The TMA producer warp: streams every op's items into the ring (FIFO order:
// base items of the CTA's tasks, then the extra items of the layers that
// decided high), running ahead of the consumers as far as the ring allows.
// ---------------------------------------------------------------------------
// Items are issued by kIssueLanes lanes at once, one task per lane (its planes
// in lockstep): a batch spans <= kIssueLanes * 8 <= kMaxSlots consecutive FIFO
// items, so the slot each lane waits for holds an item issued before the batch
// (no lane can wait on an item another lane of the batch has yet to issue).
#ifndef DPQ_ISSUE_LANES
#define DPQ_ISSUE_LANES (DPQ_RING_SLOTS / 8)
#endif
constexpr int kIssueLanes = DPQ_ISSUE_LANES;   // lanes at 8 planes per task (measured: fewer is slower)
static_assert(kIssueLanes * 8 <= kMaxSlots, "an issue batch must fit the ring");
#ifndef DPQ_DYN_LANES
#define DPQ_DYN_LANES 1
#endif
__device__ __forceinline__ int issue_lanes(int planes) {
  return DPQ_DYN_LANES ? min(32, kMaxSlots / max(planes, 1)) : kIssueLanes;
}

__device__ __forceinline__ void producer(const Prog& P, Smem& sm, int cta, int G, int n_steps, int s0) {
  const int lane = threadIdx.x & 31;
  int fifo = 0, oi = 0;
  const unsigned char* dyn0 = reinterpret_cast<const unsigned char*>(&sm);
  const unsigned long long l2pol = l2_evict_first_policy();
  // items [jb, jb + n) of task k: planes p0 .. p0 + n - 1 of its tile
  auto issue_task = [&](int k, int jb, int p0, int n, long long pstride) {
    const unsigned char* src0 = reinterpret_cast<const unsigned char*>(sm.psrc[k]) + (long long)p0 * pstride;
    for (int p = 0; p < n; ++p) {
      const int j = jb + p;
      const int slot = j % kMaxSlots;
      if (j >= kMaxSlots) {
        // the consumer's release (mbarrier arrive after its reads) orders its
        // reads of the slot before this TMA write
        const unsigned par = (unsigned)(((j / kMaxSlots) - 1) & 1);
#if DPQ_PSLOT_SLEEP > 0
        if (!mbar_test(smem_u32(&sm.empty[slot]), par))
          SPIN_UNTIL_NS((__nanosleep(DPQ_PSLOT_SLEEP), mbar_test(smem_u32(&sm.empty[slot]), par)), "producer slot", j,
                        oi, 12000000000ull);
#else
        SPIN_UNTIL_NS(mbar_test(smem_u32(&sm.empty[slot]), par), "producer slot", j, oi, 12000000000ull);
#endif
      }
      sm.seq[slot] = j;
      mbar_expect_tx(&sm.full[slot], (unsigned)kItemBytes);
      tma_load_1d(const_cast<unsigned char*>(dyn0) + slot_offset(&sm, slot), src0 + (long long)p * pstride,
                  (unsigned)kItemBytes, &sm.full[slot], l2pol);
    }
  };
  for (int step = 0; step < n_steps; ++step) {
    if (lane == 0) SPIN_UNTIL_NS(sm.step_ready >= step + 1, "producer step", step, 0, 12000000000ull);
    __syncwarp();
    __threadfence_block();
    const ECtl& C = sm.ctl[step & 1];
    for (int si = 0; si < P.n_stages; ++si) {
      const int2 st = P.stages[si];
      if (st.x != ST_OP) continue;
      load_op(P, st.y, cta, &sm.pop, &sm.pw, sm.ptask);
      const Op& O = sm.pop;
      const CtaWork& W = sm.pw;
      const I3 nb = base_bits(O, C);
      I3 fin = nb;
      const long long ps0 = O.L[0].pstride * 16, ps1 = O.L[1].pstride * 16, ps2 = O.L[2].pstride * 16;
      // plane-0 address of every task's tile
      for (int k = lane; k < W.n_tasks; k += 32) {
        const uint2 tk = sm.ptask[k];
        const Layer& L = O.L[task_layer(tk)];
        sm.psrc[k] = L.planes + ((long long)W.w * L.n_tiles + (task_tile(tk) - L.tile_off)) * (kItemBytes / 16);
      }
      __syncwarp();
      u64* pdbg = P.dbg ? P.dbg + ((size_t)si * G + cta) * kDbgRec : nullptr;
      // issue lanes per batch: a batch of nl tasks spans <= nl * (planes per
      // task) <= kMaxSlots FIFO items (see above), so nl = kMaxSlots / planes
      const int nlb = issue_lanes(max(nb.v0, max(nb.v1, nb.v2)));
      for (int k0 = 0; k0 < W.n_tasks; k0 += nlb) {
        const int k = k0 + lane;
        if (lane < nlb && k < W.n_tasks) {
          const uint2 tk = sm.ptask[k];
          const int li = task_layer(tk);
          issue_task(k, fifo + task_before(tk, nb), 0, nb[li], li == 0 ? ps0 : li == 1 ? ps1 : ps2);
        }
        __syncwarp();
      }
      const int n_base = W.cnt[0] * nb.v0 + W.cnt[1] * nb.v1 + W.cnt[2] * nb.v2;
      if (pdbg && lane == 0) pdbg[5] = gclock();
#if DPQ_EXTRA_PREFETCH
      // while the decision is pending (HBM is idle on the small ops), the
      // extra planes of the op's deciding layers go to L2 speculatively: a
      // high decision then streams them from L2
      if (C.mode == MODE_DYNAMIC && !C.force)
        for (int k = lane; k < W.n_tasks; k += 32) {
          const uint2 tk = sm.ptask[k];
          const int li = task_layer(tk);
          const Layer& L = O.L[li];
          if (L.sentinel != 0 || L.xread || nb[li] >= L.h) continue;
          const long long ps = li == 0 ? ps0 : li == 1 ? ps1 : ps2;
          const unsigned char* src = reinterpret_cast<const unsigned char*>(sm.psrc[k]) + (long long)nb[li] * ps;
          for (int q = nb[li]; q < L.h; ++q, src += ps)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(src), "r"((unsigned)kItemBytes) : "memory");
        }
#endif
      // the op's decisions (taken by the reducer warp)
      if (lane == 0) SPIN_UNTIL_NS(sm.dec_op >= oi + 1, "producer decision", oi, 0, 12000000000ull);
      __syncwarp();
      __threadfence_block();
      fin = I3{sm.dec_fin[oi % kDecRing][0], sm.dec_fin[oi % kDecRing][1], sm.dec_fin[oi % kDecRing][2]};
      if (pdbg && lane == 0) pdbg[6] = gclock();
      const I3 ex{fin.v0 - nb.v0, fin.v1 - nb.v1, fin.v2 - nb.v2};
      const int n_ext = W.cnt[0] * ex.v0 + W.cnt[1] * ex.v1 + W.cnt[2] * ex.v2;
      const int nle = issue_lanes(max(ex.v0, max(ex.v1, ex.v2)));
      if (n_ext > 0)
        for (int k0 = 0; k0 < W.n_tasks; k0 += nle) {
          const int k = k0 + lane;
          if (lane < nle && k < W.n_tasks) {
            const uint2 tk = sm.ptask[k];
            const int li = task_layer(tk);
            if (ex[li] > 0)
              issue_task(k, fifo + n_base + task_before(tk, ex), nb[li], ex[li], li == 0 ? ps0 : li == 1 ? ps1 : ps2);
          }
          __syncwarp();
        }
      fifo += n_base + n_ext;
      ++oi;
      // L2 prefetch of the next op's first DPQ_PF_ITEMS base items (FIFO
      // order): HBM keeps streaming through this op's tail (last items,
      // reduction, the next input's latency); the ring's TMA loads then hit L2
      if (DPQ_PF_ITEMS > 0) {
        const int on = (st.y + 1) % (P.n_stages - 2);
        const Op* On = P.ops + on;
        const CtaWork* Wn = On->work + cta;
        const int nt = Wn->n_tasks, t0 = Wn->task0, wn = Wn->w;
        const I3 nbn = base_bits(*On, C);
        for (int k = lane; k < nt; k += 32) {
          const uint2 tk = __ldg(P.tasks + t0 + k);
          const int li = task_layer(tk);
          const int j0 = task_before(tk, nbn);
          if (j0 >= DPQ_PF_ITEMS) continue;
          const Layer& L = On->L[li];
          const unsigned char* src = reinterpret_cast<const unsigned char*>(
              L.planes + ((long long)wn * L.n_tiles + (task_tile(tk) - L.tile_off)) * (kItemBytes / 16));
          const int np = min(nbn[li], DPQ_PF_ITEMS - j0);
          for (int q = 0; q < np; ++q)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(src + (long long)q * L.pstride * 16),
                         "r"((unsigned)kItemBytes) : "memory");
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Consumer warps: one op stage
// ---------------------------------------------------------------------------
// Horner over items [j0, j0 + n) of the FIFO (one 2 KB item per plane) for
// the tile at slot offset: S = 2 S + P_p.
__device__ __forceinline__ float stream_task(Smem& sm, int j0, int n, uint32_t lanereg) {
  const int lane = threadIdx.x & 31;
  const unsigned char* dyn0 = reinterpret_cast<const unsigned char*>(&sm);
  float S = 0.f;
  for (int q = 0; q < n; ++q) {
    const int j = j0 + q;
    const int sl = j % kMaxSlots;
#if DPQ_SEQ_SLEEP > 0
    // the item is not issued yet (the ring is behind): back off instead of a
    // tight LDS loop (MIO slots of the warps that do have data)
    if (lane == 0 && sm.seq[sl] != j) {
      __nanosleep(DPQ_SEQ_SLEEP);
      SPIN_UNTIL_NS((__nanosleep(DPQ_SEQ_SLEEP), sm.seq[sl] == j), "ring sequence", j, sm.seq[sl], 4000000000ull);
    }
#else
    if (lane == 0) SPIN_UNTIL_NS(sm.seq[sl] == j, "ring sequence", j, sm.seq[sl], 4000000000ull);
#endif
    __syncwarp();
    const uint32_t fa = smem_u32(&sm.full[sl]);
    const unsigned fpar = (unsigned)((j / kMaxSlots) & 1);
#if DPQ_SLOT_SLEEP > 0
    if (!mbar_test(fa, fpar))
      SPIN_UNTIL_NS((__nanosleep(DPQ_SLOT_SLEEP), mbar_test(fa, fpar)), "ring slot", j, fpar, 4000000000ull);
#else
    SPIN_UNTIL_NS(mbar_test(fa, fpar), "ring slot", j, fpar, 4000000000ull);
#endif
    const uint4* d = reinterpret_cast<const uint4*>(dyn0 + slot_offset(&sm, sl)) + lane;
    const uint4 d0 = d[0], d1 = d[32], d2 = d[64], d3 = d[96];
    __syncwarp();
    if (lane == 0) mbar_arrive_n(&sm.empty[sl], 1u);
    S = 2.f * S + plane_sum(d0, d1, d2, d3, lanereg);
  }
  return S;
}

__device__ __forceinline__ void cons_op(const Prog& P, Smem& sm, int oi, int op_idx, int n_ops, int si, unsigned gs,
                                        unsigned step_base, int cta, int G, int& fifo, const ECtl& C, u64* dbg) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = oi & 1;
  float* lut = reinterpret_cast<float*>(reinterpret_cast<char*>(&sm) + (kLut - smem_u32(&sm)));
  if (dbg && tid == 0) dbg[0] = gclock();
  // skew bound: this stage writes partials / attention states of parity gs
#if DPQ_STAGE_SLEEP > 0
  if (tid == 0 && !stage_done(P, gs))
    SPIN_UNTIL((__nanosleep(DPQ_STAGE_SLEEP), stage_done(P, gs)), "stage counter", gs, 0);
#else
  if (tid == 0) SPIN_UNTIL(stage_done(P, gs), "stage counter", gs, 0);
#endif
  CSYNC();
  const Op& O = sm.cop[b];
  const CtaWork& W = sm.cw[b];
  const unsigned e_in = step_base + (unsigned)O.in_stage + 1u;
  FeedPre fp;
  fp.pre = false;
  // attention units (the o op): unit u = (head u mod H, chunk u / H) on CTA G - 1 - (u mod G)
  if (O.attn_in && warp < kAttnWarps) {
    const int n_att = P.H * ((C.pos + kAttnChunk) / kAttnChunk);
    for (int u = G - 1 - cta; u < n_att; u += G) attn_unit(P, C, O, sm, u % P.H, u / P.H, warp, lut, e_in, dbg);
  }
  // the next op's descriptor, work and tasks (consumed at its start; warp NW - 1
  // is idle while the input window is awaited)
  if (warp == NW - 1) load_op(P, (op_idx + 1) % n_ops, cta, &sm.cop[b ^ 1], &sm.cw[b ^ 1], sm.ctask[b ^ 1]);
  // input window (other ops: the estimator G rows are loaded while it is awaited)
  if (O.attn_in) {
    feed_prefetch(P, C, O, W, fp);       // G rows in flight while the head states are merged
    attn_merge(P, C, W.w, e_in, sm.xw);
  } else {
    feed_prefetch(P, C, O, W, fp);
    if (O.plain_io) {                    // the caller's x (complete before the launch)
      if (tid < 128) {
        const int c0 = W.w * kWinCols + 4 * tid;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c0 + 4 <= O.cols) v = *reinterpret_cast<const float4*>(P.embed + c0);
        else
          for (int j = 0; j < 4; ++j)
            if (c0 + j < O.cols) (&v.x)[j] = P.embed[c0 + j];
        *reinterpret_cast<float4*>(sm.xw + 4 * tid) = v;
      }
    } else {
      load_window(O.in, O.cols, W.w, e_in, sm.xw);
    }
  }
  CSYNC();
  if (dbg && tid == 0) dbg[1] = gclock();
  // the window's LUT (all warps), then its estimator feeds + statistics
  // (tagged stores, off the CTA's critical path: no CSYNC after them)
  // (DPQ_FEEDS_FIRST: the feeds before the LUT, 1 = every op, 2 = q|k|v and o,
  // whose decision is on the critical path)
  const bool feeds_first = DPQ_FEEDS_FIRST == 1 || (DPQ_FEEDS_FIRST == 2 && (O.inst % 4 == 0 || O.attn_in));
  if (feeds_first) {
    feed_finish(P, C, O, W, fp, sm.xw, gs + 1u);
    if (dbg && lane == 0 && O.feed_rows > 0 && C.mode == MODE_DYNAMIC)
      atomicMax(reinterpret_cast<unsigned long long*>(dbg + 20), gclock());
  }
  lut_build(lut, sm.xw);
  CSYNC();
  if (dbg && tid == 0) dbg[2] = gclock();
  if (!feeds_first) {
    feed_finish(P, C, O, W, fp, sm.xw, gs + 1u);
    if (dbg && lane == 0 && O.feed_rows > 0 && C.mode == MODE_DYNAMIC)
      atomicMax(reinterpret_cast<unsigned long long*>(dbg + 20), gclock());
  }
  const I3 nb = base_bits(O, C);
  const uint32_t lanereg = kLut | ((uint32_t)lane * 4u);
  const size_t par = (size_t)(gs & 1u) * P.slot_half + (size_t)lane * 2;
  const unsigned epoch = gs + 1u;
  const uint2* tasks = sm.ctask[b];
  for (int k = warp; k < W.n_tasks; k += NW) {
    const uint2 tk = tasks[k];
    const int li = task_layer(tk);
    const float S = stream_task(sm, fifo + task_before(tk, nb), nb[li], lanereg);
    add_partial(P.slot + par + (size_t)task_tile(tk) * 64, S, P.err);
  }
  if (dbg && tid == 0) dbg[3] = gclock();
  const int n_base = W.cnt[0] * nb.v0 + W.cnt[1] * nb.v1 + W.cnt[2] * nb.v2;
  // extra planes of the layers that decided high
#if DPQ_DEC_SLEEP > 0
  if (lane == 0 && sm.dec_op < oi + 1)
    SPIN_UNTIL_NS((__nanosleep(DPQ_DEC_SLEEP), sm.dec_op >= oi + 1), "decision", oi, 0, 8000000000ull);
#else
  if (lane == 0) SPIN_UNTIL_NS(sm.dec_op >= oi + 1, "decision", oi, 0, 8000000000ull);
#endif
  __syncwarp();
  __threadfence_block();
  const int* df = sm.dec_fin[oi % kDecRing];
  const I3 ex{df[0] - nb.v0, O.n_layers > 1 ? df[1] - nb.v1 : 0, O.n_layers > 2 ? df[2] - nb.v2 : 0};
  const int n_ext = W.cnt[0] * ex.v0 + W.cnt[1] * ex.v1 + W.cnt[2] * ex.v2;
  if (n_ext > 0) {
    for (int k = warp; k < W.n_tasks; k += NW) {
      const uint2 tk = tasks[k];
      const int li = task_layer(tk);
      if (ex[li] <= 0) continue;
      const float S = stream_task(sm, fifo + n_base + task_before(tk, ex), ex[li], lanereg);
      add_partial(P.slotx + par + (size_t)task_tile(tk) * 64, S, P.err);
    }
  }
  fifo += n_base + n_ext;
  CSYNC();
  if (tid == 0) {
    sm.cons_ops = oi + 1;
    sm.cons_gs = gs + 1;
  }
  if (dbg && tid == 0) dbg[4] = gclock();
}

// ---------------------------------------------------------------------------
// Dual ops (exact estimators, track_exact; estimator.py:30-32, 63-73,
// runtime.py:322-324): every h plane is streamed, so each row has S_l (the l
// base planes) and S_x (the h - l extras) with S_h = 2^(h-l) S_l + S_x, and
// y_h - y_l = s_in span (2^-h S_x + sum x / 2 (2^-h - 2^-l)) (lo cancels,
// quant.py:74-78). Phase 1: every unit's raw sums -> shared memory and the
// CTA's sum of (y_h - y_l)^2 per dual layer -> the layer's packed exact set;
// exact estimators then wait for the full set and decide est > T with est =
// ||y_h - y_l||; phase 2: the outputs with the real bits.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void add_packed_d(u64* w, double v, unsigned* err) {
  long long x = 0;
  if (fabs(v) < 8.0e9) x = llrint(v * kFxPart);
  else atomicOr(err, (unsigned)ERR_RANGE);
  const long long hi = x >> 24, lo = x & 0xffffff;
  const u64 one = 1ull << kCntShift;
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(w), "l"(one + (u64)(hi + kFxBias)) : "memory");
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(w + 1), "l"(one + (u64)(lo + kFxBias)) : "memory");
}

__device__ __forceinline__ void dual_units(const Prog& P, const ECtl& C, const Op& O, Smem& sm, int cta, int G,
                                           const I3& nb, const I3& fin, I3 real, const Epi& E, unsigned epoch,
                                           unsigned e_res) {
  const int lane = threadIdx.x & 31;
  const int half = O.L[0].n_tiles;
  const int n_u = (O.n_units - cta + G - 1) / G;
  double xs[kMaxOpLayers] = {0.0, 0.0, 0.0};
  // phase 1
  for (int i = 0; i < n_u; ++i) {
    const int u = cta + i * G;
    double raw[4];
    if (O.pair) {
      tiles_S(P, O, u, fin.v0 - nb.v0, u + half, fin.v1 - nb.v1, epoch, raw);
    } else {
      const int li = layer_of(O, u);
      tiles_S(P, O, u, fin[li] - nb[li], -1, 0, epoch, raw);
    }
    sm.xraw[i][lane] = make_float4((float)raw[0], (float)raw[1], (float)raw[2], (float)raw[3]);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (t == 1 && !O.pair) break;
      const int li = O.pair ? t : layer_of(O, u);
      const Layer& L = O.L[li];
      if (!L.xread) continue;
      const int r = (O.pair ? u : u - L.tile_off) * 32 + lane;
      if (r >= L.rows) continue;
      const double sp = (double)__ldg(L.span + r);
      const double dy = (double)E.scale * sp *
                        (ldexp(raw[2 * t + 1], -L.h) + 0.5 * (double)E.sx * (ldexp(1.0, -L.h) - ldexp(1.0, -L.l)));
      const double d2 = dy * dy;
      if (li == 0) xs[0] += d2; else if (li == 1) xs[1] += d2; else xs[2] += d2;
    }
  }
  u64* xw = P.xerr + (size_t)(C.n_steps_done & (kCurSlots - 1)) * P.n_xsets * 2;
#pragma unroll
  for (int li = 0; li < kMaxOpLayers; ++li) {
    if (li >= O.n_layers || !O.L[li].xread) continue;
    // this CTA's units of the layer: contribute (possibly 0) iff it has any
    bool mine = false;
    for (int i = 0; i < n_u && !mine; ++i) {
      const int u = cta + i * G;
      mine = O.pair || (u >= O.L[li].tile_off && u < O.L[li].tile_off + O.L[li].n_tiles);
    }
    const double t = wsum(xs[li]);
    if (mine && lane == 0) add_packed_d(xw + 2 * O.L[li].xset, t, P.err);
  }
  // exact estimators: the full set, then est > T (estimator.py:63-73, runtime.py:192)
#pragma unroll
  for (int li = 0; li < kMaxOpLayers; ++li) {
    if (li >= O.n_layers || real[li] >= 0) continue;
    const Layer& L = O.L[li];
    const u64* w = xw + 2 * L.xset;
    uint4 q;
    SPIN_UNTIL((q = ld_tag2(w), (int)(q.y >> 24) == L.xcnt && (int)(q.w >> 24) == L.xcnt), "exact set", L.trace, L.xcnt);
    const double est = sqrt(fmax(partial_total(q), 0.0));
    const int bit = est > L.T ? L.h : L.l;
    real.set(li, bit);
    if (lane == 0 && cta == 0 && L.trace >= 0 && P.n_trace > 0 && C.trace_step < P.max_steps) {
      const size_t o = (size_t)C.trace_step * P.n_trace + L.trace;
      P.tr_bits[o] = (signed char)bit;
      P.tr_est[o] = (float)est;
    }
  }
  __syncwarp();
  // phase 2: the outputs with the real bits
  for (int i = 0; i < n_u; ++i) {
    const int u = cta + i * G;
    const float4 rw = sm.xraw[i][lane];
    auto S_of = [&](int li, float sb, float sx) -> float {
      const Layer& L = O.L[li];
      if (L.xread) return real[li] == L.h ? (float)(ldexp((double)sb, L.h - L.l) + (double)sx) : sb;
      const int ex = fin[li] - nb[li];
      return ex > 0 ? (float)(ldexp((double)sb, ex) + (double)sx) : sb;
    };
    auto bit_of = [&](int li) { const Layer& L = O.L[li]; return L.xread ? (real[li] == L.h ? L.h : L.l) : fin[li]; };
    if (O.pair) {
      const int r = u * 32 + lane;
      if (r < O.L[0].rows) {
        const float S0 = S_of(0, rw.x, rw.y), S1 = S_of(1, rw.z, rw.w);
        const int b0 = bit_of(0), b1 = bit_of(1);
        const float up = E.scale * (__ldg(O.L[0].lo + r) * E.sx + ldexpf(__ldg(O.L[0].span + r), -b0) * (S0 + 0.5f * E.sx));
        const float gt = E.scale * (__ldg(O.L[1].lo + r) * E.sx + ldexpf(__ldg(O.L[1].span + r), -b1) * (S1 + 0.5f * E.sx));
        const float hv = up * (gt / (1.0f + expf(-gt)));                 // runtime.py:368
        if (O.push) st_tag_all(P, O.out + O.L[0].out_off + r, hv, epoch);
        else st_tag(O.out + O.L[0].out_off + r, hv, epoch);
      }
    } else {
      const int li = layer_of(O, u);
      const Layer& L = O.L[li];
      const int r = (u - L.tile_off) * 32 + lane;
      if (r < L.rows) {
        const int o = L.out_off + r;
        const float S = S_of(li, rw.x, rw.y);
        float v = E.scale * (__ldg(L.lo + r) * E.sx + ldexpf(__ldg(L.span + r), -bit_of(li)) * (S + 0.5f * E.sx));
        if (O.add) {                                                            // runtime.py:364, 370
          u64 xr;
          SPIN_UNTIL((xr = ld_relaxed64(O.res_in + o), (unsigned)(xr >> 32) == e_res), "residual", o, e_res);
          v = __uint_as_float((unsigned)xr) + v;
        }
        if (O.push) st_tag_all(P, O.out + o, v, epoch);
        else st_tag(O.out + o, v, epoch);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// The reducer warp: every stage in order; the units of op stages as their
// partials arrive, then one arrival on the stage counter once the consumers
// are done with the stage too.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void reducer(const Prog& P, Smem& sm, int cta, int G, int n_steps, int s0) {
  const int lane = threadIdx.x & 31;
  int oi = 0;
  load_op_async(P, 0, &sm.rop[0]);
  for (int step = 0; step < n_steps; ++step) {
    if (lane == 0) SPIN_UNTIL_NS(sm.step_ready >= step + 1, "reducer step", step, 0, 12000000000ull);
    __syncwarp();
    __threadfence_block();
    const ECtl& C = sm.ctl[step & 1];
    const unsigned step_base = (unsigned)(s0 + step) * (unsigned)P.n_stages;
    for (int si = 0; si < P.n_stages; ++si) {
      const int2 st = P.stages[si];
      const unsigned gs = step_base + (unsigned)si;
      if (st.x == ST_OP) {
        asm volatile("cp.async.wait_all;" ::: "memory");   // this op's descriptor (prefetched)
        __syncwarp();
        const Op& O = sm.rop[oi & 1];
        load_op_async(P, (st.y + 1) % (P.n_stages - 2), &sm.rop[(oi + 1) & 1]);
        // the op's precision decisions, published to the producer (extra
        // planes) and the consumers; entry oi - kDecRing is free: this warp
        // only gets here once the consumers have finished op oi - 1
        const I3 nb = base_bits(O, C);
        I3 fin = nb;
        u64* rdbg = P.dbg ? P.dbg + ((size_t)si * G + cta) * kDbgRec : nullptr;
        if (rdbg && lane == 0) rdbg[16] = gclock();
        float est0 = CUDART_NAN_F;
        I3 real = nb;
        decide_op(P, C, O, sm, nb, fin, cta, step_base, rdbg, &est0, real);
        if (rdbg && lane == 0) rdbg[17] = gclock();
        if (lane == 0) {
          sm.dec_fin[oi % kDecRing][0] = fin.v0;
          sm.dec_fin[oi % kDecRing][1] = fin.v1;
          sm.dec_fin[oi % kDecRing][2] = fin.v2;
          sm.dec_est[oi % kDecRing] = est0;
          __threadfence_block();
          sm.dec_op = oi + 1;
        }
        __syncwarp();
        if (cta < O.n_units) {
          const Epi E = op_epi(P, O, gs + 1u);
          if (rdbg && lane == 0) rdbg[18] = gclock();
          if (lane == 0) SPIN_UNTIL(stage_done(P, gs), "stage counter (reducer)", gs, 0);
          __syncwarp();
          const unsigned epoch = gs + 1u;
          const unsigned e_res = O.add ? step_base + (unsigned)O.res_stage + 1u : 0u;
          const bool dual = C.mode == MODE_DYNAMIC && (O.L[0].xread || (O.n_layers > 1 && O.L[1].xread) ||
                                                       (O.n_layers > 2 && O.L[2].xread));
          if (dual) dual_units(P, C, O, sm, cta, G, nb, fin, real, E, epoch, e_res);
          // the affine epilogue (quant.py:74-78): y = s_in (lo sum x + span 2^-b (S + sum x / 2))
          // descriptor fields in registers before the unit polls: shared-memory
          // reads after a poll queue behind the consumers' LUT loads (MIO)
          const bool o_pair = O.pair != 0, o_push = O.push != 0, o_add = O.add != 0, o_plain = O.plain_io != 0;
          const bool tp1 = P.tp_size == 1;
          u64* const o_out = O.out;
          float* const y_out = P.y_out;
          auto store_out = [&](u64* dst, float v) {
            if (o_push && !tp1) st_tag_all(P, dst, v, epoch);
            else __stcg(dst, ((u64)epoch << 32) | __float_as_uint(v));
          };
          for (int u = cta; !dual && u < O.n_units; u += G) {
            if (o_pair) {
              // unit u: up tile u and gate tile u (runtime.py:366-368)
              const int half = O.L[0].n_tiles;
              const int r = u * 32 + lane;
              float lo0 = 0.f, sp0 = 0.f, lo1 = 0.f, sp1 = 0.f;
              const bool ok = r < O.L[0].rows;
              u64* const dst = o_out + O.L[0].out_off + r;
              if (ok) {
                lo0 = __ldg(O.L[0].lo + r); sp0 = __ldg(O.L[0].span + r);
                lo1 = __ldg(O.L[1].lo + r); sp1 = __ldg(O.L[1].span + r);
              }
              const float2 S = tiles_S(P, O, u, fin.v0 - nb.v0, u + half, fin.v1 - nb.v1, epoch);
              if (ok) {
                const float up = E.scale * (lo0 * E.sx + ldexpf(sp0, -fin.v0) * (S.x + 0.5f * E.sx));
                const float gt = E.scale * (lo1 * E.sx + ldexpf(sp1, -fin.v1) * (S.y + 0.5f * E.sx));
                const float hv = up * (gt / (1.0f + expf(-gt)));                 // runtime.py:368
                store_out(dst, hv);
              }
            } else {
              const int li = layer_of(O, u);
              const Layer& L = O.L[li];
              const int r = (u - L.tile_off) * 32 + lane;
              const bool ok = r < L.rows;
              const int o = L.out_off + r;
              const int bl = fin[li];
              const u64* const res_p = O.res_in + o;
              float lo = 0.f, sp = 0.f, res = 0.f;
              if (ok) {
                lo = __ldg(L.lo + r);
                sp = __ldg(L.span + r);
              }
              u64 xr = 0;
              if (o_add && ok) xr = ld_relaxed64(res_p);
              const float S = tiles_S(P, O, u, bl - nb[li], -1, 0, epoch).x;
              if (ok) {
                float v = E.scale * (lo * E.sx + ldexpf(sp, -bl) * (S + 0.5f * E.sx));
                if (o_add) {                                                            // runtime.py:364, 370
                  if ((unsigned)(xr >> 32) != e_res)
                    SPIN_UNTIL((xr = ld_relaxed64(res_p), (unsigned)(xr >> 32) == e_res), "residual", o, e_res);
                  res = __uint_as_float((unsigned)xr);
                  v = res + v;
                }
                if (o_plain) y_out[o] = v;
                else store_out(o_out + o, v);
              }
            }
            if (rdbg && lane == 0 && u == cta) rdbg[19] = gclock();
          }
        }
        ++oi;
        u64* dbg = P.dbg ? P.dbg + ((size_t)si * G + cta) * kDbgRec : nullptr;
        if (dbg && lane == 0) dbg[7] = gclock();
      }
      __syncwarp();
      if (lane == 0) {
#if DPQ_CONS_SLEEP > 0
        if (sm.cons_gs < gs + 1)
          SPIN_UNTIL_NS((__nanosleep(DPQ_CONS_SLEEP), sm.cons_gs >= gs + 1), "consumer stage", gs, sm.cons_gs,
                        12000000000ull);
#else
        SPIN_UNTIL_NS(sm.cons_gs >= gs + 1, "consumer stage", gs, sm.cons_gs, 12000000000ull);
#endif
        // the zeroed partial words (tiles_S) before the arrival: reused two stages on
#if DPQ_REL_ARRIVE
        if (P.tp_size == 1) {      // one release reduction (the warp's stores ordered by __syncwarp)
          asm volatile("red.release.gpu.global.add.u64 [%0], %1;" :: "l"(P.bar), "l"(1ull) : "memory");
        } else {
          __threadfence_system();  // this stage's peer stores before the arrival
          red_all(P, P.bar, 1ull);
        }
#else
        __threadfence();
        if (P.tp_size > 1) __threadfence_system();   // this stage's peer stores before the arrival
        red_all(P, P.bar, 1ull);
#endif
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// Head stage: final RMSNorm + lm_head logits (runtime.py:372), greedy argmax
// (runtime.py:405-408) and the end-of-step control update (runtime.py:373-380).
// ---------------------------------------------------------------------------
__device__ __noinline__ void head_stage(const Prog& P, const ECtl& C, Smem& sm, float* xs, int cta, int G,
                                        unsigned e_final) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the final residual (tagged) -> shared memory (every pair of words of a
  // thread polled in one round trip), then the sum of squares in fixed order
  {
    const int npair = P.d / 2;
    for (int p0 = tid; p0 < npair; p0 += NT * 8) {
      uint4 v[8];
      bool ok;
      SPIN_UNTIL((ok = true, [&]() {
                    for (int k = 0; k < 8; ++k) {
                      const int p = p0 + k * NT;
                      if (p < npair) {
                        v[k] = ld_tag2(P.xfinal + 2 * p);
                        ok &= v[k].y == e_final && v[k].w == e_final;
                      }
                    }
                  }(), ok), "final x", p0, e_final);
      for (int k = 0; k < 8; ++k) {
        const int p = p0 + k * NT;
        if (p < npair) {
          xs[2 * p] = __uint_as_float(v[k].x);
          xs[2 * p + 1] = __uint_as_float(v[k].z);
        }
      }
    }
    if ((P.d & 1) && tid == 0) {
      u64 x;
      SPIN_UNTIL((x = ld_relaxed64(P.xfinal + P.d - 1), (unsigned)(x >> 32) == e_final), "final x", P.d - 1, e_final);
      xs[P.d - 1] = __uint_as_float((unsigned)x);
    }
  }
  CSYNC();
  double q = 0.0;
  for (int i = tid; i < P.d; i += NT) {
    const float v = xs[i];
    q += (double)v * v;
  }
  q = wsum(q);
  if (lane == 0) sm.red[warp] = q;
  CSYNC();
  double s2 = 0.0;
  for (int w = 0; w < NW; ++w) s2 += sm.red[w];
  const float inv = (float)(1.0 / sqrt(s2 / (double)P.d + (double)P.eps));
  for (int v = cta * NW + warp; v < P.vocab; v += G * NW) {
    const float* row = P.lm + (size_t)v * P.d;
    float a = 0.f;
    if ((P.d & 3) == 0) {
      for (int i = lane * 4; i < P.d; i += 128) {
        const float4 w4 = __ldg(reinterpret_cast<const float4*>(row + i));
        const float4 x4 = *reinterpret_cast<const float4*>(xs + i);
        a += w4.x * x4.x + w4.y * x4.y + w4.z * x4.z + w4.w * x4.w;
      }
    } else {
      for (int k = lane; k < P.d; k += 32) a += row[k] * xs[k];
    }
    a = wsum(a);
    if (lane == 0) P.logits[v] = a * inv;
  }
  // exact errors of the step's dual layers (track_exact / exact estimators) -> trace
  if (cta == 0 && C.mode == MODE_DYNAMIC && P.n_trace > 0 && C.trace_step < P.max_steps) {
    const u64* xw = P.xerr + (size_t)(C.n_steps_done & (kCurSlots - 1)) * P.n_xsets * 2;
    for (int j = tid; j < P.n_xsets; j += NT) {
      const int2 xs = P.xsets[j];
      uint4 q;
      SPIN_UNTIL((q = ld_tag2(xw + 2 * j), (int)(q.y >> 24) == xs.y && (int)(q.w >> 24) == xs.y), "exact set (head)", j, xs.y);
      const float xe = (float)sqrt(fmax(partial_total(q), 0.0));
      const size_t o = (size_t)C.trace_step * P.n_trace + (xs.x & 0xffff);
      P.tr_exact[o] = xe;
      if (xs.x >> 16) P.tr_est[o] = xe;         // exact estimators: the estimate is the exact error
    }
  }
#if DPQ_REL_ARRIVE
  CSYNC();
  if (tid == 0) {              // the CTA's logits before the count; the last CTA acquires the others'
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(P.head_cnt) : "memory");
    sm.head_last = old == (unsigned)G - 1;
  }
  CSYNC();
  if (!sm.head_last) return;
#else
  __threadfence();
  CSYNC();
  if (tid == 0) sm.head_last = atomicAdd(P.head_cnt, 1u) == (unsigned)G - 1;
  CSYNC();
  if (!sm.head_last) return;
  __threadfence();
#endif
  float best = -CUDART_INF_F;
  int bi = 0x7fffffff;
  for (int i = tid; i < P.vocab; i += NT) {
    const float z = __ldcg(P.logits + i);
    if (z > best || (z == best && i < bi)) { best = z; bi = i; }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float zb = __shfl_xor_sync(0xffffffffu, best, off);
    const int ib = __shfl_xor_sync(0xffffffffu, bi, off);
    if (zb > best || (zb == best && ib < bi)) { best = zb; bi = ib; }
  }
  if (lane == 0) { sm.head_v[warp] = best; sm.head_i[warp] = bi; }
  CSYNC();
  if (tid == 0) {
    for (int w = 1; w < NW; ++w)
      if (sm.head_v[w] > best || (sm.head_v[w] == best && sm.head_i[w] < bi)) { best = sm.head_v[w]; bi = sm.head_i[w]; }
    if (bi == 0x7fffffff) bi = 0;       // all-NaN logits
    P.head_cnt[0] = 0u;
    ECtl* c = P.ctl;
    const int dyn = C.mode == MODE_DYNAMIC;
    c->token = bi;
    if (C.n_steps_done < P.max_steps) P.tok_log[C.n_steps_done] = bi;
    c->pos = C.pos + 1;
    if (dyn) c->trace_step = C.trace_step + 1;
    if (dyn || C.prime) {
      c->rot = C.rot + 1;
      c->has_prev = 1;
    }
    // (the release store orders this thread's control writes before the count)
    asm volatile("st.release.gpu.global.s32 [%0], %1;" :: "l"(&c->n_steps_done), "r"(C.n_steps_done + 1) : "memory");
  }
}

// BEGIN: the step's control block (-> ctl[step & 1]), zeroing of the
// accumulator slots used two steps ahead, x = embed[token] (runtime.py:345)
// as a tagged vector.
__device__ __forceinline__ void begin_stage(const Prog& P, Smem& sm, int cta, int G, int step, int expect_done,
                                            unsigned gs) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    SPIN_UNTIL(ld_acq_s32(&P.ctl->n_steps_done) >= expect_done, "step control", expect_done, 0);
    SPIN_UNTIL(stage_done(P, gs), "stage counter", gs, 0);
  }
  CSYNC();
  ECtl& Cw = sm.ctl[step & 1];
  {
    const int* src = reinterpret_cast<const int*>(P.ctl);
    int* dst = reinterpret_cast<int*>(&Cw);
    if (tid < (int)(sizeof(ECtl) / 4)) dst[tid] = __ldcg(src + tid);
  }
  CSYNC();
  if (P.gemv_mode > 0 && tid == 0) {      // single-op program: this call's mode / bit
    Cw.mode = P.gemv_mode;
    Cw.force = P.gemv_force;
    Cw.token = 0;
    Cw.trace_step = 0;
    sm.gemv_bits[0] = (signed char)P.gemv_bit;
    Cw.forced_bits = sm.gemv_bits;
  }
  CSYNC();
  if (tid == 0) {
    __threadfence_block();
    sm.step_ready = step + 1;                   // the producer and reducer may run this step
  }
  const ECtl& C = Cw;
  {  // estimator-set slots used two steps / rotations ahead
    u64* a = P.fpart + (size_t)((C.n_steps_done + 2) & (kCurSlots - 1)) * P.set_stride;
    u64* z = P.fpart + (size_t)(kCurSlots + ((C.rot + 1) & (kPrevSlots - 1))) * P.set_stride;
    for (long long i = cta * NT + tid; i < P.set_stride; i += G * NT) { a[i] = 0; z[i] = 0; }
    u64* xz = P.xerr + (size_t)((C.n_steps_done + 2) & (kCurSlots - 1)) * P.n_xsets * 2;
    for (int i = cta * NT + tid; i < 2 * P.n_xsets; i += G * NT) xz[i] = 0;
  }
  for (int i = cta * NT + tid; i < P.d; i += G * NT) st_tag(P.xe + i, __ldg(P.embed + (size_t)C.token * P.d + i), gs + 1u);
}

// ST_OUT (single-op programs): the op's tagged output -> plain floats, the
// decision / estimate of its first layer, then the step count (last CTA).
__device__ __noinline__ void out_stage(const Prog& P, const ECtl& C, Smem& sm, int cta, int G, unsigned e_out,
                                       int oi_last) {
  const int tid = threadIdx.x;
  const u64* out = P.ops[0].out;
  if (!P.ops[0].plain_io)
    for (int i = cta * NT + tid; i < P.out_rows; i += G * NT) {
      u64 x;
      SPIN_UNTIL((x = ld_relaxed64(out + i), (unsigned)(x >> 32) == e_out), "gemv output", i, e_out);
      P.y_out[i] = __uint_as_float((unsigned)x);
    }
  if (cta == 0 && tid == 0) {
    const int e = (oi_last + kDecRing) % kDecRing;
    if (P.bit_out) *P.bit_out = sm.dec_fin[e][0];
    if (P.est_out) *P.est_out = sm.dec_est[e];
  }
  __threadfence();
  CSYNC();
  if (tid == 0) sm.head_last = atomicAdd(P.head_cnt, 1u) == (unsigned)G - 1;
  CSYNC();
  if (!sm.head_last || tid != 0) return;
  __threadfence();
  P.head_cnt[0] = 0u;
  asm volatile("st.release.gpu.global.s32 [%0], %1;" :: "l"(&P.ctl->n_steps_done), "r"(C.n_steps_done + 1) : "memory");
}

// ---------------------------------------------------------------------------
// The kernel: n_steps decode steps (greedy token feedback on the device when
// n_steps > 1; the host writes the token / mode of a single step).
// ---------------------------------------------------------------------------
#ifndef DPQ_MAXNREG
#define DPQ_MAXNREG 168
#endif
extern "C" __global__ void __maxnreg__(DPQ_MAXNREG) engine_kernel(const Prog Pk, int n_steps) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int cta = blockIdx.x, G = gridDim.x, tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    sm.prog = Pk;
    sm.dec_op = 0;
    sm.cons_ops = 0;
    sm.cons_gs = 0;
    sm.step_ready = 0;
    // ring slots: below the LUT (after Smem) and above its zero row
    const uint32_t base = smem_u32(smem_raw);
    uint32_t lo = (base + (uint32_t)sizeof(Smem) + 127u) & ~127u;
    int n = 0;
    while (lo + kItemBytes <= kLut && n < kMaxSlots) { sm.slot_off[n++] = lo - base; lo += kItemBytes; }
    uint32_t hi = kLut + kLutBytes;
    while (hi + kItemBytes <= base + (uint32_t)Pk.smem_dyn && n < kMaxSlots) {
      sm.slot_off[n++] = hi - base;
      hi += kItemBytes;
    }
    if (n < kMaxSlots) __trap();        // host sizing guarantees kMaxSlots ring slots
    for (int q = 0; q < kMaxSlots; ++q) {
      mbar_init(&sm.full[q], 1);
      mbar_init(&sm.empty[q], 1);
      sm.seq[q] = -1;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const Prog& P = sm.prog;
  const int s0 = __ldcg(&P.ctl->n_steps_done);   // steps completed before this launch
  if (warp == kProdWarp) {
    producer(P, sm, cta, G, n_steps, s0);
    return;
  }
  if (warp == kRedWarp) {
    reducer(P, sm, cta, G, n_steps, s0);
    return;
  }
  float* lut = reinterpret_cast<float*>(smem_raw + (kLut - smem_u32(smem_raw)));
  const int n_ops = P.n_stages - 2;
  if (warp == 0) load_op(P, 0, cta, &sm.cop[0], &sm.cw[0], sm.ctask[0]);
  int oi = 0, fifo = 0;
  for (int step = 0; step < n_steps; ++step) {
    const unsigned step_base = (unsigned)(s0 + step) * (unsigned)P.n_stages;
    for (int si = 0; si < P.n_stages; ++si) {
      const int2 st = P.stages[si];
      const unsigned gs = step_base + (unsigned)si;
      u64* dbg = P.dbg ? P.dbg + ((size_t)si * G + cta) * kDbgRec : nullptr;
      if (st.x == ST_OP) {
        cons_op(P, sm, oi, st.y, n_ops, si, gs, step_base, cta, G, fifo, sm.ctl[step & 1], dbg);
        ++oi;
      } else {
        if (dbg && tid == 0) dbg[0] = gclock();
        if (st.x == ST_BEGIN) begin_stage(P, sm, cta, G, step, s0 + step, gs);
        else if (st.x == ST_OUT) out_stage(P, sm.ctl[step & 1], sm, cta, G, step_base + (unsigned)P.out_op_stage + 1u, oi - 1);
        else head_stage(P, sm.ctl[step & 1], sm, lut, cta, G, step_base + (unsigned)P.final_stage + 1u);
        CSYNC();
        if (tid == 0) sm.cons_gs = gs + 1;
        if (dbg && tid == 0) dbg[4] = gclock();
      }
    }
  }
}
}  // namespace eng
}  // namespace dpq
