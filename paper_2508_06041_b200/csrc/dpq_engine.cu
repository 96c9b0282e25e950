// Persistent decode-step engine for sm_100a (the fast path of dpq_session).
//
// One cooperative kernel runs whole decode steps (reference DecodeEngine.step,
// runtime.py:330-381) on one CTA per SM. A step is a fixed list of stages
//   BEGIN | per block: QKV  ATTN  O  UPGATE  DOWN | HEAD
// separated by a grid barrier (monotonic arrival counter). Per op:
//
//  * precision selection (runtime.py:184-193, estimator.py:35-60) costs no
//    extra pass and no extra grid sync: the estimator's G.v partials and the
//    input statistics (sum, sum of squares) are accumulated by the PRODUCER of
//    the op's input, tile by tile, in its epilogue, into fixed-point int64
//    accumulators (deterministic). Every CTA of the consuming op reads the
//    completed accumulators after the barrier and takes the identical
//    decision est > T (strict, runtime.py:192) before streaming any plane it
//    depends on;
//  * the any-precision GEMV streams only planes 0..b-1 of the nested store
//    (quant.py:74): base planes (known before the decision) are split evenly
//    over the grid at (tile, window) granularity; a layer that decides high
//    adds its extra planes [nb, fin) for the same groups of the same CTA;
//    per item a warp does 64 conflict-free byte-LUT lookups (8 weight bits
//    per LDS);
//  * one TMA producer warp per CTA streams (run, plane) bulk copies into a
//    shared-memory ring (mbarrier full / empty per slot) that runs ahead
//    across op boundaries: the next op's base planes are issued before the
//    barrier, its extra planes once the decision is published;
//  * reduce unit u (a tile, or an up|gate tile pair) belongs to CTA u mod G,
//    which sums its window partials in fixed window order and applies the
//    affine epilogue
//    y = s_in * (lo * sum x + span 2^-b (S + sum x / 2)) (exact restatement of
//    quant.py:74-78 @ x), residual add / SiLU(gate)*up (runtime.py:364-370),
//    and feeds the next estimators.
#include "dpq_common.cuh"

// Consumer-only CTA barrier (the producer warp never joins).
#define CSYNC() asm volatile("bar.sync 1, %0;" :: "n"(dpq::eng::NT) : "memory")

namespace dpq {
namespace eng {

constexpr int NT = 480;            // consumer threads per CTA (warps 0..14): 16 warps in all -> 128 registers
constexpr int NW = NT / 32;        // consumer warps
constexpr int NTB = NT + 32;       // block: consumers + one TMA producer warp (warp 15)
constexpr int kSlotTiles = 8;      // tiles per ring slot (one plane of up to 8 consecutive tiles)
constexpr int kSlotBytes = kSlotTiles * 2048;
constexpr int kMaxSlots = 8;       // ring slots (power of two: index arithmetic by shifts)
constexpr int kMaxRuns = 96;       // (layer, window, <= 8 tiles) runs per op per CTA
constexpr int kMaxTiles = 128;     // tasks whose parked base sums live in shared memory
// Estimator accumulator element i of a set (and each input-statistics word)
// lives at word i * kAccSpread: one 128-byte L2 line per element, so the
// fixed-point red.adds every output tile sends to the same k + 1 elements do
// not serialize on a handful of lines. (Replicas per element, summed by the
// deciding warps, measured slower: the decision's loads are on the critical path.)
constexpr int kAccSpread = 16;
constexpr int kMaxTasks = 384;     // (tile, window) groups per CTA and op; parked sums of tasks
                                   // [kMaxTiles, kMaxTasks) go to a per-CTA global scratch (Prog.park)

constexpr int kDbgRec = 128;   // debug record per (stage, CTA): [0,8) phase stamps, [8,88) 5 per consumer warp, [88,96) producer, [96,128) clock64 sub-stamps
constexpr double kFxSum = 4294967296.0;       // 2^32: sum v
constexpr double kFxSq = 16777216.0;          // 2^24: sum v^2

enum { ST_BEGIN = 0, ST_OP = 1, ST_ATTN = 2, ST_HEAD = 3, ST_EMIT = 4 };
enum { SRC_IMM = 0, SRC_PREV_STEP = 1, SRC_PREV_BLOCK = 2 };
enum { FEED_CUR = 0, FEED_CURFB = 1, FEED_PREV = 2 };

struct Layer {
  const uint4* planes;
  long long pstride;       // uint4 per plane
  const float* lo;
  const float* span;
  int rows, n_tiles, tile_off, out_off;
  int l, h, prefill_bit;
  int sentinel;            // 0 estimate, 1 low (T = +inf), 2 high (T = -inf)
  int est;                 // EST_NONE / EST_LINEAR / EST_PROJECTION
  int src;                 // SRC_*
  int k, fb;               // projection rank, fixed-point fraction bits of G.v
  int acc;                 // offset of the accumulator set (k + 1 int64) in an acc slot
  int trace;               // trace column
  double T, slope, intercept;
  double fbscale;          // 2^-fb
};

struct alignas(16) Op {
  Layer L[kMaxOpLayers];
  int n_layers;
  int cols, n_win, n_tiles;
  int rms;                 // input RMS-normalised (runtime.py:383-384)
  int pair;                // up|gate SiLU pair epilogue -> h
  int add;                 // residual add into out
  int in_inst, out_inst;   // vector instances (stats, feeds); out_inst < 0: none
  const float* in;
  float* out;
};

static_assert(sizeof(Op) % 16 == 0, "Op is copied to shared memory in 16-byte words");

// Producer-side estimator feed of one vector instance.
struct Feed {
  const uint4* Gt;         // tile-blocked G^T (see host), nullptr for linear
  int f16, k, kpad, fb;
  int acc;                 // accumulator set offset
  int kind;                // FEED_*
};

struct Prog {
  int n_stages;
  const int2* stages;      // (kind, index)
  const Op* ops;
  const int* feed_begin;   // [n_inst + 1]
  const Feed* feeds;
  int n_inst;
  int d, H, KV, hd, dkv, f, vocab, seq_cap, n_blocks;
  float eps;
  const float* embed;
  const float* lm;
  const float* cosv;
  const float* sinv;
  float* x;
  float* qkv;
  float* attn;
  float* h;
  float* logits;
  float* const* kc;        // [n_blocks] -> [seq_cap][dkv]
  float* const* vc;
  unsigned long long* slot;  // [max_win][slot_stride]: float S | epoch << 32 (single-copy atomic)
  float* slot_extra;
  int slot_stride;
  int slot_max_win;
  float* attn_part;        // [H][max_chunks][hd + 2]
  float* park;             // [G][kMaxTasks - kMaxTiles][32] parked base sums beyond the shared table
  unsigned* attn_cnt;      // [KV]
  int attn_max_chunks;
  int attn_emit;           // attention emits its heads' tiles (head_dim % 32 == 0), else an EMIT stage
  unsigned* head_cnt;
  long long* acc;          // [5][acc_stride]: cur0 cur1 prev0 prev1 prev2
  int acc_stride;
  long long* vstat;        // [2][n_inst][2]
  unsigned long long* bar;
  signed char* tr_bits;
  float* tr_est;
  int n_trace, max_steps;
  int* tok_log;
  struct ECtl* ctl;
  int smem_dyn;             // dynamic shared memory bytes of the launch
  int upper_slots;          // ring slots above the LUT too
  unsigned long long* dbg; // optional per-stage timestamps [stages][grid][kDbgRec]
};

struct ECtl {
  int mode;                // MODE_PREFILL / MODE_DYNAMIC
  int token;
  int force;
  int pos;
  int trace_step;
  int has_prev;
  int prime;
  int async_prev_block;
  int n_steps_done;        // all steps since reset (cur slot parity)
  int prev_w, prev_r, prev_z;
  const signed char* forced_bits;
  unsigned long long bar_base;   // barrier arrivals completed before this launch / CTA count
};

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_nc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void l1_prefetch(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" :: "l"(p));
}
__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acq64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add64(long long* p, long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gclock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Spin-wait watchdog: a wait beyond 4 s records (line, block, thread, a, b)
// in mapped host memory (dpq_engine_diag) and traps (a launch error instead of
// a hang). No call, so nothing is spilled around the polling loops.
__device__ unsigned long long* g_diag = nullptr;
__device__ volatile int* g_prog = nullptr;     // optional mapped progress words [grid][4] (debug)
#ifdef DPQ_PROFILE_WARPS
#define CSTAMP(st, i) do { if (st) (st)[96 + (i)] = clock64(); } while (0)
#else
#define CSTAMP(st, i) do { } while (0)
#endif
#ifdef DPQ_ENGINE_TRACE
#define PROGRESS(slot, v) do { if (g_prog) g_prog[blockIdx.x * 4 + (slot)] = (v); } while (0)
#define WSTATE(v) do { if (lane == 0) sm.wstate[warp] = (v); } while (0)
#else
#define PROGRESS(slot, v) do { } while (0)
#define WSTATE(v) do { } while (0)
#endif
#define hang(what, a, b)                                                                   \
  do {                                                                                     \
    if (g_diag) {                                                                          \
      volatile unsigned long long* d_ = g_diag;                                            \
      d_[1] = (unsigned long long)__LINE__; d_[2] = blockIdx.x; d_[3] = threadIdx.x;       \
      d_[4] = (unsigned long long)(long long)(a); d_[5] = (unsigned long long)(long long)(b); \
      __threadfence_system(); d_[0] = 1ull; __threadfence_system();                        \
    }                                                                                      \
    __trap();                                                                              \
  } while (0)
// Poll cheaply; read the (slow) global timer only every 4096 polls.
#define SPIN_UNTIL_NS(cond, what, a, b, NS)                                                \
  do {                                                                                     \
    unsigned n_ = 0;                                                                       \
    unsigned long long t0_ = 0;                                                            \
    while (!(cond)) {                                                                      \
      if ((++n_ & 4095u) == 0) {                                                           \
        const unsigned long long t_ = gclock();                                            \
        if (t0_ == 0) t0_ = t_;                                                            \
        else if (t_ - t0_ > (NS)) hang(what, a, b);                                         \
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
__device__ __forceinline__ long long fx(double v, double scale) { return llrint(v * scale); }
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
#define ENG_LDS(dst, addr, IMM) asm("ld.shared.f32 %0, [%1+%2];" : "=f"(dst) : "r"(addr), "n"(IMM))

__device__ __forceinline__ float plane_sum(const uint4 d0, const uint4 d1, const uint4 d2, const uint4 d3,
                                           uint32_t lanereg) {
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

// LUT of one 512-column window: row e, slot g = sum_{t: bit t of e} x[8g + t];
// row 256 = 0 (target of the wrapped "e - 1" encoding for e = 0). Thread u <
// 256 builds rows [64 q, 64 q + 64) of group g (u = 64 q + g) straight from
// the input in global memory (lut_load issues the loads, lut_store writes
// the rows once they arrived; no staging, no barrier in between).
struct LutSrc { float4 a, b; };
__device__ __forceinline__ LutSrc lut_load(const float* x, int cols, int w) {
  LutSrc r;
  r.a = r.b = make_float4(0.f, 0.f, 0.f, 0.f);
  const int u = threadIdx.x;
  if (u < 256) {
    const int c0 = w * kWinCols + 8 * (u & 63);
    if (c0 + 8 <= cols) {
      r.a = __ldcg(reinterpret_cast<const float4*>(x + c0));
      r.b = __ldcg(reinterpret_cast<const float4*>(x + c0 + 4));
    } else {
      float t[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) t[j] = c0 + j < cols ? __ldcg(x + c0 + j) : 0.f;
      r.a = make_float4(t[0], t[1], t[2], t[3]);
      r.b = make_float4(t[4], t[5], t[6], t[7]);
    }
  }
  return r;
}
__device__ __forceinline__ void lut_store(float* lut, const LutSrc& x) {
  const int u = threadIdx.x;
  if (u >= 256) return;
  const int g = u & 63, q = u >> 6;
  const float xs[4] = {x.a.x, x.a.y, x.a.z, x.a.w};
  float L[16];
  L[0] = 0.f;
#pragma unroll
  for (int n = 1; n < 16; ++n) {
    const int low = n & (-n);
    L[n] = L[n ^ low] + xs[__ffs(low) - 1];
  }
#pragma unroll
  for (int mm = 0; mm < 4; ++mm) {
    const int m = 4 * q + mm;
    float H = 0.f;
    if (m & 1) H += x.b.x;
    if (m & 2) H += x.b.y;
    if (m & 4) H += x.b.z;
    if (m & 8) H += x.b.w;
#pragma unroll
    for (int i = 0; i < 16; ++i) lut[(16 * m + i) * kGroups + g] = L[i] + H;
  }
  if (u < 64) lut[256 * kGroups + u] = 0.f;
}

// ---------------------------------------------------------------------------
// Per-op work of one CTA.
// A group is (32-row tile t, 512-column window w), linear index g = w * n_tiles
// + t (window-major). Groups are split over the grid by their base planes
// (known before the decision), CTA c owning [ga, gb) starting at the first
// group at or after item c*N/G. The range is cut into runs of <= 8 tiles of
// one layer inside one window. The TMA producer warp streams, per run and
// plane, one bulk copy of the run's tiles into a 16 KB ring slot: base planes
// [0, nb) of all runs (window ascending), then - once the decision is
// published - extra planes [nb, fin) of the runs whose layer decided high
// (window descending, so the LUT changes at most three times). Consumer task
// (run, tile) goes to warp k % NW; S is accumulated per tile by Horner over
// planes (S_{p+1} = 2 S_p + P_p), the base part parked in shared memory.
// ---------------------------------------------------------------------------
constexpr uint32_t kLut = 0x20000;   // the window LUT (absolute shared address)

struct Work {
  int nb[kMaxOpLayers], fin[kMaxOpLayers];
  int ga, gb;
  int valid;
};

struct Run {
  short li, w;
  short t0, nt;            // op tiles [t0, t0 + nt)
  short k0;                // first tile index inside the CTA range (parking slot)
  short pad;
};

struct RunList {
  int n;
  Run r[kMaxRuns];
};

struct Smem {
  Prog prog;               // program descriptor (kernel parameter copy)
  ECtl ctl;                // control block of the current step (read at BEGIN)
  Op op[2];                // consumer copies of the current / next op descriptors
  Work work[2];            // consumer work of the current / next op
  RunList runs;            // consumer run list of the current op
  Op pop;                  // producer copy of the op it streams
  Work pw;                 // producer work
  RunList pruns;           // producer run list
  short pfo[kMaxRuns];     // producer scratch (FIFO offsets / task table it does not need)
  unsigned char ptask[kMaxTasks];
  unsigned long long full[kMaxSlots], empty[kMaxSlots];   // ring mbarriers
  volatile int seq[kMaxSlots];       // FIFO index armed in each slot (phase disambiguation)
  unsigned slot_off[kMaxSlots];      // slot byte offset from the dynamic smem base
  int n_slots;
  volatile int dec_op;               // op counter whose decision is published
  int runs_op;                       // op counter whose base runs / FIFO offsets are in runs, fo_bo, last
  volatile int step_ready;           // step whose control block consumers have loaded
  volatile int cons_op, cons_j;      // consumer progress (watchdog diagnostics)
  unsigned long long* stamp;         // current stage's timestamps (profiling) or nullptr
  volatile int wstate[NW];           // per consumer warp: item it waits for * 16 + state
  int dec_fin[2][kMaxOpLayers];      // published final bits (op counter parity)
  float scale, sx;         // op input scale (1/rms or 1) and sum of raw input
  int last;                // base FIFO items of the current op (op stage) / last-arriver flag
  int n_ext_items, t_ext;  // extra FIFO items / extra tasks of the current op (after the decision)
  double red[32];
  float head_v[NW];
  int head_i[NW];
  float sbuf[kMaxTiles][32];         // base-pass S of tiles whose layer has extra planes
  short fo_bo[kMaxRuns], fo_eo[kMaxRuns], fo_xt[kMaxRuns];
  unsigned char task_rb[kMaxTasks], task_rx[kMaxTasks];   // run of each base / extra task (kMaxRuns <= 255)
  int vtile[kMaxTiles];              // reduce: emit tile of the CTA's i-th unit (values in sbuf)
};

__device__ __forceinline__ int layer_of(const Op& O, int t) {
  int li = 0;
  while (li + 1 < O.n_layers && t >= O.L[li + 1].tile_off) ++li;
  return li;
}

// First group whose first base item is >= item i.
__device__ __forceinline__ int group_at(const Op& O, const int* nb, int wsum, int i) {
  const int w = i / wsum;
  int r = i - w * wsum;
  for (int li = 0; li < O.n_layers; ++li) {
    const int seg = O.L[li].n_tiles * nb[li];
    if (r < seg) return w * O.n_tiles + O.L[li].tile_off + (r + nb[li] - 1) / nb[li];
    r -= seg;
  }
  return (w + 1) * O.n_tiles;
}

// Base planes per layer for the step mode (known before the decision).
__device__ __forceinline__ int base_bit(const Layer& L, const ECtl& C) {
  if (C.mode == MODE_PREFILL) return L.prefill_bit;
  if (C.force && L.trace >= 0) return C.forced_bits[L.trace];
  if (L.sentinel == 2) return L.h;
  return L.l;
}

// Work of CTA cta: lanes 0..1 of the calling warp compute ga / gb in parallel.
__device__ __forceinline__ void build_work_warp(const Op& O, const ECtl& C, int cta, int G, Work& W) {
  const int lane = threadIdx.x & 31;
  // base bits straight into the (shared-memory) work record: a dynamically
  // indexed local array would live in local memory
  const int nbl = lane < O.n_layers ? base_bit(O.L[lane], C) : 0;
  if (lane < O.n_layers) {
    W.nb[lane] = nbl;
    W.fin[lane] = nbl;
  }
  const int wtot = wsum(lane < O.n_layers ? O.L[lane].n_tiles * nbl : 0);
  __syncwarp();
  const int* nb = W.nb;
  const unsigned N = (unsigned)wtot * (unsigned)O.n_win;   // host guarantees N * G < 2^32
  if (lane < 2) {
    int item;
    if (O.n_win <= G) {
      // window-aligned: CTAs [ceil(w G / n_win), ceil((w + 1) G / n_win)) share
      // window w (one LUT per CTA, no rebuild), its items split evenly
      const int w = (int)((unsigned)cta * (unsigned)O.n_win / (unsigned)G);
      const int cb = (w * G + O.n_win - 1) / O.n_win, ce = ((w + 1) * G + O.n_win - 1) / O.n_win;
      const int m = ce - cb, idx = cta - cb + lane;
      item = w * wtot + (int)((unsigned)idx * (unsigned)wtot / (unsigned)m);
    } else {
      item = (int)(N * (unsigned)(cta + lane) / (unsigned)G);
    }
    const int g = group_at(O, nb, wtot, item);
    if (lane == 0) W.ga = g;
    else W.gb = g;
  }
}

// Warp-parallel run list + base FIFO offsets + task -> run table of work W
// (the serial loops were a dependent chain of shared-memory round trips,
// ~1-3 us per op). Segments = (window, layer) pieces of [ga, gb), one per
// lane (<= 32: host sizing keeps CTA ranges within a few windows); runs of
// <= kSlotTiles tiles per segment; returns the number of base items.
__device__ int build_runs_warp(const Op& O, const Work& W, RunList& R, short* fo_bo, unsigned char* task_r) {
  const int lane = threadIdx.x & 31;
  const int nt = O.n_tiles;
  if (W.ga >= W.gb) {
    if (lane == 0) R.n = 0;
    __syncwarp();
    return 0;
  }
  const int wa = W.ga / nt, wb = (W.gb - 1) / nt;
  const int S = (wb - wa + 1) * O.n_layers;
  if (S > 32) __trap();                 // host sizing guarantees this cannot happen
  int lo = 0, len = 0, nr = 0, items = 0, li = 0, w = wa;
  if (lane < S) {
    w = wa + lane / O.n_layers;
    li = lane - (lane / O.n_layers) * O.n_layers;
    const Layer& L = O.L[li];
    lo = max(max(W.ga - w * nt, 0), L.tile_off);
    const int hi = min(min(W.gb - w * nt, nt), L.tile_off + L.n_tiles);
    len = max(hi - lo, 0);
    nr = (len + kSlotTiles - 1) / kSlotTiles;
    items = nr * W.nb[li];
  }
  // exclusive prefix sums over the segments (lane order = window-major, layer order)
  int rb = nr, ib = items;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, rb, o), b = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) { rb += a; ib += b; }
  }
  const int n_runs = __shfl_sync(0xffffffffu, rb, 31), n_items = __shfl_sync(0xffffffffu, ib, 31);
  rb -= nr;
  ib -= items;
  if (n_runs > kMaxRuns || W.gb - W.ga > kMaxTasks) __trap();   // host sizing (engine_eligible) violated
  for (int q = 0; q < nr; ++q) {
    Run& r = R.r[rb + q];
    r.li = (short)li;
    r.w = (short)w;
    r.t0 = (short)(lo + q * kSlotTiles);
    r.nt = (short)min(kSlotTiles, len - q * kSlotTiles);
    r.k0 = (short)(w * nt + lo + q * kSlotTiles - W.ga);
    fo_bo[rb + q] = (short)(ib + q * W.nb[li]);
  }
  // task kt = tile ga + kt -> its run
  for (int k0 = 0; k0 < W.gb - W.ga; k0 += 32) {   // uniform trip count: the shuffles need every lane
    const int kt = k0 + lane;
    const bool ok = kt < W.gb - W.ga;
    const int g = W.ga + (ok ? kt : 0), ww = g / nt, t = g - ww * nt;
    int l2 = 0;
    while (l2 + 1 < O.n_layers && t >= O.L[l2 + 1].tile_off) ++l2;
    const int sg = (ww - wa) * O.n_layers + l2;
    const int slo = __shfl_sync(0xffffffffu, lo, sg & 31), srb = __shfl_sync(0xffffffffu, rb, sg & 31);
    if (ok) task_r[kt] = (unsigned char)(srb + (t - slo) / kSlotTiles);
  }
  if (lane == 0) R.n = n_runs;
  __syncwarp();
  return n_items;
}

// Warp-parallel FIFO offsets of the extra planes [nb, fin) once the decision
// is known: runs in reverse order (the producer's issue order), exclusive
// prefix sums of items and tasks, and the extra task -> run table.
__device__ void extra_fifo_warp(const Op& O, const Work& W, const RunList& R, int base_items, short* fo_eo,
                                short* fo_xt, unsigned char* task_rx, int& n_items, int& n_tasks) {
  const int lane = threadIdx.x & 31;
  int carry_i = base_items, carry_t = 0;
  for (int c0 = 0; c0 < R.n; c0 += 32) {
    const int idx = c0 + lane;                  // position in the reversed order
    const int r = R.n - 1 - idx;
    int ex = 0, nt = 0;
    if (idx < R.n) {
      ex = W.fin[R.r[r].li] - W.nb[R.r[r].li];
      nt = ex > 0 ? R.r[r].nt : 0;
    }
    int si = ex, st = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, si, o), b = __shfl_up_sync(0xffffffffu, st, o);
      if (lane >= o) { si += a; st += b; }
    }
    if (idx < R.n) {
      fo_eo[r] = (short)(carry_i + si - ex);
      fo_xt[r] = (short)(carry_t + st - nt);
      for (int t = 0; t < nt; ++t) task_rx[carry_t + st - nt + t] = (unsigned char)r;
    }
    carry_i += __shfl_sync(0xffffffffu, si, 31);
    carry_t += __shfl_sync(0xffffffffu, st, 31);
  }
  n_items = carry_i - base_items;
  n_tasks = carry_t;
}

// ---------------------------------------------------------------------------
// TMA / mbarrier helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_n(unsigned long long* bar, unsigned n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const uint32_t a = smem_u32(bar);
  unsigned ok = 0;
  auto test = [&]() {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    return ok != 0;
  };
  SPIN_UNTIL_NS(test(), "ring slot", (long long)a, (long long)parity, 1000000000ull);
}
// Bitplanes are streamed once per step (GBs >> L2): marked evict-first so they
// do not push the small, re-read state (vectors, window slots, accumulators,
// G^T, KV rows) out of L2.
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
__device__ __forceinline__ uint4 ld_stream(const uint4* p, unsigned long long policy) {
  uint4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(policy));
  return r;
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                            unsigned long long policy) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}

// ---------------------------------------------------------------------------
// Vector emission: statistics + estimator feeds of one 32-row tile (a warp;
// lane = row). v = value (0 for padding rows).
// ---------------------------------------------------------------------------

// Statistics of one 32-row tile of vector instance inst: sum v, sum v^2.
__device__ __forceinline__ void emit_stats(const Prog& P, const ECtl& C, int inst, float v) {
  const int lane = threadIdx.x & 31;
  const double dv = (double)v;
  const double s = wsum(dv), q = wsum(dv * dv);
  if (lane == 0) {
    long long* vs = P.vstat + ((size_t)(C.n_steps_done & 1) * P.n_inst + inst) * 2 * kAccSpread;
    red_add64(vs, fx(s, kFxSum));
    red_add64(vs + kAccSpread, fx(q, kFxSq));
  }
}

// Feed fi (an estimator reading the vector) with tile `tile`: G_tile^T v
// partials and sum v^2 into its fixed-point accumulators (a warp, lane = row).

__device__ __forceinline__ void emit_feed(const Prog& P, const ECtl& C, int fi, int tile, float v,
                                          const uint4 (*pre)[8] = nullptr) {
  const int lane = threadIdx.x & 31;
  Feed F;
  {
    const int4* fp = reinterpret_cast<const int4*>(P.feeds + fi);
    int4* fd = reinterpret_cast<int4*>(&F);
#pragma unroll
    for (int q = 0; q < (int)(sizeof(Feed) / 16); ++q) fd[q] = __ldg(fp + q);
  }
  const int cur = C.n_steps_done & 1;
  const bool dyn = C.mode == MODE_DYNAMIC;
  long long* acc;
  if (F.kind == FEED_PREV) {
    if (!(dyn || C.prime)) return;
    acc = P.acc + (size_t)(2 + C.prev_w) * P.acc_stride + F.acc;
  } else {
    if (!dyn) return;
    if (F.kind == FEED_CURFB && C.has_prev) return;
    acc = P.acc + (size_t)cur * P.acc_stride + F.acc;
  }
  if (F.Gt) {
    // block of tile: [sub][chunk][lane][16 B]; f16 chunk = 4 rows x half2,
    // f32 chunk = 2 rows x float2; lane owns k pair (2 lane, 2 lane + 1) of sub.
    const int nsub = F.kpad / 64;
    const double sc = ldexp(1.0, F.fb);
    const unsigned long long pol = l2_evict_first_policy();   // G^T (~150 MB/step at 8B) streams like the planes
    for (int sub = 0; sub < nsub; ++sub) {
      float g0 = 0.f, g1 = 0.f;
      if (F.f16) {
        const uint4* blk = F.Gt + ((size_t)tile * nsub + sub) * 256 + lane;
        uint4 c[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = pre ? (*pre)[i] : ld_stream(blk + 32 * i, pol);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const __half2* hh = reinterpret_cast<const __half2*>(&c[i]);
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            const float xr = __shfl_sync(0xffffffffu, v, 4 * i + rr);
            const float2 gg = __half22float2(hh[rr]);
            g0 = fmaf(gg.x, xr, g0);
            g1 = fmaf(gg.y, xr, g1);
          }
        }
      } else {
        const uint4* blk = F.Gt + ((size_t)tile * nsub + sub) * 512 + lane;
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
          uint4 c[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) c[i] = ld_stream(blk + 32 * (8 * hb + i), pol);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float* ff = reinterpret_cast<const float*>(&c[i]);
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
              const float xr = __shfl_sync(0xffffffffu, v, 2 * (8 * hb + i) + rr);
              g0 = fmaf(ff[2 * rr], xr, g0);
              g1 = fmaf(ff[2 * rr + 1], xr, g1);
            }
          }
        }
      }
      const int k0 = sub * 64 + 2 * lane;
      if (k0 < F.k) red_add64(acc + (size_t)k0 * kAccSpread, fx((double)g0, sc));
      if (k0 + 1 < F.k) red_add64(acc + (size_t)(k0 + 1) * kAccSpread, fx((double)g1, sc));
    }
  }
  const double dv = (double)v;
  const double q = wsum(dv * dv);
  if (lane == 0) red_add64(acc + (size_t)F.k * kAccSpread, fx(q, kFxSq));
}

// Statistics + every feed of one tile (one warp).
__device__ __forceinline__ void emit_tile(const Prog& P, const ECtl& C, int inst, int tile, float v) {
  emit_stats(P, C, inst, v);
  for (int fi = P.feed_begin[inst]; fi < P.feed_begin[inst + 1]; ++fi) emit_feed(P, C, fi, tile, v);
}

// ---------------------------------------------------------------------------
// Grid barrier (monotonic 64-bit arrival counter)
// ---------------------------------------------------------------------------
// Grid barrier: monotonic arrival counter bar[0] (G arrivals per stage);
// waiters poll it relaxed and fence after (cheapest variant measured by
// tools/ubench_barrier.cu on B200: ~1.3 us for 148 CTAs).
__device__ __forceinline__ void bar_arrive(const Prog& P, unsigned long long epoch, int G) {
  CSYNC();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" :: "l"(P.bar) : "memory");
  }
}
__shared__ unsigned long long s_bar_seen;     // last barrier epoch seen released (zeroed at kernel start)
__device__ __forceinline__ void bar_wait(const Prog& P, unsigned long long epoch) {
  // lane 0 of warps 0..kPollers-1 poll, staggered by a fraction of the L2
  // round trip; the first to see the release publishes it in shared memory
  constexpr int kPollers = 4;
  volatile unsigned long long& s_seen = s_bar_seen;
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && warp < kPollers) {
    const unsigned long long target = epoch * (unsigned long long)gridDim.x;
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(P.bar) : "memory");
    if (v < target && s_seen < epoch) {
      if (warp) __nanosleep(120u * (unsigned)warp);
      auto poll = [&]() {
        if (s_seen >= epoch) return true;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(P.bar) : "memory");
        return v >= target;
      };
      SPIN_UNTIL_NS(poll(), "grid barrier", 0, (long long)epoch, 3000000000ull);
    }
    if (v >= target && s_seen < epoch) s_seen = epoch;
    __threadfence();
  }
  CSYNC();
}

__device__ __forceinline__ void read_ctl(const Prog& P, ECtl& C) {
  const int* src = reinterpret_cast<const int*>(P.ctl);
  int* dst = reinterpret_cast<int*>(&C);
  CSYNC();
  if (threadIdx.x < (int)(sizeof(ECtl) / 4)) dst[threadIdx.x] = __ldcg(src + threadIdx.x);
  CSYNC();
}

// ---------------------------------------------------------------------------
// Op stage
// ---------------------------------------------------------------------------
__device__ __forceinline__ void load4(uint4* dst, const uint4* a) {
  dst[0] = ld_nc(a);
  dst[1] = ld_nc(a + 32);
  dst[2] = ld_nc(a + 64);
  dst[3] = ld_nc(a + 96);
}


// L2 prefetch of the G^T blocks this CTA's reduce units will feed (one 4 KB
// block per (unit, feed) for f16, k <= 64), issued in the prologue so the
// feed loads at the end of the stage hit L2.
__device__ __forceinline__ void prefetch_own_feeds(const Prog& P, const ECtl& C, const Op& O, int cta, int G) {
  if (O.out_inst < 0 || (C.mode != MODE_DYNAMIC && !C.prime)) return;
  const int lane = threadIdx.x & 31;
  const int f0 = P.feed_begin[O.out_inst], nf = P.feed_begin[O.out_inst + 1] - f0;
  const int n_units = O.pair ? O.L[0].n_tiles : O.n_tiles;
  const int mine = n_units > cta ? (n_units - cta + G - 1) / G : 0;
  for (int q = lane; q < mine * nf; q += 32) {
    const int i = q / nf, u = cta + i * G;
    const Feed* F = P.feeds + f0 + (q - i * nf);
    if (!F->Gt) continue;
    const int li = layer_of(O, u);
    const int et = O.pair ? u : (O.L[li].out_off >> 5) + (u - O.L[li].tile_off);
    const int blk = (F->kpad / 64) * (F->f16 ? 4096 : 8192);
    l2_prefetch(reinterpret_cast<const char*>(F->Gt) + (size_t)et * blk, (unsigned)blk);
  }
}

// ---------------------------------------------------------------------------
// Tile reduction + epilogue (one warp, lane = row of the tile)
// ---------------------------------------------------------------------------
// S of op tile t: sum of the window slots in fixed window order, each slot
// awaited until it carries this op's epoch (no fence / counter needed: the
// 64-bit slot store is single-copy atomic).
__device__ __forceinline__ float tile_S(const Prog& P, const Op& O, int t, unsigned epoch) {
  const int lane = threadIdx.x & 31;
  const unsigned long long* base = P.slot + (size_t)t * 32 + lane;
  float acc = 0.f;
  for (int w0 = 0; w0 < O.n_win; w0 += 8) {
    const int nw = min(8, O.n_win - w0);
    unsigned long long v[8];
    bool ok;
    unsigned n_ = 0;
    unsigned long long t0 = 0;
    do {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < nw) v[j] = __ldcg(base + (size_t)(w0 + j) * P.slot_stride);
      ok = true;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < nw) ok &= (unsigned)(v[j] >> 32) == epoch;
      if ((++n_ & 1023u) == 0) {
        const unsigned long long t_ = gclock();
        if (t0 == 0) t0 = t_;
        else if (t_ - t0 > 4000000000ull) hang("window slots", t, 0);
      }
    } while (!__all_sync(0xffffffffu, ok));
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < nw) acc += __uint_as_float((unsigned)v[j]);
  }
  return acc;
}

// y of op tile t (layer li) at the final plane count; valid = row exists.
__device__ __forceinline__ float tile_y(const Prog& P, const Op& O, const Work& W, const Smem& sm, int t,
                                        unsigned epoch, int& li, int& r, bool& valid) {
  const int lane = threadIdx.x & 31;
  li = layer_of(O, t);
  const Layer& L = O.L[li];
  const int fin = W.fin[li];
  const float S = tile_S(P, O, t, epoch);
  r = (t - L.tile_off) * 32 + lane;
  valid = r < L.rows;
  if (!valid) return 0.f;
  const float lo = __ldg(L.lo + r), span = __ldg(L.span + r);
  return sm.scale * (lo * sm.sx + ldexpf(span, -fin) * (S + 0.5f * sm.sx));
}

// Reduce unit u (tile, or up|gate tile pair) of op O: window sum, affine
// epilogue, residual add / SiLU (runtime.py:364-370), output store. Returns the
// value the output instance is fed with (0 for padding rows) and its tile.
__device__ __forceinline__ float reduce_unit(const Prog& P, const Op& O, const Work& W, const Smem& sm, int u,
                                          unsigned epoch, int& etile) {
  const int lane = threadIdx.x & 31;
  // independent operands first (they do not wait for the window slots)
  {
    const int t = u, li = layer_of(O, t);
    const Layer& L = O.L[li];
    const int r = (t - L.tile_off) * 32 + lane;
    if (r < L.rows) { l1_prefetch(L.lo + r); l1_prefetch(L.span + r); }
    if (O.pair) {
      const int t2 = u + O.L[0].n_tiles, li2 = layer_of(O, t2);
      const Layer& L2 = O.L[li2];
      const int r2 = (t2 - L2.tile_off) * 32 + lane;
      if (r2 < L2.rows) { l1_prefetch(L2.lo + r2); l1_prefetch(L2.span + r2); }
    } else if (O.add && r < L.rows) {
      l1_prefetch(O.out + L.out_off + r);
    }
  }
  unsigned long long* stp = (threadIdx.x == 0 && u == blockIdx.x) ? sm.stamp : nullptr;
  if (stp) stp[2] = gclock();
  CSTAMP(stp, 11);
  float v = 0.f;
  if (O.pair) {
    const int half = O.L[0].n_tiles;
    int li, r, li2, r2;
    bool ok, ok2;
    const float up = tile_y(P, O, W, sm, u, epoch, li, r, ok);
    const float gt = tile_y(P, O, W, sm, u + half, epoch, li2, r2, ok2);
    v = ok ? up * (gt / (1.0f + expf(-gt))) : 0.f;                 // runtime.py:368
    if (ok) O.out[r] = v;
    etile = u;
  } else {
    int li, r;
    bool ok;
    const float y = tile_y(P, O, W, sm, u, epoch, li, r, ok);
    const int o = O.L[li].out_off + r;
    if (ok) {
      v = O.add ? O.out[o] + y : y;                                 // runtime.py:364, 370
      O.out[o] = v;
    }
    etile = (O.L[li].out_off >> 5) + (u - O.L[li].tile_off);
  }
  if (stp) stp[3] = gclock();
  CSTAMP(stp, 12);
  return v;
}

// ---------------------------------------------------------------------------
// The op stage (consumer warps 0..NW-1)
// ---------------------------------------------------------------------------
// Reduction of the op's units: unit u belongs to CTA u mod G (spread over the
// grid so every CTA has at most a few), its i-th unit to warp i mod NW. Phase
// A: window sums + epilogue per unit (values parked in shared memory); phase
// B: the estimator feeds of the output instance, one (unit, feed) task per
// warp in parallel (independent fixed-point sums). Warp NW - 1 first prepares
// the next op's descriptor and work.
__device__ __forceinline__ void reduce_duty(const Prog& P, const ECtl& C, const Op& O, const Work& W, Smem& sm,
                                          int cta, int G, unsigned epoch, Op* On, Work* Wn, const Op* On_global,
                                          int op_no) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_units = O.pair ? O.L[0].n_tiles : O.n_tiles;
  const int mine = n_units > cta ? (n_units - cta + G - 1) / G : 0;     // units of this CTA
  if (warp == NW - 1 && On && !Wn->valid) {
    // (descriptor copied into *On during the prologue)
    build_work_warp(*On, C, cta, G, *Wn);
    __syncwarp();
    // the next op's base runs, FIFO offsets and task table (this op's are dead
    // after its items): off the next stage's pre-barrier path
    const int nbi = build_runs_warp(*On, *Wn, sm.runs, sm.fo_bo, sm.task_rb);
    if (lane == 0) {
      Wn->valid = 1;
      sm.last = nbi;
      sm.runs_op = op_no + 1;
    }
  }
  const int f0 = O.out_inst >= 0 ? P.feed_begin[O.out_inst] : 0;
  const int nf = O.out_inst >= 0 ? P.feed_begin[O.out_inst + 1] - f0 : 0;
  for (int i = warp; i < mine; i += NW) {
    int et;
    const float v = reduce_unit(P, O, W, sm, cta + i * G, epoch, et);
    if (O.out_inst >= 0) {
      emit_stats(P, C, O.out_inst, v);
      sm.sbuf[i][lane] = v;              // parked base sums are dead after the extra pass
      if (lane == 0) sm.vtile[i] = et;
    }
  }
  if (nf == 0) return;
  CSYNC();
  for (int q = warp; q < mine * nf; q += NW) {
    const int i = q / nf;
    emit_feed(P, C, f0 + (q - i * nf), sm.vtile[i], sm.sbuf[i][lane]);
  }
  if (threadIdx.x == 0) CSTAMP(sm.stamp, 13);
}

// FIFO layout of an op (relative to its first FIFO index): base items run by
// run, planes [0, nb); then extra items for runs in reverse order, planes
// [nb, fin). Returns the total and fills per-run offsets (lane-parallel).
// Returns the number of ring items the op consumed (FIFO advance).
__device__ __forceinline__ int op_stage(const Prog& P, const ECtl& C, const Op& O, Work& W, Op* On, Work* Wn,
                                     const Op* On_global, Smem& sm, int cta, int G,
                                     unsigned long long wait_target, bool do_wait, unsigned long long* stamp,
                                     int op_no, int j_op) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned epoch = (unsigned)(wait_target + 1);     // this stage's epoch: tags the window slots
  const int cur = C.n_steps_done & 1;
  // ---- base work and run list (decision independent), before the barrier
  // every thread reads W.valid before anyone can change it: the decision to
  // join the CSYNC below must be uniform (a named-barrier count mismatch
  // would silently misalign all later consumer barriers)
  const bool built = W.valid != 0;
  CSYNC();
  if (!built) {
    if (warp == 0) build_work_warp(O, C, cta, G, W);
    CSYNC();
  }
  if (warp == 0 && sm.runs_op != op_no) {   // not prepared during the previous op's reduce phase
    const int nbi = build_runs_warp(O, W, sm.runs, sm.fo_bo, sm.task_rb);
    if (lane == 0) sm.last = nbi;
  }
  if (tid == 0) {
    sm.stamp = stamp;
    sm.cons_op = op_no;
    sm.cons_j = j_op;
  }
  if (do_wait) bar_wait(P, wait_target);
  if (stamp && tid == 0) stamp[0] = gclock();
  if (tid == 0) CSTAMP(stamp, 0);

  // ---- prologue. Critical path: the first window's input -> LUT -> base
  // items. The selector inputs (accumulators, statistics) are loaded in the
  // same round trip and finished after the LUT build (runtime.py:184-193).
  const int w_first = sm.runs.n > 0 ? sm.runs.r[0].w : -1;
  const LutSrc xsrc = lut_load(O.in, O.cols, max(w_first, 0));
  // decision warps: accumulator loads in flight (k <= 128: 4 per lane)
  // roles: warps 0..7 build the LUT (lut_store: threads < 256), warps 8.. take
  // the decisions (one per layer) and the input statistics
  constexpr int kDecW = 8, kStatW = kDecW + kMaxOpLayers;
  static_assert(kStatW + 2 < NW - 1, "prologue roles need more consumer warps");
  const int li_d = warp - kDecW;
  const bool dec_warp = li_d >= 0 && li_d < O.n_layers;
  const Layer& Ld = O.L[dec_warp ? li_d : 0];
  const bool estimating = dec_warp && C.mode == MODE_DYNAMIC && Ld.sentinel == 0 && Ld.est != EST_NONE;
  long long ga[4] = {0, 0, 0, 0}, gsq = 0;
  if (estimating) {
    const int slot = (Ld.src == SRC_PREV_STEP && C.has_prev) ? 2 + C.prev_r : cur;
    const long long* acc = P.acc + (size_t)slot * P.acc_stride + Ld.acc;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (lane + 32 * q < Ld.k) ga[q] = __ldcg(acc + (size_t)(lane + 32 * q) * kAccSpread);
    gsq = __ldcg(acc + (size_t)Ld.k * kAccSpread);
  }
  long long vs1 = 0, vs2 = 0;
  if (warp == kStatW + 1) prefetch_own_feeds(P, C, O, cta, G);
  if (warp == kStatW + 2 && On && !Wn->valid) {
    // the next op's descriptor -> shared memory now (its work and runs are
    // built during this op's reduce phase, no global round trip there)
    const int nw4 = (int)(sizeof(Op) / 16);
    const int4* src = reinterpret_cast<const int4*>(On_global);
    int4* dst = reinterpret_cast<int4*>(On);
    for (int q = lane; q < nw4; q += 32) dst[q] = __ldg(src + q);
  }
  if (warp == kStatW && lane == 0) {
    const long long* vs = P.vstat + ((size_t)cur * P.n_inst + O.in_inst) * 2 * kAccSpread;
    vs1 = __ldcg(vs);
    vs2 = __ldcg(vs + kAccSpread);
  }
  if (tid == 0) CSTAMP(stamp, 1);
  float* lut = reinterpret_cast<float*>(reinterpret_cast<char*>(&sm) + (kLut - smem_u32(&sm)));
  int lut_w = -1;
  if (w_first >= 0) {                 // LUT of the first window
    lut_store(lut, xsrc);
    lut_w = w_first;
  }
  if (tid == 0) CSTAMP(stamp, 2);
  if (dec_warp) {
    const int li = li_d;
    int bit = W.nb[li];
    double est = CUDART_NAN;
    if (estimating) {
      double q = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double g = (double)ga[i] * Ld.fbscale;
        q += g * g;
      }
      q = wsum(q);
      const double sq = (double)gsq * (1.0 / kFxSq);
      const double sc = O.rms ? rsqrt_d(sq / (double)O.cols + (double)P.eps) : 1.0;
      if (Ld.est == EST_PROJECTION) est = q > 0.0 ? sc * q * rsqrt_d(q) : 0.0;
      else est = Ld.slope * (sq > 0.0 ? sc * sq * rsqrt_d(sq) : 0.0) + Ld.intercept;
      if (!C.force) bit = est > Ld.T ? Ld.h : Ld.l;                      // strict > (runtime.py:192)
    }
    if (lane == 0) {
      CSTAMP(stamp, 4 + li);
      W.fin[li] = bit;
      sm.dec_fin[op_no & 1][li] = bit;
      if (C.mode == MODE_DYNAMIC && cta == 0 && Ld.trace >= 0 && P.n_trace > 0 && C.trace_step < P.max_steps) {
        const size_t o = (size_t)C.trace_step * P.n_trace + Ld.trace;
        P.tr_bits[o] = (signed char)bit;
        P.tr_est[o] = estimating ? (float)est : CUDART_NAN_F;
      }
    }
  } else if (warp == kStatW && lane == 0) {
    sm.sx = (float)((double)vs1 * (1.0 / kFxSum));
    sm.scale = O.rms ? (float)rsqrt_d((double)vs2 * (1.0 / kFxSq) / (double)O.cols + (double)P.eps) : 1.f;
    CSTAMP(stamp, 7);
  }
  CSYNC();                             // decisions and LUT visible
  const RunList& R = sm.runs;
  if (warp == NW - 1) {                 // last warp: fewest items (tasks go round-robin from warp 0)
    if (lane == 0) {
      __threadfence_block();
      sm.dec_op = op_no + 1;          // the producer may now stream the extra planes
    }
    // FIFO offsets of the extra planes (base offsets were set before the barrier)
    int ni, nt;
    extra_fifo_warp(O, W, R, sm.last, sm.fo_eo, sm.fo_xt, sm.task_rx, ni, nt);
    if (lane == 0) {
      sm.n_ext_items = ni;
      sm.t_ext = nt;
    }
  }
  const int n_base = sm.last;
  if (stamp && tid == 0) stamp[1] = gclock();
  if (tid == 0) CSTAMP(stamp, 3);
  if (tid == 0) PROGRESS(1, 1);
  const int n_tasks_base = W.gb - W.ga;
#ifdef DPQ_PROFILE_WARPS
  unsigned long long w_first_t = 0, w_last_t = 0, w_seq = 0, w_mb = 0, w_task0 = 0;   // per-warp profiling (stamp != nullptr)
  int w_planes = 0;
#define WPROF(x) do { if (stamp) { x; } } while (0)
#else
#define WPROF(x) do { } while (0)
#endif
  // ---- stream: tasks (run, tile) in FIFO order, LUT rebuilt per window segment
  const unsigned char* dyn0 = reinterpret_cast<const unsigned char*>(&sm);
  for (int kind = 0; kind < 2; ++kind) {
    const int n_tasks = kind ? sm.t_ext : n_tasks_base;
    int k = 0;                          // task index at the segment start
    int rr = kind ? R.n - 1 : 0;        // run index at the segment start
    while (k < n_tasks) {
      // segment: consecutive runs (task order) of one window
      while (kind && W.fin[R.r[rr].li] == W.nb[R.r[rr].li]) --rr;
      const int w = R.r[rr].w;
      int k_end = k, re = rr;
      while (kind ? re >= 0 : re < R.n) {
        const Run& q = R.r[re];
        if (q.w != w) break;
        if (!kind || W.fin[q.li] > W.nb[q.li]) k_end += q.nt;
        re += kind ? -1 : 1;
      }
      if (w != lut_w) {
        const LutSrc xs2 = lut_load(O.in, O.cols, w);
        CSYNC();                          // previous LUT users done
        lut_store(lut, xs2);
        CSYNC();
        lut_w = w;
      }
      const uint32_t lanereg = kLut | ((uint32_t)lane * 4u);
      for (int kt = k + warp; kt < k_end; kt += NW) {
        WPROF(if (!w_task0) w_task0 = clock64());
        // task kt -> run and tile (tables built with the FIFO offsets)
        const int r = kind ? sm.task_rx[kt] : sm.task_rb[kt];
        const Run& q = R.r[r];
        const int i = kt - (kind ? sm.fo_xt[r] : q.k0);
        const int nb = W.nb[q.li], fin = W.fin[q.li];
        const int p0 = kind ? nb : 0, p1 = kind ? fin : nb;
        const int jr = sm.cons_j + (kind ? sm.fo_eo[r] : sm.fo_bo[r]);   // FIFO base from shared memory (no spill reload)
        const int pk = q.k0 + i;                                   // task (group) index in [ga, gb)
        float S = 0.f;
        if (kind) S = pk < kMaxTiles ? sm.sbuf[pk][lane]
                                     : __ldcg(P.park + ((size_t)cta * (kMaxTasks - kMaxTiles) + pk - kMaxTiles) * 32 + lane);
        for (int p = p0; p < p1; ++p) {
          const int j = jr + (p - p0);
          const int slot = j & (kMaxSlots - 1);
          WSTATE(j * 16 + 1);
#ifdef DPQ_PROFILE_WARPS
          const unsigned long long tw0 = stamp ? clock64() : 0;
#endif
          if (lane == 0) SPIN_UNTIL_NS(sm.seq[slot] == j, "ring sequence", j, sm.seq[slot], 1000000000ull);
          __syncwarp();
          WSTATE(j * 16 + 2);
#ifdef DPQ_PROFILE_WARPS
          const unsigned long long tw1 = stamp ? clock64() : 0;
#endif
          mbar_wait(&sm.full[slot], (unsigned)((j / kMaxSlots) & 1));
          WSTATE(j * 16 + 3);
#ifdef DPQ_PROFILE_WARPS
          if (stamp) {
            const unsigned long long tn = clock64();
            w_seq += tw1 - tw0;
            w_mb += tn - tw1;
            if (!w_first_t) w_first_t = tn;
            w_last_t = tn;
            ++w_planes;
          }
#endif
          const uint4* d = reinterpret_cast<const uint4*>(dyn0 + sm.slot_off[slot] + i * kTileBytes) + lane;
          const uint4 d0 = d[0], d1 = d[32], d2 = d[64], d3 = d[96];
          S = 2.f * S + plane_sum(d0, d1, d2, d3, lanereg);       // Horner over planes
          __syncwarp();                                            // every lane has used its slot data
          if (lane == 0) mbar_arrive_n(&sm.empty[slot], i == q.nt - 1 ? (unsigned)(kSlotTiles + 1 - q.nt) : 1u);
          WSTATE(j * 16 + 4);
        }
        const int t = q.t0 + i;
        if (!kind && fin > nb) {
          if (pk < kMaxTiles) sm.sbuf[pk][lane] = S;                // park the base part
          else __stcg(P.park + ((size_t)cta * (kMaxTasks - kMaxTiles) + pk - kMaxTiles) * 32 + lane, S);
        } else {
          __stcg(P.slot + (size_t)q.w * P.slot_stride + (size_t)t * 32 + lane,
                 (unsigned long long)epoch << 32 | __float_as_uint(S));
        }
      }
      k = k_end;
      rr = re;
    }
#ifdef DPQ_PROFILE_WARPS
    if (stamp && lane == 0) {
      unsigned long long* ws = stamp + 8 + warp * 5;
      ws[0] = w_task0; ws[1] = w_first_t; ws[2] = w_last_t; ws[3] = clock64(); ws[4] = (unsigned long long)w_planes | (min(w_seq, 0xffffffull) << 16) | (min(w_mb, 0xffffffull) << 40);
    }
#endif
    // kind 0: parked base sums visible before the extra pass; kind 1: every warp
    // done with the runs before the reduce phase rebuilds them for the next op
    if (!kind || n_tasks > 0) CSYNC();
  }
  if (tid == 0) PROGRESS(1, 2);
  if (stamp && tid == 0) stamp[5] = gclock();
  if (tid == 0) CSTAMP(stamp, 10);
  reduce_duty(P, C, O, W, sm, cta, G, epoch, On, Wn, On_global, op_no);
  if (tid == 0) PROGRESS(1, 3);
  if (stamp && tid == 0) stamp[6] = gclock();
  if (tid == 0) CSTAMP(stamp, 15);
  CSYNC();
  if (tid == 0) { W.valid = 0; CSTAMP(stamp, 16); }
  return n_base + sm.n_ext_items;
}

// ---------------------------------------------------------------------------
// The TMA producer warp: streams every op's planes into the ring, running
// ahead of the consumers across stage barriers (bounded by ring space, and by
// each op's decision for its extra planes).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void producer(const Prog& P, Smem& sm, int cta, int G, int n_steps) {
  const int lane = threadIdx.x & 31;
  int j = 0, op_no = 0;
  const unsigned char* dyn0 = reinterpret_cast<const unsigned char*>(&sm);
  const unsigned long long l2pol = l2_evict_first_policy();
  auto issue = [&](const Op& O, const Run& r, int p) {
    const int slot = j & (kMaxSlots - 1);
    if (j >= kMaxSlots) {
      const uint32_t a = smem_u32(&sm.empty[slot]);
      const unsigned par = (unsigned)(((j / kMaxSlots) - 1) & 1);
      unsigned ok = 0;
      auto test = [&]() {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(a), "r"(par) : "memory");
        return ok != 0;
      };
      SPIN_UNTIL_NS(test(), "producer slot", ((long long)j << 32) | (unsigned)op_no,
                    ((long long)sm.cons_op << 32) | (unsigned)sm.cons_j, 12000000000ull);
      // the consumers' generic reads of the slot precede this async-proxy write
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    sm.seq[slot] = j;
    PROGRESS(2, j);
    PROGRESS(3, op_no);
    const Layer& L = O.L[r.li];
    const uint4* src = L.planes + p * L.pstride + ((long long)r.w * L.n_tiles + (r.t0 - L.tile_off)) * (kTileBytes / 16);
    mbar_expect_tx(&sm.full[slot], (unsigned)r.nt * kTileBytes);
    tma_load_1d(const_cast<unsigned char*>(dyn0) + sm.slot_off[slot], src, (unsigned)r.nt * kTileBytes, &sm.full[slot],
                l2pol);
    ++j;
  };
  for (int step = 0; step < n_steps; ++step) {
    if (lane == 0) SPIN_UNTIL_NS(sm.step_ready >= step + 1, "producer step", step, 0, 12000000000ull);
    __syncwarp();
    __threadfence_block();
    const ECtl& C = sm.ctl;
    for (int si = 0; si < P.n_stages; ++si) {
      const int2 st = P.stages[si];
      if (st.x != ST_OP) continue;
      const int nw4 = (int)(sizeof(Op) / 16);
      const int4* src = reinterpret_cast<const int4*>(P.ops + st.y);
      int4* dst = reinterpret_cast<int4*>(&sm.pop);
      for (int q = lane; q < nw4; q += 32) dst[q] = __ldg(src + q);
      __syncwarp();
      build_work_warp(sm.pop, C, cta, G, sm.pw);
      __syncwarp();
      // (no L2 bulk prefetch of the next op's planes: measured slower -- it
      // competes with the current stage's loads; the ring alone runs ahead)
      build_runs_warp(sm.pop, sm.pw, sm.pruns, sm.pfo, sm.ptask);   // same runs as the consumers'
      if (lane == 0) {
        unsigned long long* pd = P.dbg ? P.dbg + ((size_t)si * G + cta) * kDbgRec + 8 + 5 * NW : nullptr;
        const int j0 = j;
        if (pd) pd[0] = gclock();
        const Op& O = sm.pop;
        const RunList& R = sm.pruns;
        for (int r = 0; r < R.n; ++r)
          for (int p = 0; p < sm.pw.nb[R.r[r].li]; ++p) {
            issue(O, R.r[r], p);
            if (pd && j == j0 + 1) pd[1] = gclock();
          }
        if (pd) pd[2] = gclock();
        bool may_extra = false;
        if (C.mode == MODE_DYNAMIC && !C.force)
          for (int li = 0; li < O.n_layers; ++li) may_extra |= O.L[li].sentinel == 0 && O.L[li].l < O.L[li].h;
        if (may_extra && R.n > 0) {
          SPIN_UNTIL_NS(sm.dec_op >= op_no + 1, "producer decision", op_no, 0, 12000000000ull);
          __threadfence_block();
          if (pd) pd[3] = gclock();
          for (int r = R.n - 1; r >= 0; --r) {
            const int li = R.r[r].li;
            const int fin = sm.dec_fin[op_no & 1][li];
            for (int p = sm.pw.nb[li]; p < fin; ++p) issue(O, R.r[r], p);
          }
        }
        if (pd) { pd[4] = gclock(); pd[5] = (unsigned long long)(j - j0); }
      }
      __syncwarp();
      ++op_no;
    }
  }
}

// ---------------------------------------------------------------------------
// Attention stage (runtime.py:351-362): RoPE, KV append, causal softmax.
// ---------------------------------------------------------------------------
// Unit = (query head h, chunk of <= kAttnChunkE positions). Warp w takes the
// chunk's positions s0 + w, s0 + w + NW, ... with a per-warp online softmax
// (lane = 4 consecutive dims, float4 loads; RoPE half-split recomputed per
// warp from the q / k outputs, runtime.py:351-352); the NW partial (m, l, o)
// are merged in shared memory in fixed warp order. Chunk partials of a head
// are merged by the last unit of the head. The unit holding position t of the
// first query head of each KV group appends k_t / v_t (runtime.py:355-356).
constexpr int kAttnPerWarp = 16;                 // positions per warp and chunk
constexpr int kAttnStaged = 3;                   // of which staged in shared memory (LUT region)
constexpr int kAttnChunkE = NW * kAttnPerWarp;   // positions per unit

// RoPE of 4 consecutive dims [i0, i0 + 4) of a head vector v (i0 % 4 == 0,
// hd % 8 == 0), with the position's cos / sin of those dims preloaded.
__device__ __forceinline__ float4 rope4(const float* v, int i0, int hd, float4 c, float4 s) {
  const int half = hd / 2;
  const bool lo = i0 < half;
  const float4 a = __ldcg(reinterpret_cast<const float4*>(v + i0));
  const float4 b = __ldcg(reinterpret_cast<const float4*>(v + (lo ? i0 + half : i0 - half)));
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

// Statistics + feeds of head h's output tiles (values in vals[hd]): one
// (tile, feed) task per warp.
__device__ __forceinline__ void attn_emit_head(const Prog& P, const ECtl& C, int inst, int h, const float* vals) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nt = (P.hd + 31) / 32;
  const int f0 = P.feed_begin[inst], nf = P.feed_begin[inst + 1] - f0;
  for (int q = warp; q < nt * (nf + 1); q += NW) {
    const int tt = q / (nf + 1), f = q - tt * (nf + 1);
    const int i = tt * 32 + lane;
    const float v = i < P.hd ? vals[i] : 0.f;
    const int tile = (h * P.hd) / 32 + tt;
    if (f == nf) emit_stats(P, C, inst, v);
    else emit_feed(P, C, f0 + f, tile, v);
  }
}

__device__ __forceinline__ void attn_stage(const Prog& P, const ECtl& C, int b, float* sh, int cta, int G, int* s_last,
                                       unsigned long long wait_target, bool do_wait, unsigned long long* stamp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = C.pos, n = t + 1;
  const int hd = P.hd, qh = P.H / P.KV, nv = hd / 4;
  const int nch = (n + kAttnChunkE - 1) / kAttnChunkE;
  const int units = P.H * nch;
  const float scale = 1.0f / sqrtf((float)hd);
  const float* cs = P.cosv + (size_t)t * (hd / 2);
  const float* sn = P.sinv + (size_t)t * (hd / 2);
  float* kc = P.kc[b];
  float* vc = P.vc[b];
  const int inst = 4 * b + 1;
  // shared memory (LUT region): K / V staging [NW][kAttnStaged][2][hd], the
  // per-warp partials [NW][hd + 4] and the merged head output [hd]
  float* kvs = sh;
  const int ps = hd + 4;                   // part row stride (16-byte aligned)
  float* part = sh + NW * kAttnStaged * 2 * hd;
  float* outv = part + NW * ps;
  const bool act = lane < nv;
  const int i0 = 4 * lane;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const unsigned long long kvpol = l2_evict_last_policy();   // the KV cache is re-read every step: keep it in L2
  // Rows of unit positions s0 + warp + NW j: j < kAttnStaged are copied
  // asynchronously into shared memory (for the CTA's first unit before the
  // barrier: cached positions do not depend on this step; a lane copies and
  // later reads only its own 16 bytes), the rest stream through a 4-deep
  // register pipeline.
#define ATTN_STAGE_ROWS(u_)                                                              \
  do {                                                                                   \
    const int h_ = (u_) / nch, g_ = h_ / qh;                                             \
    const int s0_ = ((u_) - h_ * nch) * kAttnChunkE, lim_ = min(t, s0_ + kAttnChunkE);   \
    _Pragma("unroll") for (int j = 0; j < kAttnStaged; ++j) {                            \
      const int s_ = s0_ + warp + NW * j;                                                \
      if (act && s_ < lim_) {                                                            \
        const size_t off_ = (size_t)s_ * P.dkv + g_ * hd + i0;                           \
        float* d_ = kvs + ((warp * kAttnStaged + j) * 2) * hd + i0;                      \
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" :: "r"(smem_u32(d_)), "l"(kc + off_), "l"(kvpol) : "memory"); \
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" :: "r"(smem_u32(d_ + hd)), "l"(vc + off_), "l"(kvpol) : "memory"); \
      }                                                                                  \
    }                                                                                    \
  } while (0)
#define ATTN_ROW(s_, lim_, g_, K_, V_)                                             \
  do {                                                                             \
    if (act && (s_) < (lim_)) {                                                    \
      const size_t off_ = (size_t)(s_) * P.dkv + (g_) * hd + i0;                   \
      K_ = ld_keep(kc + off_, kvpol);                                             \
      V_ = ld_keep(vc + off_, kvpol);                                             \
    }                                                                              \
  } while (0)
  if (cta < units) ATTN_STAGE_ROWS(cta);
  const int j0 = i0 < hd / 2 ? i0 : i0 - hd / 2;
  const float4 c4 = act ? __ldg(reinterpret_cast<const float4*>(cs + j0)) : z4;
  const float4 s4 = act ? __ldg(reinterpret_cast<const float4*>(sn + j0)) : z4;
  if (do_wait) bar_wait(P, wait_target);
  if (stamp && tid == 0) stamp[0] = gclock();
  if (tid == 0) CSTAMP(stamp, 0);
  for (int u = cta; u < units; u += G) {
    const int h = u / nch, ch = u - h * nch;
    const int g = h / qh;
    unsigned long long* stp = (tid == 0 && u == cta) ? stamp : nullptr;
    const int s0 = ch * kAttnChunkE, s1 = min(n, s0 + kAttnChunkE);
    const int lim = min(t, s1);            // cached rows of the chunk: [s0, lim)
    if (u != cta) {
      CSYNC();                             // previous unit's readers of the staging done
      ATTN_STAGE_ROWS(u);
    }
    // per-warp online softmax (lane = dims 4 lane .. 4 lane + 3)
    float m = -CUDART_INF_F, l = 0.f;
    float4 o = z4;
    const float4 q4 = act ? rope4(P.qkv + h * hd, i0, hd, c4, s4) : o;
    float4 kt = o, vt = o;
    const bool own_t = act && s1 == n && (t - s0) % NW == warp;   // this warp holds the new position t
    if (own_t) {
      kt = rope4(P.qkv + P.d + g * hd, i0, hd, c4, s4);      // RoPE'd k of this step
      vt = __ldcg(reinterpret_cast<const float4*>(P.qkv + P.d + P.dkv + g * hd + i0));
    }
    // register pipeline rows (j = kAttnStaged ..., 2 deep), in flight with q / k_t / v_t
    const int sr = s0 + warp + NW * kAttnStaged;
    float4 k0 = z4, v0 = z4, k1 = z4, v1 = z4;
    ATTN_ROW(sr, lim, g, k0, v0);
    ATTN_ROW(sr + NW, lim, g, k1, v1);
    if (own_t && h % qh == 0) {          // runtime.py:355-356 (KV append)
      *reinterpret_cast<float4*>(kc + (size_t)t * P.dkv + g * hd + i0) = kt;
      *reinterpret_cast<float4*>(vc + (size_t)t * P.dkv + g * hd + i0) = vt;
    }
#define ATTN_UPDATE(s_, K_, V_)                                                    \
    {                                                                              \
      const float4 k4 = (s_) == t ? kt : K_, v4 = (s_) == t ? vt : V_;             \
      const float a = wsum(dot4(q4, k4)) * scale;            /* runtime.py:358 */  \
      const float mn = fmaxf(m, a);                                                \
      const float corr = expf(m - mn), p = expf(a - mn);     /* runtime.py:359-361 */ \
      l = l * corr + p;                                                            \
      o.x = o.x * corr + p * v4.x; o.y = o.y * corr + p * v4.y;                    \
      o.z = o.z * corr + p * v4.z; o.w = o.w * corr + p * v4.w;                    \
      m = mn;                                                                      \
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
    for (int j = 0; j < kAttnStaged; ++j) {
      const int s = s0 + warp + NW * j;
      if (s < s1) {
        const float* r_ = kvs + ((warp * kAttnStaged + j) * 2) * hd + i0;
        const float4 ks = act ? *reinterpret_cast<const float4*>(r_) : z4;
        const float4 vs = act ? *reinterpret_cast<const float4*>(r_ + hd) : z4;
        ATTN_UPDATE(s, ks, vs)
      }
    }
#define ATTN_STEP(s_, K_, V_)                                                      \
    if ((s_) < s1) ATTN_UPDATE(s_, K_, V_)                                         \
    ATTN_ROW((s_) + 2 * NW, lim, g, K_, V_);   /* refill this register slot */
    for (int s = sr; s < s1; s += 2 * NW) {
      ATTN_STEP(s, k0, v0)
      ATTN_STEP(s + NW, k1, v1)
    }
    CSTAMP(stp, 2);
    CSYNC();                                 // previous unit's readers of part / outv done
    if (act) *reinterpret_cast<float4*>(part + warp * ps + i0) = o;
    // warp weights (fixed order): lane w of every warp computes the global max M
    // and e_w = exp(m_w - M); L = sum_w e_w l_w
    if (lane == 0) { part[warp * ps + hd] = m; part[warp * ps + hd + 1] = l; }
    CSYNC();
    CSTAMP(stp, 7);
    {
      const float mw = lane < NW ? part[lane * ps + hd] : -CUDART_INF_F;
      const float lw = lane < NW ? part[lane * ps + hd + 1] : 0.f;
      float M = mw;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
      const float e = mw == -CUDART_INF_F ? 0.f : expf(mw - M);      // warps without positions: 0
      // fixed-order sum over lanes 0..NW-1 (the shuffle tree is the same in every warp)
      const float L = wsum(e * lw);
      const int di = tid < hd ? tid : 0;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) acc += __shfl_sync(0xffffffffu, e, w) * part[w * ps + di];
      CSTAMP(stp, 8);
      if (tid < hd) {
        if (nch == 1) {
          const float r = acc / L;            // runtime.py:362
          P.attn[h * hd + tid] = r;
          outv[tid] = r;
        } else {
          float* pp = P.attn_part + ((size_t)h * P.attn_max_chunks + ch) * (hd + 2);
          pp[tid] = acc;
          if (tid == 0) { pp[hd] = M; pp[hd + 1] = L; }
        }
      }
    }
    if (nch == 1) {
      CSYNC();
      CSTAMP(stp, 4);
      if (P.attn_emit) attn_emit_head(P, C, inst, h, outv);
      CSTAMP(stp, 5);
      continue;
    }
    __threadfence();
    CSYNC();
    if (tid == 0) *s_last = atomicAdd(P.attn_cnt + h, 1u) == (unsigned)nch - 1;
    CSYNC();
    if (!*s_last) continue;
    __threadfence();
    const float* base = P.attn_part + (size_t)h * P.attn_max_chunks * (hd + 2);
    if (tid < hd) {
      float M = -CUDART_INF_F;
#pragma unroll 1
      for (int c = 0; c < nch; ++c) M = fmaxf(M, __ldcg(base + c * (hd + 2) + hd));
      float Ls = 0.f, acc = 0.f;
#pragma unroll 1
      for (int c = 0; c < nch; ++c) {
        const float e = expf(__ldcg(base + c * (hd + 2) + hd) - M);
        Ls += __ldcg(base + c * (hd + 2) + hd + 1) * e;
        acc += __ldcg(base + c * (hd + 2) + tid) * e;
      }
      const float r = acc / Ls;
      P.attn[h * hd + tid] = r;
      outv[tid] = r;
    }
    if (tid == 0) P.attn_cnt[h] = 0u;
    CSYNC();
    CSTAMP(stp, 4);
    if (P.attn_emit) attn_emit_head(P, C, inst, h, outv);
    CSTAMP(stp, 5);
  }
  if (tid == 0) CSTAMP(stamp, 6);
}

// EMIT: statistics + feeds of a whole vector (attention output when heads
// are not 32-aligned).
__device__ __forceinline__ void emit_stage(const Prog& P, const ECtl& C, const float* v, int n, int inst, int cta, int G) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_t = (n + 31) / 32;
  for (int tt = cta * NW + warp; tt < n_t; tt += G * NW) {
    const int i = tt * 32 + lane;
    emit_tile(P, C, inst, tt, i < n ? __ldcg(v + i) : 0.f);
  }
}

// ---------------------------------------------------------------------------
// Head stage: final RMSNorm + lm_head logits (runtime.py:372), greedy argmax
// (runtime.py:405-408) and the end-of-step control update (runtime.py:373-380).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void head_stage(const Prog& P, const ECtl& C, Smem& sm, int cta, int G) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cur = C.n_steps_done & 1;
  const int fin_inst = 4 * P.n_blocks;
  const double s2 =
      (double)__ldcg(P.vstat + (((size_t)cur * P.n_inst + fin_inst) * 2 + 1) * kAccSpread) * (1.0 / kFxSq);
  const float inv = (float)(1.0 / sqrt(s2 / (double)P.d + (double)P.eps));
  for (int v = cta * NW + warp; v < P.vocab; v += G * NW) {
    const float* row = P.lm + (size_t)v * P.d;
    float a = 0.f;
    int i = lane * 4;
    if ((P.d & 3) == 0) {
      for (; i + 7 * 128 < P.d; i += 8 * 128) {
        float4 w4[8], x4[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          w4[u] = __ldg(reinterpret_cast<const float4*>(row + i + u * 128));
          x4[u] = __ldcg(reinterpret_cast<const float4*>(P.x + i + u * 128));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) a += w4[u].x * x4[u].x + w4[u].y * x4[u].y + w4[u].z * x4[u].z + w4[u].w * x4[u].w;
      }
      for (; i < P.d; i += 128) {
        const float4 w4 = __ldg(reinterpret_cast<const float4*>(row + i));
        const float4 x4 = __ldcg(reinterpret_cast<const float4*>(P.x + i));
        a += w4.x * x4.x + w4.y * x4.y + w4.z * x4.z + w4.w * x4.w;
      }
    } else {
      for (int k = lane; k < P.d; k += 32) a += row[k] * __ldcg(P.x + k);
    }
    a = wsum(a);
    if (lane == 0) P.logits[v] = a * inv;
  }
  __threadfence();
  CSYNC();
  if (tid == 0) sm.last = atomicAdd(P.head_cnt, 1u) == (unsigned)G - 1;
  CSYNC();
  if (!sm.last) return;
  __threadfence();
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
      c->prev_r = C.prev_w;
      c->prev_w = C.prev_z;
      c->prev_z = C.prev_r;
      c->has_prev = 1;
    }
    c->n_steps_done = C.n_steps_done + 1;
    __threadfence();
  }
}

// BEGIN: zero the next step's accumulator slots, x = embed[token]
// (runtime.py:345) with its statistics and block-0 estimator feeds.
__device__ __forceinline__ void begin_stage(const Prog& P, const ECtl& C, int cta, int G) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nxt = (C.n_steps_done + 1) & 1;
  {
    long long* a = P.acc + (size_t)nxt * P.acc_stride;
    long long* z = P.acc + (size_t)(2 + C.prev_z) * P.acc_stride;
    long long* vs = P.vstat + (size_t)nxt * P.n_inst * 2 * kAccSpread;
    for (int i = cta * NT + tid; i < P.acc_stride / kAccSpread; i += G * NT) {   // the used words only
      a[(size_t)i * kAccSpread] = 0;
      z[(size_t)i * kAccSpread] = 0;
    }
    for (int i = cta * NT + tid; i < P.n_inst * 2; i += G * NT) vs[(size_t)i * kAccSpread] = 0;
  }
  const int n_t = (P.d + 31) / 32;
  for (int tt = cta * NW + warp; tt < n_t; tt += G * NW) {
    const int i = tt * 32 + lane;
    const float v = i < P.d ? __ldg(P.embed + (size_t)C.token * P.d + i) : 0.f;
    if (i < P.d) P.x[i] = v;
    emit_tile(P, C, 0, tt, v);
  }
}

// ---------------------------------------------------------------------------
// The kernel: n_steps decode steps (greedy token feedback on the device when
// n_steps > 1; the host writes the token / mode of a single step).
// ---------------------------------------------------------------------------
extern "C" __global__ void __launch_bounds__(NTB, 1) engine_kernel(const Prog Pk, int n_steps) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int cta = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
  if (tid == 0) {
    sm.prog = Pk;
    sm.work[0].valid = 0;
    sm.work[1].valid = 0;
    sm.dec_op = 0;
    sm.runs_op = -1;
    sm.step_ready = 0;
    s_bar_seen = 0;
    // ring slots: below the LUT (after Smem) and above its zero row
    const uint32_t base = smem_u32(smem_raw);
    uint32_t lo = (base + (uint32_t)sizeof(Smem) + 1023u) & ~1023u;
    int n = 0;
    while (lo + kSlotBytes <= kLut && n < kMaxSlots) { sm.slot_off[n++] = lo - base; lo += kSlotBytes; }
    uint32_t hi = kLut + 256 * 256 + 256;
    while (Pk.upper_slots && hi + kSlotBytes <= base + (uint32_t)Pk.smem_dyn && n < kMaxSlots) {
      sm.slot_off[n++] = hi - base;
      hi += kSlotBytes;
    }
    if (n < kMaxSlots) __trap();        // host sizing guarantees kMaxSlots ring slots
    sm.n_slots = n;
    for (int q = 0; q < n; ++q) {
      mbar_init(&sm.full[q], 1);
      mbar_init(&sm.empty[q], kSlotTiles);
      sm.seq[q] = -1;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const Prog& P = sm.prog;
  if (tid >= NT) {                        // TMA producer warp
    producer(P, sm, cta, G, n_steps);
    return;
  }
  float* lut = reinterpret_cast<float*>(smem_raw + (kLut - smem_u32(smem_raw)));
  __shared__ int s_last;
  int wi = 0, op_no = 0, j_op = 0;
  // barrier epochs continue from previous launches (counter = G x stages so far)
  const unsigned long long e0 = ld_acq64(P.bar) / (unsigned long long)G;   // stages completed before
  unsigned long long k = 0;     // stages completed in this launch
  ECtl& C = sm.ctl;
  for (int step = 0; step < n_steps; ++step) {
    for (int si = 0; si < P.n_stages; ++si) {
      const int2 st = P.stages[si];
      const bool wait = k > 0;
      const unsigned long long target = e0 + k;        // epoch of the previous stage
      if (tid == 0) PROGRESS(0, (step << 16) | si);
      if (st.x == ST_OP) {
        int nsi = si + 1;
        while (nsi < P.n_stages && P.stages[nsi].x != ST_OP) ++nsi;
        const bool has_next = nsi < P.n_stages;
        const bool have_desc = sm.work[wi].valid != 0;
        if (!have_desc) {
          const int nw4 = (int)(sizeof(Op) / 16);
          const int4* src = reinterpret_cast<const int4*>(P.ops + st.y);
          int4* dst = reinterpret_cast<int4*>(&sm.op[wi]);
          for (int q = tid; q < nw4; q += NT) dst[q] = __ldg(src + q);
          CSYNC();
        }
        j_op += op_stage(P, C, sm.op[wi], sm.work[wi], has_next ? &sm.op[wi ^ 1] : nullptr, &sm.work[wi ^ 1],
                         has_next ? P.ops + P.stages[nsi].y : nullptr, sm, cta, G, target, wait,
                         P.dbg ? P.dbg + ((size_t)si * G + cta) * kDbgRec : nullptr, op_no, j_op);
        ++op_no;
        wi ^= 1;
      } else {
        if (wait && st.x != ST_ATTN) bar_wait(P, target);     // attention waits after its K/V prefetch
        if (P.dbg && tid == 0 && st.x != ST_ATTN) P.dbg[((size_t)si * G + cta) * kDbgRec] = gclock();
        if (st.x == ST_BEGIN) {
          read_ctl(P, C);
          if (tid == 0) {
            __threadfence_block();
            sm.step_ready = step + 1;                   // the producer may stream this step
          }
          begin_stage(P, C, cta, G);
        } else if (st.x == ST_ATTN) {
          attn_stage(P, C, st.y, lut, cta, G, &s_last, target, wait,
                     P.dbg ? P.dbg + ((size_t)si * G + cta) * kDbgRec : nullptr);
        } else if (st.x == ST_EMIT) {
          emit_stage(P, C, P.attn, P.d, 4 * st.y + 1, cta, G);
        } else {
          head_stage(P, C, sm, cta, G);
        }
      }
      if (P.dbg && tid == 0) P.dbg[((size_t)si * G + cta) * kDbgRec + 7] = gclock();
      bar_arrive(P, e0 + k + 1, G);
      if (tid == 0) CSTAMP(P.dbg ? P.dbg + ((size_t)si * G + cta) * kDbgRec : nullptr, 17);
      ++k;
    }
  }
}
}  // namespace eng
}  // namespace dpq
