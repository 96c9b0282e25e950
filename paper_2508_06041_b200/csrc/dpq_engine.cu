// Persistent decode-step engine for sm_100a (the fast path of dpq_session).
//
// One cooperative kernel runs whole decode steps (reference DecodeEngine.step,
// runtime.py:330-381) on one CTA per SM. A step is the stage list
//   BEGIN | per block: QKV  O  UPGATE  DOWN | HEAD
// with NO grid barrier between stages: every vector a stage publishes (the
// residual stream, q|k|v, SiLU(gate)*up) and every cross-window partial sum
// is a 64-bit word {float value, u32 epoch} (single-copy atomic, so no fence),
// and a consumer waits only for the words it reads, tagged with the epoch of
// the stage that produces them. A relaxed stage counter (arrive after each
// stage, wait for stage E-2 before writing the buffers of stage E) bounds the
// skew between CTAs so double-buffered state is never overwritten early.
//
// Per op stage (layers sharing one input vector), CTA c owns one 512-column
// window w of the input and a range of (32-row tile, window) groups:
//  * input: the window's 512 values (tagged) -> shared memory; for the o op
//    the window is the attention output of the 512 / head_dim heads it holds,
//    computed in the prologue by every CTA of the window (RoPE, KV append by
//    one CTA, causal softmax over the KV cache; runtime.py:351-362);
//  * byte LUT of the window (257 x 64 fp32) from shared memory;
//  * precision selection (runtime.py:184-193, estimator.py:35-60), fused into
//    the prologue: the CTAs of window w split the estimator rows; each row is
//    a G[w] . x[w] partial (G in f32 / f16 / e4m3), added in fixed point
//    (deterministic) to the layer's accumulator with a release count; the
//    window's first CTA adds sum x, sum x^2. The TMA producer warp of every
//    CTA waits for the counts once it has queued the op's base planes,
//    computes est > T (strict, runtime.py:192) from the same integers, and
//    only then queues the extra planes of the layers that decided high;
//  * the any-precision GEMV streams planes 0..b-1 of the nested store
//    (quant.py:74) through a TMA ring (8 x 16 KB slots, mbarrier full/empty),
//    64 conflict-free byte-LUT lookups (8 weight bits per LDS) per 2 KB item,
//    Horner over planes, the per-(tile, window) sum published as a tagged word;
//  * reduce unit u (a tile, or an up|gate tile pair) belongs to CTA u mod G:
//    it sums its window partials in fixed window order, applies the affine
//    epilogue y = s_in (lo sum x + span 2^-b (S + sum x / 2)) (an exact
//    restatement of quant.py:74-78 @ x), the residual add / SiLU(gate)*up
//    (runtime.py:364-370), and publishes the output tile.
#include "dpq_common.cuh"

// Consumer-only CTA barrier (the producer warp never joins).
#define CSYNC() asm volatile("bar.sync 1, %0;" :: "n"(dpq::eng::NT) : "memory")

namespace dpq {
namespace eng {

constexpr int NT = 480;            // consumer threads per CTA (warps 0..14); 16 warps -> 128 registers
constexpr int NW = NT / 32;        // consumer warps
constexpr int NTB = NT + 32;       // + one TMA producer warp (warp 15)
constexpr int kSlotTiles = 8;      // tiles per ring slot (one plane of up to 8 consecutive tiles)
constexpr int kSlotBytes = kSlotTiles * 2048;
constexpr int kMaxSlots = 8;       // ring slots (power of two)
constexpr int kMaxRuns = 96;       // (layer, window, <= 8 tiles) runs per op per CTA
constexpr int kMaxTiles = 128;     // groups whose parked base sums live in shared memory
constexpr int kMaxTasks = 384;     // (tile, window) groups per CTA and op (the rest park in Prog.park)
constexpr int kCurSlots = 4;       // accumulator slots of the current step (step % 4)
constexpr int kPrevSlots = 4;      // previous-step slots (rotation % 4)
constexpr int kAccSlots = kCurSlots + kPrevSlots;
constexpr int kStatSpread = 16;    // statistics words: one 128-byte line each
constexpr int kDbgRec = 8;         // debug stamps per (stage, CTA): [0] start .. [7] end
constexpr double kFxSum = 4294967296.0;   // 2^32: sum x
constexpr double kFxSq = 16777216.0;      // 2^24: sum x^2
constexpr uint32_t kLut = 0x20000;        // the window LUT (absolute shared address)

enum { ST_BEGIN = 0, ST_OP = 1, ST_HEAD = 3 };
enum { SRC_IMM = 0, SRC_PREV_STEP = 1, SRC_PREV_BLOCK = 2 };
enum { FEED_CUR = 0, FEED_CURFB = 1, FEED_PREV = 2 };
enum { IN_VEC = 0, IN_ATTN = 1 };
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
  int est;                 // EST_NONE / EST_LINEAR / EST_PROJECTION
  int src;                 // SRC_*
  int k;                   // projection rank (0: linear)
  int acc;                 // accumulator set offset in a slot: [k values][sum x^2][count]
  int cnt_expect;          // count of a complete set: n_win(cols) * (k + 1)
  int trace;               // trace column
  double T, slope, intercept;
  double fbscale;          // 2^-fb of the set's G.x values
};

struct alignas(16) Op {
  Layer L[kMaxOpLayers];
  int n_layers;
  int cols, n_win, n_tiles;
  int rms;                 // input RMS-normalised (runtime.py:383-384)
  int pair;                // up|gate SiLU pair epilogue
  int add;                 // residual add: out = res_in + y
  int in_kind;             // IN_VEC / IN_ATTN
  int in_stage;            // stage (index in the step) publishing `in` (IN_ATTN: the q|k|v stage)
  int res_stage;           // stage publishing res_in
  int inst;                // input instance: statistics + estimator feeds
  int block;
  int feed_rows;           // projection rows of the input's feeds (split over the window's CTAs)
  const u64* in;           // tagged input (IN_ATTN: q|k|v)
  const u64* res_in;       // tagged residual input (add)
  u64* out;                // tagged output
};
static_assert(sizeof(Op) % 16 == 0, "Op is copied to shared memory in 16-byte words");

// Estimator feed of one input instance: G [n_win][k][512] (f32 / f16 / e4m3 +
// per-row scale) applied to each window, into the accumulator set `acc`.
struct Feed {
  const void* G;
  const float* gscale;
  int dtype, k, row0;      // row0: first row of this feed in the instance's row list
  int acc;
  int kind;                // FEED_*
  int pad;
  double fxscale;          // 2^fb
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
  const int* feed_begin;   // [n_inst + 1]
  const Feed* feeds;
  int n_inst;
  int d, H, KV, hd, dkv, f, vocab, seq_cap, n_blocks;
  float eps;
  const float* embed;
  const float* lm;
  const float* cosv;
  const float* sinv;
  u64* xe;                 // tagged x = embed[token]
  const u64* xfinal;       // tagged residual after the last block
  int final_stage;
  float* logits;
  float* const* kc;        // [n_blocks] -> [seq_cap][dkv]
  float* const* vc;
  u64* slot;               // [2][slot_half] tagged (tile, window) partial sums
  long long slot_half;
  float* park;             // [G][kMaxTasks - kMaxTiles][32] parked base sums beyond the shared table
  long long* acc;          // [kAccSlots][acc_stride]
  int acc_stride;
  long long* vstat;        // [kCurSlots][n_inst][3 (sum, sumsq, count)][kStatSpread]
  u64* bar;                // stage arrivals (G per stage)
  unsigned* head_cnt;
  unsigned* err;           // sticky error flags (ERR_RANGE: fixed-point range exceeded)
  signed char* tr_bits;
  float* tr_est;
  int n_trace, max_steps;
  int* tok_log;
  ECtl* ctl;
  int smem_dyn;
  u64* dbg;                // optional [n_stages][G][kDbgRec] %globaltimer stamps
};

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
// fixed point with a range check (sticky error flag instead of a silent wrap)
__device__ __forceinline__ long long fx(double v, double scale, unsigned* err) {
  const double s = v * scale;
  if (!(fabs(s) < 4.0e18)) { atomicOr(err, (unsigned)ERR_RANGE); return 0; }
  return llrint(s);
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

// LUT of one 512-column window from the staged window xw: row e, slot g =
// sum_{t: bit t of e} x[8g + t]; row 256 = 0 (target of the wrapped "e - 1"
// encoding for e = 0). Thread u < 256 builds rows [64 q, 64 q + 64) of group
// g (u = 64 q + g).
__device__ __forceinline__ void lut_build(float* lut, const float* xw) {
  const int u = threadIdx.x;
  if (u >= 256) return;
  const int g = u & 63, q = u >> 6;
  const float4 xa = *reinterpret_cast<const float4*>(xw + 8 * g);
  const float4 xb = *reinterpret_cast<const float4*>(xw + 8 * g + 4);
  const float xs[4] = {xa.x, xa.y, xa.z, xa.w};
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
    if (m & 1) H += xb.x;
    if (m & 2) H += xb.y;
    if (m & 4) H += xb.z;
    if (m & 8) H += xb.w;
#pragma unroll
    for (int i = 0; i < 16; ++i) lut[(16 * m + i) * kGroups + g] = L[i] + H;
  }
  if (u < 64) lut[256 * kGroups + u] = 0.f;
}

// ---------------------------------------------------------------------------
// Per-op work of one CTA.
// A group is (32-row tile t, 512-column window w), linear index g = w * n_tiles
// + t (window-major). Window w gets CTAs [ceil(w G / n_win), ceil((w+1) G /
// n_win)) (host guarantees n_win <= G), its groups split among them evenly by
// base planes (known before the decision). The range is cut into runs of <= 8
// tiles of one layer. The TMA producer streams, per run and plane, one bulk
// copy of the run's tiles into a 16 KB ring slot: base planes [0, nb) of all
// runs, then - once the decision is taken - extra planes [nb, fin) of the runs
// whose layer decided high (reverse run order). Consumer task (run, tile) goes
// to warp k % NW; S is accumulated per tile by Horner over planes (S_{p+1} =
// 2 S_p + P_p), the base part parked in shared memory.
// ---------------------------------------------------------------------------
struct Work {
  int nb[kMaxOpLayers];
  int ga, gb;
  int w, cb, m;            // window, its first CTA, CTA count of the window
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
  Prog prog;
  ECtl ctl;                          // control block of the current step
  Op op[2];                          // consumer copies of the current / next op descriptors
  Work work[2];
  RunList runs;                      // consumer run list of the current op
  Op pop;                            // producer copy of the op it streams
  Work pw;
  RunList pruns;
  short pfo[kMaxRuns];
  unsigned char ptask[kMaxTasks];
  unsigned long long full[kMaxSlots], empty[kMaxSlots];   // ring mbarriers
  volatile int seq[kMaxSlots];       // FIFO index armed in each slot (phase disambiguation)
  unsigned slot_off[kMaxSlots];
  volatile int dec_op;               // op counter whose decision and extra tables are published
  volatile int cons_done;            // ops the consumers have finished (tables of op n - 2 are free)
  int runs_op;                       // op counter whose base runs are in runs / fo_bo / task_rb
  volatile int step_ready;           // step whose control block the consumers have loaded
  int dec_fin[2][kMaxOpLayers];      // final bits (op parity)
  short fo_bo[kMaxRuns];
  short fo_eo[2][kMaxRuns], fo_xt[2][kMaxRuns];
  unsigned char task_rb[kMaxTasks];
  unsigned char task_rx[2][kMaxTasks];
  int n_ext_items[2], t_ext[2];
  int last;                          // base items of the current op
  int head_last;
  float head_v[NW];
  int head_i[NW];
  double red[32];
  float sbuf[kMaxTiles][32];         // base-pass S of groups whose layer has extra planes
  float xw[kWinCols];                // the op's input window
};

__device__ __forceinline__ int layer_of(const Op& O, int t) {
  int li = 0;
  while (li + 1 < O.n_layers && t >= O.L[li + 1].tile_off) ++li;
  return li;
}

// First group whose first base item is >= item i (window-local item index).
__device__ __forceinline__ int group_at(const Op& O, const int* nb, int wsum_, int w, int r) {
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

// Work of CTA cta (one warp).
__device__ __forceinline__ void build_work_warp(const Op& O, const ECtl& C, int cta, int G, Work& W) {
  const int lane = threadIdx.x & 31;
  const int nbl = lane < O.n_layers ? base_bit(O.L[lane], C) : 0;
  if (lane < O.n_layers) W.nb[lane] = nbl;
  const int wtot = wsum(lane < O.n_layers ? O.L[lane].n_tiles * nbl : 0);
  __syncwarp();
  const int w = (int)((unsigned)cta * (unsigned)O.n_win / (unsigned)G);
  const int cb = (w * G + O.n_win - 1) / O.n_win, ce = ((w + 1) * G + O.n_win - 1) / O.n_win;
  const int m = ce - cb;
  if (lane < 2) {
    const int idx = cta - cb + lane;
    const int item = (int)((unsigned)idx * (unsigned)wtot / (unsigned)m);
    const int g = group_at(O, W.nb, wtot, w, item);
    if (lane == 0) W.ga = g;
    else W.gb = g;
  }
  if (lane == 0) { W.w = w; W.cb = cb; W.m = m; }
  __syncwarp();
}

// Warp-parallel run list + base FIFO offsets + task -> run table of work W
// (one window; segments = layers, one per lane). Returns the base item count.
__device__ int build_runs_warp(const Op& O, const Work& W, RunList& R, short* fo_bo, unsigned char* task_r) {
  const int lane = threadIdx.x & 31;
  const int nt = O.n_tiles;
  if (W.ga >= W.gb) {
    if (lane == 0) R.n = 0;
    __syncwarp();
    return 0;
  }
  const int w = W.w;
  int lo = 0, len = 0, nr = 0, items = 0;
  const int li = lane;
  if (lane < O.n_layers) {
    const Layer& L = O.L[li];
    lo = max(W.ga - w * nt, L.tile_off);
    const int hi = min(W.gb - w * nt, L.tile_off + L.n_tiles);
    len = max(hi - lo, 0);
    nr = (len + kSlotTiles - 1) / kSlotTiles;
    items = nr * W.nb[li];
  }
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
  for (int k0 = 0; k0 < W.gb - W.ga; k0 += 32) {
    const int kt = k0 + lane;
    const bool ok = kt < W.gb - W.ga;
    const int t = W.ga + (ok ? kt : 0) - w * nt;
    int l2 = 0;
    while (l2 + 1 < O.n_layers && t >= O.L[l2 + 1].tile_off) ++l2;
    const int slo = __shfl_sync(0xffffffffu, lo, l2), srb = __shfl_sync(0xffffffffu, rb, l2);
    if (ok) task_r[kt] = (unsigned char)(srb + (t - slo) / kSlotTiles);
  }
  if (lane == 0) R.n = n_runs;
  __syncwarp();
  return n_items;
}

// Warp-parallel FIFO offsets of the extra planes [nb, fin) once the decision
// is known: runs in reverse order (the producer's issue order), exclusive
// prefix sums of items and tasks, and the extra task -> run table.
__device__ void extra_fifo_warp(const Work& W, const int* fin, const RunList& R, int base_items, short* fo_eo,
                                short* fo_xt, unsigned char* task_rx, int& n_items, int& n_tasks) {
  const int lane = threadIdx.x & 31;
  int carry_i = base_items, carry_t = 0;
  for (int c0 = 0; c0 < R.n; c0 += 32) {
    const int idx = c0 + lane;
    const int r = R.n - 1 - idx;
    int ex = 0, nt = 0;
    if (idx < R.n) {
      ex = fin[R.r[r].li] - W.nb[R.r[r].li];
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
// Epochs, the stage counter and the step control
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned stage_epoch(const Prog& P, int step_no, int si) {
  return (unsigned)step_no * (unsigned)P.n_stages + (unsigned)si + 1u;
}
// every CTA arrives once per stage after its last read of that stage's inputs
__device__ __forceinline__ void stage_arrive(const Prog& P) {
  CSYNC();
  if (threadIdx.x == 0) red_rel_addu64(P.bar, 1ull);
}
// before writing the double-buffered state of stage E: all CTAs are done with E - 2
__device__ __forceinline__ bool stage_done(const Prog& P, unsigned E) {
  if (E <= 2) return true;
  return ld_acq64(P.bar) >= (u64)(E - 2) * gridDim.x;
}

// ---------------------------------------------------------------------------
// Estimator accumulators (fixed point, per step slot) and statistics
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long* acc_slot(const Prog& P, int slot) { return P.acc + (size_t)slot * P.acc_stride; }
__device__ __forceinline__ long long* stat_words(const Prog& P, int cur, int inst) {
  return P.vstat + ((size_t)cur * P.n_inst + inst) * 3 * kStatSpread;
}

// Feed rows of the op's input window (consumer prologue). Rows of all feeds
// of the instance are numbered 0..feed_rows-1; CTA j of the window's m takes
// rows j, j + m, ...; its i-th row goes to warp kFeedW0 + i % kFeedWarps.
// Row r of feed F: partial G_F[w][r] . x[w] in fp32 lanes + double warp sum,
// fixed point at 2^fb, added to the set's accumulator, then a release count.
constexpr int kFeedW0 = 8, kFeedWarps = 6;      // warps 8..13 (warps 0..7 build the LUT)
constexpr int kStatW = 14;                       // statistics warp

struct FeedSel {      // the feed a row belongs to and where it accumulates
  const Feed* F;
  long long* acc;
  int r;
};

__device__ __forceinline__ bool feed_active(const Feed& F, const ECtl& C) {
  const bool dyn = C.mode == MODE_DYNAMIC;
  if (F.kind == FEED_PREV) return dyn || C.prime;
  if (F.kind == FEED_CURFB) return dyn && !C.has_prev;
  return dyn;
}
__device__ __forceinline__ long long* feed_acc(const Prog& P, const ECtl& C, const Feed& F) {
  const int slot = F.kind == FEED_PREV ? kCurSlots + (C.rot & (kPrevSlots - 1)) : (C.n_steps_done & (kCurSlots - 1));
  return acc_slot(P, slot) + F.acc;
}

// Window partial of G row r (lanes: 16 columns each) against xw.
__device__ __forceinline__ double feed_row_dot(const Feed& F, int w, int r, const float* xw) {
  const int lane = threadIdx.x & 31;
  const float* xl = xw + 16 * lane;
  float s = 0.f;
  const size_t base = ((size_t)w * F.k + r) * kWinCols + 16 * lane;
  if (F.dtype == G_F16) {
    const uint4* g = reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(F.G) + base);
    const uint4 a = ld_nc16(g), b = ld_nc16(g + 1);
    const __half2* ha = reinterpret_cast<const __half2*>(&a);
    const __half2* hb = reinterpret_cast<const __half2*>(&b);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 u = __half22float2(ha[i]), v = __half22float2(hb[i]);
      s = fmaf(u.x, xl[2 * i], s);
      s = fmaf(u.y, xl[2 * i + 1], s);
      s = fmaf(v.x, xl[8 + 2 * i], s);
      s = fmaf(v.y, xl[8 + 2 * i + 1], s);
    }
  } else if (F.dtype == G_F32) {
    const uint4* g = reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(F.G) + base);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 a = ld_nc16(g + q);
      s = fmaf(__uint_as_float(a.x), xl[4 * q], s);
      s = fmaf(__uint_as_float(a.y), xl[4 * q + 1], s);
      s = fmaf(__uint_as_float(a.z), xl[4 * q + 2], s);
      s = fmaf(__uint_as_float(a.w), xl[4 * q + 3], s);
    }
  } else {   // e4m3 with a per-row scale
    const uint4 a = ld_nc16(reinterpret_cast<const unsigned char*>(F.G) + base);
    const unsigned wd[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_fp8_e4m3 e;
        e.__x = (unsigned char)(wd[q] >> (8 * j));
        s = fmaf((float)e, xl[4 * q + j], s);
      }
    s *= __ldg(F.gscale + r);
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

// Statistics + feeds of the op's input window (warps kFeedW0.. / kStatW), after
// the LUT build started (xw complete).
__device__ __forceinline__ void window_feeds(const Prog& P, const ECtl& C, const Op& O, const Work& W,
                                             const float* xw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cta = blockIdx.x;
  const int j = cta - W.cb, m = W.m;
  if (warp >= kFeedW0 && warp < kFeedW0 + kFeedWarps) {
    // projection rows: this CTA's i-th row -> warp kFeedW0 + i % kFeedWarps
    for (int i = warp - kFeedW0;; i += kFeedWarps) {
      const int q = j + i * m;
      if (q >= O.feed_rows) break;
      const Feed* F = feed_of_row(P, O.inst, q);
      if (!feed_active(*F, C)) continue;
      const int r = q - F->row0;
      const double v = feed_row_dot(*F, W.w, r, xw);
      if (lane == 0) {
        long long* a = feed_acc(P, C, *F);
        red_add64(a + r, fx(v, F->fxscale, P.err));
        red_rel_add64(a + F->k + 1, 1);          // count (release: the value above is visible first)
      }
    }
  } else if (warp == kStatW && j == 0) {
    // sum x, sum x^2 of the window: op statistics + the feeds' sum x^2 words
    double s = 0.0, q = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double v = (double)xw[16 * lane + i];
      s += v;
      q += v * v;
    }
    s = wsum(s);
    q = wsum(q);
    if (lane == 0) {
      long long* st = stat_words(P, C.n_steps_done & (kCurSlots - 1), O.inst);
      red_add64(st, fx(s, kFxSum, P.err));
      red_add64(st + kStatSpread, fx(q, kFxSq, P.err));
      red_rel_add64(st + 2 * kStatSpread, 1);
    }
    const long long qf = fx(q, kFxSq, P.err);
    for (int f = P.feed_begin[O.inst] + lane; f < P.feed_begin[O.inst + 1]; f += 32) {
      const Feed& F = P.feeds[f];
      if (!feed_active(F, C)) continue;
      long long* a = feed_acc(P, C, F);
      red_add64(a + F.k, qf);
      red_rel_add64(a + F.k + 1, 1);
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

__device__ __noinline__ void attn_window(const Prog& P, const ECtl& C, const Op& O, const Work& W, float* scratch,
                                         float* xw, unsigned e_qkv) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hd = P.hd, qh = P.H / P.KV, b = O.block;
  const int t = C.pos;
  const int h0 = W.w * kWinCols / hd;
  const int nh = min(kWinCols / hd, P.H - h0);
  const int nsub = max(1, NW / nh);
  const int units = nh * nsub;
  const float scale = 1.0f / sqrtf((float)hd);
  const int i0 = 4 * lane;
  const bool act = i0 < hd;
  const int jj = i0 < hd / 2 ? i0 : i0 - hd / 2;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 c4 = act ? __ldg(reinterpret_cast<const float4*>(P.cosv + (size_t)t * (hd / 2) + jj)) : z4;
  const float4 s4 = act ? __ldg(reinterpret_cast<const float4*>(P.sinv + (size_t)t * (hd / 2) + jj)) : z4;
  float* kc = P.kc[b];
  float* vc = P.vc[b];
  const unsigned long long kvpol = l2_evict_last_policy();   // the KV cache is re-read every step
  const int ps = hd + 4;
  bool wrote = false;
  for (int u = warp; u < units; u += NW) {
    const int hh = u % nh, sub = u / nh;
    const int h = h0 + hh, g = h / qh;
    const float4 q4 = act ? rope4(O.in + (size_t)h * hd, i0, hd, c4, s4, e_qkv) : z4;
    float4 kt = z4, vt = z4;
    const bool own_t = (t % nsub) == sub;
    if (own_t && act) {
      kt = rope4(O.in + P.d + (size_t)g * hd, i0, hd, c4, s4, e_qkv);      // RoPE'd k of this step
      vt = tag4(O.in + P.d + P.dkv + (size_t)g * hd + i0, e_qkv);
      if (W.cb == (int)blockIdx.x && h % qh == 0) {                        // KV append (runtime.py:355-356)
        *reinterpret_cast<float4*>(kc + (size_t)t * P.dkv + g * hd + i0) = kt;
        *reinterpret_cast<float4*>(vc + (size_t)t * P.dkv + g * hd + i0) = vt;
        wrote = true;
      }
    }
    float m = -CUDART_INF_F, l = 0.f;
    float4 o = z4;
    // cached positions s < t, 2-deep register pipeline
    float4 k0 = z4, v0 = z4, k1 = z4, v1 = z4;
    int s = sub;
    const size_t goff = (size_t)g * hd + i0;
    if (act && s < t) { k0 = ld_keep(kc + (size_t)s * P.dkv + goff, kvpol); v0 = ld_keep(vc + (size_t)s * P.dkv + goff, kvpol); }
    if (act && s + nsub < t) {
      k1 = ld_keep(kc + (size_t)(s + nsub) * P.dkv + goff, kvpol);
      v1 = ld_keep(vc + (size_t)(s + nsub) * P.dkv + goff, kvpol);
    }
#define ATTN_UPDATE(K_, V_)                                                          \
    {                                                                                \
      const float a = wsum(dot4(q4, K_)) * scale;              /* runtime.py:358 */  \
      const float mn = fmaxf(m, a);                                                  \
      const float corr = expf(m - mn), p = expf(a - mn);       /* runtime.py:359-361 */ \
      l = l * corr + p;                                                              \
      o.x = o.x * corr + p * V_.x; o.y = o.y * corr + p * V_.y;                      \
      o.z = o.z * corr + p * V_.z; o.w = o.w * corr + p * V_.w;                      \
      m = mn;                                                                        \
    }
    for (; s < t; s += 2 * nsub) {
      ATTN_UPDATE(k0, v0)
      if (act && s + 2 * nsub < t) {
        k0 = ld_keep(kc + (size_t)(s + 2 * nsub) * P.dkv + goff, kvpol);
        v0 = ld_keep(vc + (size_t)(s + 2 * nsub) * P.dkv + goff, kvpol);
      }
      if (s + nsub < t) {
        ATTN_UPDATE(k1, v1)
        if (act && s + 3 * nsub < t) {
          k1 = ld_keep(kc + (size_t)(s + 3 * nsub) * P.dkv + goff, kvpol);
          v1 = ld_keep(vc + (size_t)(s + 3 * nsub) * P.dkv + goff, kvpol);
        }
      }
    }
    if (own_t) ATTN_UPDATE(kt, vt)
#undef ATTN_UPDATE
    float* pr = scratch + u * ps;
    if (act) *reinterpret_cast<float4*>(pr + i0) = o;
    if (lane == 0) { pr[hd] = m; pr[hd + 1] = l; }
  }
  if (wrote) __threadfence();        // the appended rows are read by other CTAs in later steps
  CSYNC();
  // merge the nsub units of each head in fixed order -> xw
  for (int q = tid; q < kWinCols; q += NT) {
    const int hh = q / hd, i = q - hh * hd;
    float r = 0.f;
    if (hh < nh) {
      float M = -CUDART_INF_F;
      for (int sb = 0; sb < nsub; ++sb) M = fmaxf(M, scratch[(sb * nh + hh) * ps + hd]);
      float L = 0.f, acc = 0.f;
      for (int sb = 0; sb < nsub; ++sb) {
        const float* pr = scratch + (sb * nh + hh) * ps;
        const float mw = pr[hd];
        const float e = mw == -CUDART_INF_F ? 0.f : expf(mw - M);
        L += e * pr[hd + 1];
        acc += e * pr[i];
      }
      r = acc / L;                                             // runtime.py:362
    }
    xw[q] = r;
  }
}

// ---------------------------------------------------------------------------
// Tile reduction + epilogue (one warp, lane = row of the tile)
// ---------------------------------------------------------------------------
// S of op tile t: sum of the window partials in fixed window order, each
// awaited until it carries this stage's epoch.
__device__ __forceinline__ float tile_S(const u64* slot, const Op& O, int t, unsigned epoch) {
  const int lane = threadIdx.x & 31;
  const int rows = O.n_tiles * 32;
  const u64* base = slot + (size_t)t * 32 + lane;
  float acc = 0.f;
  for (int w0 = 0; w0 < O.n_win; w0 += 8) {
    const int nw = min(8, O.n_win - w0);
    u64 v[8];
    bool ok;
    unsigned n_ = 0;
    u64 t0 = 0;
    do {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < nw) v[j] = ld_relaxed64(base + (size_t)(w0 + j) * rows);
      ok = true;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < nw) ok &= (unsigned)(v[j] >> 32) == epoch;
      if ((++n_ & 1023u) == 0) {
        const u64 t_ = gclock();
        if (t0 == 0) t0 = t_;
        else if (t_ - t0 > 4000000000ull) hang("window partials", t, epoch);
      }
    } while (!__all_sync(0xffffffffu, ok));
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < nw) acc += __uint_as_float((unsigned)v[j]);
  }
  return acc;
}

struct Epi { float scale, sx; };

// op input statistics (sum x, sum x^2) once every window has added them
__device__ __forceinline__ Epi op_epi(const Prog& P, const ECtl& C, const Op& O) {
  const long long* st = stat_words(P, C.n_steps_done & (kCurSlots - 1), O.inst);
  SPIN_UNTIL(ld_acq_s64(st + 2 * kStatSpread) >= O.n_win, "statistics", O.inst, 0);
  const double s = (double)__ldcg(st) * (1.0 / kFxSum);
  const double q = (double)__ldcg(st + kStatSpread) * (1.0 / kFxSq);
  Epi e;
  e.sx = (float)s;
  e.scale = O.rms ? (float)rsqrt_d(q / (double)O.cols + (double)P.eps) : 1.f;
  return e;
}

__device__ __forceinline__ float tile_y(const u64* slot, const Op& O, const int* fin, const Epi& E, int t,
                                        unsigned epoch, int& li, int& r, bool& valid) {
  const int lane = threadIdx.x & 31;
  li = layer_of(O, t);
  const Layer& L = O.L[li];
  const float S = tile_S(slot, O, t, epoch);
  r = (t - L.tile_off) * 32 + lane;
  valid = r < L.rows;
  if (!valid) return 0.f;
  const float lo = __ldg(L.lo + r), span = __ldg(L.span + r);
  return E.scale * (lo * E.sx + ldexpf(span, -fin[li]) * (S + 0.5f * E.sx));
}

// ---------------------------------------------------------------------------
// The TMA producer warp: streams every op's planes into the ring, running
// ahead of the consumers (bounded by ring space), and takes each op's
// decisions (runtime.py:184-193) once the base planes are queued.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void decide_op(const Prog& P, const ECtl& C, const Op& O, const Work& W, int* fin,
                                          int cta) {
  const int lane = threadIdx.x & 31;
  const bool dyn = C.mode == MODE_DYNAMIC;
  for (int li = 0; li < O.n_layers; ++li) {
    const Layer& L = O.L[li];
    int bit = W.nb[li];
    double est = CUDART_NAN;
    const bool estimating = dyn && L.sentinel == 0 && L.est != EST_NONE;
    if (estimating) {
      const int slot = (L.src == SRC_PREV_STEP && C.has_prev) ? kCurSlots + ((C.rot - 1) & (kPrevSlots - 1))
                                                              : (C.n_steps_done & (kCurSlots - 1));
      const long long* a = acc_slot(P, slot) + L.acc;
      if (lane == 0) SPIN_UNTIL(ld_acq_s64(a + L.k + 1) >= L.cnt_expect, "estimator feeds", L.trace, L.cnt_expect);
      __syncwarp();
      double q = 0.0;
      for (int i = lane; i < L.k; i += 32) {
        const double g = (double)__ldcg(a + i) * L.fbscale;
        q += g * g;
      }
      q = wsum(q);
      const double sq = (double)__ldcg(a + L.k) * (1.0 / kFxSq);
      const double sc = O.rms ? rsqrt_d(sq / (double)O.cols + (double)P.eps) : 1.0;
      if (L.est == EST_PROJECTION) est = q > 0.0 ? sc * q * rsqrt_d(q) : 0.0;                 // estimator.py:56-57
      else est = L.slope * (sq > 0.0 ? sc * sq * rsqrt_d(sq) : 0.0) + L.intercept;           // estimator.py:41-42
      if (!C.force) bit = est > L.T ? L.h : L.l;                                              // strict > (runtime.py:192)
    }
    fin[li] = bit;
    if (lane == 0 && dyn && cta == 0 && L.trace >= 0 && P.n_trace > 0 && C.trace_step < P.max_steps) {
      const size_t o = (size_t)C.trace_step * P.n_trace + L.trace;
      P.tr_bits[o] = (signed char)bit;
      P.tr_est[o] = estimating ? (float)est : CUDART_NAN_F;
    }
  }
  __syncwarp();
}

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
      SPIN_UNTIL_NS(mbar_test(a, par), "producer slot", j, op_no, 12000000000ull);
      // the consumers' generic reads of the slot precede this async-proxy write
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    sm.seq[slot] = j;
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
      {
        const int nw4 = (int)(sizeof(Op) / 16);
        const int4* src = reinterpret_cast<const int4*>(P.ops + st.y);
        int4* dst = reinterpret_cast<int4*>(&sm.pop);
        for (int q = lane; q < nw4; q += 32) dst[q] = __ldg(src + q);
      }
      __syncwarp();
      const Op& O = sm.pop;
      build_work_warp(O, C, cta, G, sm.pw);
      const int nbi = build_runs_warp(O, sm.pw, sm.pruns, sm.pfo, sm.ptask);   // same runs as the consumers'
      const RunList& R = sm.pruns;
      if (lane == 0)
        for (int r = 0; r < R.n; ++r)
          for (int p = 0; p < sm.pw.nb[R.r[r].li]; ++p) issue(O, R.r[r], p);
      __syncwarp();
      const int par = op_no & 1;
      int fin[kMaxOpLayers];
      decide_op(P, C, O, sm.pw, fin, cta);
      // the decision tables are double-buffered by op parity: the consumers
      // must be done with op op_no - 2 before they are overwritten
      if (lane == 0) SPIN_UNTIL_NS(sm.cons_done >= op_no - 1, "consumer progress", op_no, sm.cons_done, 12000000000ull);
      __syncwarp();
      if (lane < O.n_layers) sm.dec_fin[par][lane] = lane == 0 ? fin[0] : lane == 1 ? fin[1] : fin[2];
      int ni, nt;
      extra_fifo_warp(sm.pw, fin, R, nbi, sm.fo_eo[par], sm.fo_xt[par], sm.task_rx[par], ni, nt);
      if (lane == 0) {
        sm.n_ext_items[par] = ni;
        sm.t_ext[par] = nt;
        __threadfence_block();
        sm.dec_op = op_no + 1;          // the consumers may now run the extra planes
        for (int r = R.n - 1; r >= 0; --r) {
          const int li = R.r[r].li;
          for (int p = sm.pw.nb[li]; p < fin[li]; ++p) issue(O, R.r[r], p);
        }
      }
      __syncwarp();
      ++op_no;
    }
  }
}

// ---------------------------------------------------------------------------
// The op stage (consumer warps 0..NW-1)
// ---------------------------------------------------------------------------
// Reduction of the op's units: unit u belongs to CTA u mod G, its i-th unit to
// warp i mod NW. Warp NW - 1 first prepares the next op's work and runs.
__device__ __forceinline__ void reduce_duty(const Prog& P, const ECtl& C, const Op& O, Smem& sm, int cta, int G,
                                            unsigned epoch, const int* fin, const u64* slot, Op* On, Work* Wn,
                                            int op_no, unsigned e_res) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_units = O.pair ? O.L[0].n_tiles : O.n_tiles;
  const int mine = n_units > cta ? (n_units - cta + G - 1) / G : 0;
  if (warp == NW - 1 && On && !Wn->valid) {
    build_work_warp(*On, C, cta, G, *Wn);
    const int nbi = build_runs_warp(*On, *Wn, sm.runs, sm.fo_bo, sm.task_rb);
    if (lane == 0) {
      Wn->valid = 1;
      sm.last = nbi;
      sm.runs_op = op_no + 1;
    }
  }
  if (mine == 0) return;
  const Epi E = op_epi(P, C, O);
  for (int i = warp; i < mine; i += NW) {
    const int u = cta + i * G;
    if (O.pair) {
      const int half = O.L[0].n_tiles;
      int li, r, li2, r2;
      bool ok, ok2;
      const float up = tile_y(slot, O, fin, E, u, epoch, li, r, ok);
      const float gt = tile_y(slot, O, fin, E, u + half, epoch, li2, r2, ok2);
      if (ok) st_tag(O.out + r, up * (gt / (1.0f + expf(-gt))), epoch);        // runtime.py:368
    } else {
      int li, r;
      bool ok;
      const float y = tile_y(slot, O, fin, E, u, epoch, li, r, ok);
      if (ok) {
        const int o = O.L[li].out_off + r;
        float v = y;
        if (O.add) {                                                            // runtime.py:364, 370
          u64 x;
          SPIN_UNTIL((x = ld_relaxed64(O.res_in + o), (unsigned)(x >> 32) == e_res), "residual", o, e_res);
          v = __uint_as_float((unsigned)x) + y;
        }
        st_tag(O.out + o, v, epoch);
      }
    }
  }
}

__device__ __forceinline__ int op_stage(const Prog& P, const ECtl& C, const Op& O, Work& W, Op* On, Work* Wn,
                                        const Op* On_global, Smem& sm, int cta, int G, unsigned epoch,
                                        unsigned step_base, u64* dbg, int op_no, int j_op) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = op_no & 1;
  // ---- work and base runs (decision independent)
  const bool built = W.valid != 0;
  CSYNC();
  if (!built) {
    if (warp == 0) build_work_warp(O, C, cta, G, W);
    CSYNC();
  }
  if (warp == 0 && sm.runs_op != op_no) {
    const int nbi = build_runs_warp(O, W, sm.runs, sm.fo_bo, sm.task_rb);
    if (lane == 0) sm.last = nbi;
  }
  if (dbg && tid == 0) dbg[0] = gclock();
  // the next op's descriptor -> shared memory (its work is built in the reduce phase)
  if (warp == NW - 1 && On && !Wn->valid) {
    const int nw4 = (int)(sizeof(Op) / 16);
    const int4* src = reinterpret_cast<const int4*>(On_global);
    int4* dst = reinterpret_cast<int4*>(On);
    for (int q = lane; q < nw4; q += 32) dst[q] = __ldg(src + q);
  }
  // ---- input window -> xw (skew bound checked on the way: stage E - 2 done)
  float* lut = reinterpret_cast<float*>(reinterpret_cast<char*>(&sm) + (kLut - smem_u32(&sm)));
  if (tid == 32) SPIN_UNTIL(stage_done(P, epoch), "stage counter", epoch, 0);
  if (O.in_kind == IN_ATTN) {
    attn_window(P, C, O, W, lut, sm.xw, step_base + (unsigned)O.in_stage + 1u);
  } else {
    load_window(O.in, O.cols, W.w, step_base + (unsigned)O.in_stage + 1u, sm.xw);
  }
  CSYNC();
  if (dbg && tid == 0) dbg[1] = gclock();
  // ---- LUT (warps 0..7) | estimator feeds and statistics (warps 8..14)
  lut_build(lut, sm.xw);
  window_feeds(P, C, O, W, sm.xw);
  CSYNC();
  if (dbg && tid == 0) dbg[2] = gclock();
  // ---- stream: tasks (run, tile) in FIFO order
  const RunList& R = sm.runs;
  const unsigned char* dyn0 = reinterpret_cast<const unsigned char*>(&sm);
  const uint32_t lanereg = kLut | ((uint32_t)lane * 4u);
  const int n_base = sm.last;
  u64* slot = P.slot + (size_t)(epoch & 1u) * P.slot_half + (size_t)W.w * O.n_tiles * 32;
  for (int kind = 0; kind < 2; ++kind) {
    if (kind) {
      if (lane == 0) SPIN_UNTIL_NS(sm.dec_op >= op_no + 1, "decision", op_no, 0, 8000000000ull);
      __syncwarp();
      __threadfence_block();
    }
    const int n_tasks = kind ? sm.t_ext[par] : W.gb - W.ga;
    for (int kt = warp; kt < n_tasks; kt += NW) {
      const int r = kind ? sm.task_rx[par][kt] : sm.task_rb[kt];
      const Run& q = R.r[r];
      const int i = kt - (kind ? sm.fo_xt[par][r] : q.k0);
      const int nb = W.nb[q.li];
      const int fin = kind ? sm.dec_fin[par][q.li] : nb;
      const int p0 = kind ? nb : 0, p1 = kind ? fin : nb;
      const int jr = j_op + (kind ? sm.fo_eo[par][r] : sm.fo_bo[r]);
      const int pk = q.k0 + i;                                   // group index in [ga, gb)
      float S = 0.f;
      if (kind) S = pk < kMaxTiles ? sm.sbuf[pk][lane]
                                   : __ldcg(P.park + ((size_t)cta * (kMaxTasks - kMaxTiles) + pk - kMaxTiles) * 32 + lane);
      for (int p = p0; p < p1; ++p) {
        const int j = jr + (p - p0);
        const int sl = j & (kMaxSlots - 1);
        if (lane == 0) SPIN_UNTIL_NS(sm.seq[sl] == j, "ring sequence", j, sm.seq[sl], 2000000000ull);
        __syncwarp();
        const uint32_t fa = smem_u32(&sm.full[sl]);
        const unsigned fpar = (unsigned)((j / kMaxSlots) & 1);
        SPIN_UNTIL_NS(mbar_test(fa, fpar), "ring slot", j, fpar, 2000000000ull);
        const uint4* d = reinterpret_cast<const uint4*>(dyn0 + sm.slot_off[sl] + i * kTileBytes) + lane;
        const uint4 d0 = d[0], d1 = d[32], d2 = d[64], d3 = d[96];
        __syncwarp();
        if (lane == 0) mbar_arrive_n(&sm.empty[sl], i == q.nt - 1 ? (unsigned)(kSlotTiles + 1 - q.nt) : 1u);
        S = 2.f * S + plane_sum(d0, d1, d2, d3, lanereg);       // Horner over planes
      }
      const int t = q.t0 + i;
      // base pass of a layer that may still add planes: park; else publish
      const bool may_extra = !kind && C.mode == MODE_DYNAMIC && !C.force && O.L[q.li].sentinel == 0 &&
                             O.L[q.li].est != EST_NONE && O.L[q.li].h > nb;
      if (may_extra) {
        if (pk < kMaxTiles) sm.sbuf[pk][lane] = S;
        else __stcg(P.park + ((size_t)cta * (kMaxTasks - kMaxTiles) + pk - kMaxTiles) * 32 + lane, S);
      }
      if (!may_extra || kind) st_tag(slot + (size_t)t * 32 + lane, S, epoch);
    }
    if (!kind) {
      CSYNC();          // parked base sums visible
      // groups that parked but whose layer decided low: publish the base sum
      if (lane == 0) SPIN_UNTIL_NS(sm.dec_op >= op_no + 1, "decision", op_no, 0, 8000000000ull);
      __syncwarp();
      __threadfence_block();
      for (int kt = warp; kt < W.gb - W.ga; kt += NW) {
        const int r = sm.task_rb[kt];
        const Run& q = R.r[r];
        const int nb = W.nb[q.li];
        const bool may_extra = C.mode == MODE_DYNAMIC && !C.force && O.L[q.li].sentinel == 0 &&
                               O.L[q.li].est != EST_NONE && O.L[q.li].h > nb;
        if (!may_extra || sm.dec_fin[par][q.li] > nb) continue;
        const int i = kt - q.k0, pk = kt;
        const float S = pk < kMaxTiles ? sm.sbuf[pk][lane]
                                       : __ldcg(P.park + ((size_t)cta * (kMaxTasks - kMaxTiles) + pk - kMaxTiles) * 32 + lane);
        st_tag(slot + (size_t)(q.t0 + i) * 32 + lane, S, epoch);
      }
    }
  }
  CSYNC();              // every warp is done with the run tables (the reduce phase rebuilds them)
  if (dbg && tid == 0) dbg[3] = gclock();
  // ---- reduce this CTA's units of the op, then the stage is done
  const int fin3[kMaxOpLayers] = {sm.dec_fin[par][0], sm.dec_fin[par][1], sm.dec_fin[par][2]};
  const int n_ext = sm.n_ext_items[par];
  const unsigned e_res = O.add ? step_base + (unsigned)O.res_stage + 1u : 0u;
  reduce_duty(P, C, O, sm, cta, G, epoch, fin3, P.slot + (size_t)(epoch & 1u) * P.slot_half, On, Wn, op_no, e_res);
  if (dbg && tid == 0) dbg[4] = gclock();
  CSYNC();
  if (tid == 0) {
    W.valid = 0;
    sm.cons_done = op_no + 1;
  }
  return n_base + n_ext;
}

// ---------------------------------------------------------------------------
// Head stage: final RMSNorm + lm_head logits (runtime.py:372), greedy argmax
// (runtime.py:405-408) and the end-of-step control update (runtime.py:373-380).
// ---------------------------------------------------------------------------
__device__ __noinline__ void head_stage(const Prog& P, const ECtl& C, Smem& sm, float* xs, int cta, int G,
                                        unsigned e_final) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the final residual (tagged) -> shared memory, sum of squares in fixed order
  double q = 0.0;
  for (int i = tid; i < P.d; i += NT) {
    u64 x;
    SPIN_UNTIL((x = ld_relaxed64(P.xfinal + i), (unsigned)(x >> 32) == e_final), "final x", i, e_final);
    const float v = __uint_as_float((unsigned)x);
    xs[i] = v;
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
  __threadfence();
  CSYNC();
  if (tid == 0) sm.head_last = atomicAdd(P.head_cnt, 1u) == (unsigned)G - 1;
  CSYNC();
  if (!sm.head_last) return;
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
      c->rot = C.rot + 1;
      c->has_prev = 1;
    }
    __threadfence();
    asm volatile("st.release.gpu.global.s32 [%0], %1;" :: "l"(&c->n_steps_done), "r"(C.n_steps_done + 1) : "memory");
  }
}

// BEGIN: the step's control block, zeroing of the accumulator slots used two
// steps ahead, x = embed[token] (runtime.py:345) as a tagged vector.
__device__ __forceinline__ void begin_stage(const Prog& P, Smem& sm, int cta, int G, int step, int expect_done,
                                            unsigned epoch) {
  const int tid = threadIdx.x;
  if (tid == 0) SPIN_UNTIL(ld_acq_s32(&P.ctl->n_steps_done) >= expect_done, "step control", expect_done, 0);
  CSYNC();
  {
    const int* src = reinterpret_cast<const int*>(P.ctl);
    int* dst = reinterpret_cast<int*>(&sm.ctl);
    if (tid < (int)(sizeof(ECtl) / 4)) dst[tid] = __ldcg(src + tid);
  }
  CSYNC();
  if (tid == 0) {
    __threadfence_block();
    sm.step_ready = step + 1;                   // the producer may stream this step
  }
  const ECtl& C = sm.ctl;
  {
    long long* a = acc_slot(P, (C.n_steps_done + 2) & (kCurSlots - 1));
    long long* z = acc_slot(P, kCurSlots + ((C.rot + 1) & (kPrevSlots - 1)));
    long long* vs = stat_words(P, (C.n_steps_done + 2) & (kCurSlots - 1), 0);
    for (int i = cta * NT + tid; i < P.acc_stride; i += G * NT) { a[i] = 0; z[i] = 0; }
    for (int i = cta * NT + tid; i < P.n_inst * 3; i += G * NT) vs[(size_t)i * kStatSpread] = 0;
  }
  for (int i = cta * NT + tid; i < P.d; i += G * NT) st_tag(P.xe + i, __ldg(P.embed + (size_t)C.token * P.d + i), epoch);
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
    sm.cons_done = 0;
    sm.runs_op = -1;
    sm.step_ready = 0;
    // ring slots: below the LUT (after Smem) and above its zero row
    const uint32_t base = smem_u32(smem_raw);
    uint32_t lo = (base + (uint32_t)sizeof(Smem) + 1023u) & ~1023u;
    int n = 0;
    while (lo + kSlotBytes <= kLut && n < kMaxSlots) { sm.slot_off[n++] = lo - base; lo += kSlotBytes; }
    uint32_t hi = kLut + kLutBytes;
    while (hi + kSlotBytes <= base + (uint32_t)Pk.smem_dyn && n < kMaxSlots) {
      sm.slot_off[n++] = hi - base;
      hi += kSlotBytes;
    }
    if (n < kMaxSlots) __trap();        // host sizing guarantees kMaxSlots ring slots
    for (int q = 0; q < kMaxSlots; ++q) {
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
  const int s0 = __ldcg(&P.ctl->n_steps_done);   // steps completed before this launch
  int wi = 0, op_no = 0, j_op = 0;
  for (int step = 0; step < n_steps; ++step) {
    const unsigned step_base = (unsigned)(s0 + step) * (unsigned)P.n_stages;
    for (int si = 0; si < P.n_stages; ++si) {
      const int2 st = P.stages[si];
      const unsigned epoch = step_base + (unsigned)si + 1u;
      u64* dbg = P.dbg ? P.dbg + ((size_t)si * G + cta) * kDbgRec : nullptr;
      if (st.x == ST_OP) {
        int nsi = si + 1;
        while (nsi < P.n_stages && P.stages[nsi].x != ST_OP) ++nsi;
        const bool has_next = nsi < P.n_stages;
        if (sm.work[wi].valid == 0) {
          CSYNC();
          const int nw4 = (int)(sizeof(Op) / 16);
          const int4* src = reinterpret_cast<const int4*>(P.ops + st.y);
          int4* dst = reinterpret_cast<int4*>(&sm.op[wi]);
          for (int q = tid; q < nw4; q += NT) dst[q] = __ldg(src + q);
          CSYNC();
        }
        j_op += op_stage(P, sm.ctl, sm.op[wi], sm.work[wi], has_next ? &sm.op[wi ^ 1] : nullptr, &sm.work[wi ^ 1],
                         has_next ? P.ops + P.stages[nsi].y : nullptr, sm, cta, G, epoch, step_base, dbg, op_no,
                         j_op);
        ++op_no;
        wi ^= 1;
      } else if (st.x == ST_BEGIN) {
        if (dbg && tid == 0) dbg[0] = gclock();
        begin_stage(P, sm, cta, G, step, s0 + step, epoch);
      } else {
        if (dbg && tid == 0) dbg[0] = gclock();
        head_stage(P, sm.ctl, sm, lut, cta, G, step_base + (unsigned)P.final_stage + 1u);
      }
      if (dbg && tid == 0) dbg[7] = gclock();
      stage_arrive(P);
    }
  }
}
}  // namespace eng
}  // namespace dpq
