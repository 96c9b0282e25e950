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
//    over the grid at (tile, window) granularity, decision-dependent extra
//    planes are split evenly again after the decision; per item a warp does
//    64 conflict-free byte-LUT lookups (8 weight bits per LDS);
//  * every warp keeps a DEPTH-deep register ring of plane loads that runs
//    ahead across op boundaries (the next op's base planes are issued before
//    the barrier), and each CTA prefetches its next-op share into L2;
//  * the last contributor of a (tile | up-gate tile pair) reduces it over
//    windows in fixed order and applies the affine epilogue
//    y = s_in * (lo * sum x + span 2^-b (S + sum x / 2)) (exact restatement of
//    quant.py:74-78 @ x), residual add / SiLU(gate)*up (runtime.py:364-370),
//    and feeds the next estimators.
#include "dpq_common.cuh"

namespace dpq {
namespace eng {

constexpr int NT = 384;            // threads per CTA
constexpr int NW = NT / 32;        // warps per CTA
constexpr int DEPTH = 4;           // register ring depth (plane items in flight per warp; slots a, b, c, e)
constexpr int kMaxRuns = 48;
constexpr int kMaxChunks = 48;
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
  float* slot_base;        // [max_win][slot_stride]
  float* slot_extra;
  int slot_stride;
  unsigned* tile_cnt;
  float* attn_part;        // [H][max_chunks][hd + 2]
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
  unsigned long long* dbg; // optional per-stage timestamps [stages][grid][8]
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
// Spin-wait watchdog: a wait beyond 4 s traps (a launch error instead of a
// hang). No call, so nothing is spilled around the polling loops.
#define hang(what, a, b) __trap()
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
// row 256 = 0 (target of the wrapped "e - 1" encoding for e = 0).
__device__ __forceinline__ void build_lut(float* lut, const float* xw) {
  for (int u = threadIdx.x; u < 512; u += NT) {
    const int g = u & 63, rb = u >> 6;   // rb: 8 blocks of 32 rows
    const float* xg = xw + 8 * g;
    float L[16];
    L[0] = 0.f;
#pragma unroll
    for (int n = 1; n < 16; ++n) {
      const int low = n & (-n);
      L[n] = L[n ^ low] + xg[__ffs(low) - 1];
    }
    const float x4 = xg[4], x5 = xg[5], x6 = xg[6], x7 = xg[7];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int m = 2 * rb + hh;
      float H = 0.f;
      if (m & 1) H += x4;
      if (m & 2) H += x5;
      if (m & 4) H += x6;
      if (m & 8) H += x7;
#pragma unroll
      for (int i = 0; i < 16; ++i) lut[(16 * m + i) * kGroups + g] = L[i] + H;
    }
    if (rb == 0) lut[256 * kGroups + g] = 0.f;
  }
}

// ---------------------------------------------------------------------------
// Per-op work of one CTA.
// A group is (32-row tile t, 512-column window w), linear index g = w * n_tiles
// + t (window-major). Groups are split over the grid by their base planes
// (known before the decision), CTA c owning [ga, gb) starting at the first
// group at or after item c*N/G. Warp k of a CTA owns groups ga + k + NW*j and
// streams, in order, the base planes of all its groups, then the extra planes
// (l..b-1) of those whose layer decided high; S is accumulated per group by
// Horner over planes (S_{p+1} = 2 S_p + P_p), the base part parked in shared
// memory between the two passes.
// ---------------------------------------------------------------------------
constexpr int kMaxGroups = 16;     // groups per warp per op
constexpr int kMaxItems = kMaxGroups * 8;
constexpr uint32_t kLutA = 0x10000, kLutB = 0x20000;   // two resident window LUTs

struct Work {
  int nb[kMaxOpLayers], fin[kMaxOpLayers];
  int ga, gb;
  int valid;
};

struct Smem {
  Prog prog;               // program descriptor (kernel parameter copy)
  ECtl ctl;                // control block of the current step (read at BEGIN)
  Op op[2];                // shared-memory copies of the current / next op descriptors
  Work work[2];            // current / next op
  float xw[2][kWinCols];
  float scale, sx;         // op input scale (1/rms or 1) and sum of raw input
  int last;
  double red[32];
  float head_v[NW];
  int head_i[NW];
  float sbuf[NW][kMaxGroups][32];   // base-pass S of groups with extra planes
  const uint4* ia[NW][kMaxItems];   // per-warp item list: plane address (lane 0)
  unsigned im[NW][kMaxItems];       // item meta: k | p << 8 | pass << 12 | last << 13 | lutB << 14
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
  int nb[kMaxOpLayers];
  int wsum = 0;
  for (int li = 0; li < O.n_layers; ++li) {
    nb[li] = base_bit(O.L[li], C);
    wsum += O.L[li].n_tiles * nb[li];
  }
  const unsigned N = (unsigned)wsum * (unsigned)O.n_win;   // host guarantees N * G < 2^32
  if (lane < 2) {
    const int g = group_at(O, nb, wsum, (int)(N * (unsigned)(cta + lane) / (unsigned)G));
    if (lane == 0) W.ga = g;
    else W.gb = g;
  }
  if (lane < O.n_layers) {
    W.nb[lane] = nb[lane];
    W.fin[lane] = nb[lane];
  }
  if (lane == 0) W.valid = 1;
}

// Plane address (lane 0) of plane p of group g.
__device__ __forceinline__ const uint4* group_plane(const Op& O, int g, int p) {
  const int w = g / O.n_tiles, t = g - w * O.n_tiles;
  const Layer& L = O.L[layer_of(O, t)];
  return L.planes + p * L.pstride + ((long long)w * L.n_tiles + (t - L.tile_off)) * (kTileBytes / 16);
}

// ---------------------------------------------------------------------------
// Vector emission: statistics + estimator feeds of one 32-row tile (a warp;
// lane = row). v = value (0 for padding rows).
// ---------------------------------------------------------------------------
__device__ __noinline__ void emit_tile(const Prog& P, const ECtl& C, int inst, int tile, float v) {
  const int lane = threadIdx.x & 31;
  const int cur = C.n_steps_done & 1;
  const double dv = (double)v;
  const double s = wsum(dv), q = wsum(dv * dv);
  if (lane == 0) {
    long long* vs = P.vstat + ((size_t)cur * P.n_inst + inst) * 2;
    red_add64(vs, fx(s, kFxSum));
    red_add64(vs + 1, fx(q, kFxSq));
  }
  const bool dyn = C.mode == MODE_DYNAMIC;
  const bool upd = dyn || C.prime;
  for (int fi = P.feed_begin[inst]; fi < P.feed_begin[inst + 1]; ++fi) {
    Feed F;
    {
      const int4* fp = reinterpret_cast<const int4*>(P.feeds + fi);
      int4* fd = reinterpret_cast<int4*>(&F);
#pragma unroll
      for (int q = 0; q < (int)(sizeof(Feed) / 16); ++q) fd[q] = __ldg(fp + q);
    }
    long long* acc;
    if (F.kind == FEED_PREV) {
      if (!upd) continue;
      acc = P.acc + (size_t)(2 + C.prev_w) * P.acc_stride + F.acc;
    } else {
      if (!dyn) continue;
      if (F.kind == FEED_CURFB && C.has_prev) continue;
      acc = P.acc + (size_t)cur * P.acc_stride + F.acc;
    }
    if (F.Gt) {
      // block of tile: [sub][chunk][lane][16 B]; f16 chunk = 4 rows x half2,
      // f32 chunk = 2 rows x float2; lane owns k pair (2 lane, 2 lane + 1) of sub.
      const int nsub = F.kpad / 64;
      for (int sub = 0; sub < nsub; ++sub) {
        float g0 = 0.f, g1 = 0.f;
        if (F.f16) {
          const uint4* blk = F.Gt + ((size_t)tile * nsub + sub) * 256 + lane;
          uint4 c[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) c[i] = __ldg(blk + 32 * i);
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
            for (int i = 0; i < 8; ++i) c[i] = __ldg(blk + 32 * (8 * hb + i));
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
        const double sc = ldexp(1.0, F.fb);
        if (k0 < F.k) red_add64(acc + k0, fx((double)g0, sc));
        if (k0 + 1 < F.k) red_add64(acc + k0 + 1, fx((double)g1, sc));
      }
    }
    if (lane == 0) red_add64(acc + F.k, fx(q, kFxSq));
  }
}

// ---------------------------------------------------------------------------
// Grid barrier (monotonic 64-bit arrival counter)
// ---------------------------------------------------------------------------
// bar[0]: arrival counter (G per stage, monotonic); bar[16 * (1 + i)], i < 8:
// release flags (the stage epoch), written by the last arriver; CTA c polls
// flag c % 8 (separate lines: polling never contends with the arrivals).
__device__ __forceinline__ void bar_arrive(const Prog& P, unsigned long long epoch, int G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long old = atomicAdd(P.bar, 1ull);
    if (old + 1 == epoch * (unsigned long long)G) {
      __threadfence();
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(P.bar + 16 * (1 + i)), "l"(epoch) : "memory");
    }
  }
}
__device__ __forceinline__ void bar_wait(const Prog& P, unsigned long long epoch) {
  if (threadIdx.x == 0) {
    const unsigned long long* f = P.bar + 16 * (1 + (blockIdx.x & 7));
    if (ld_acq64(f) < epoch) {
      const unsigned long long t0 = gclock();
      while (ld_acq64(f) < epoch) {
        if (gclock() - t0 > 4000000000ull) hang("grid barrier", 0, (long long)epoch);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void read_ctl(const Prog& P, ECtl& C) {
  const int* src = reinterpret_cast<const int*>(P.ctl);
  int* dst = reinterpret_cast<int*>(&C);
  __syncthreads();
  if (threadIdx.x < (int)(sizeof(ECtl) / 4)) dst[threadIdx.x] = __ldcg(src + threadIdx.x);
  __syncthreads();
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

// L2 prefetch of this CTA's base planes of op O: one (window, layer, plane)
// contiguous stripe per thread.
__device__ __noinline__ void prefetch_work_l2(const Op& O, const Work& W) {
  if (W.ga >= W.gb) return;
  int idx = 0;
  for (int w = W.ga / O.n_tiles; w <= (W.gb - 1) / O.n_tiles; ++w) {
    const int t_lo = max(W.ga - w * O.n_tiles, 0), t_hi = min(W.gb - w * O.n_tiles, O.n_tiles);
    for (int li = 0; li < O.n_layers; ++li) {
      const Layer& L = O.L[li];
      const int t0 = max(t_lo, L.tile_off), t1 = min(t_hi, L.tile_off + L.n_tiles);
      if (t0 >= t1) continue;
      for (int p = 0; p < W.nb[li]; ++p, ++idx) {
        if ((idx % NT) != (int)threadIdx.x) continue;
        const char* a = reinterpret_cast<const char*>(L.planes + p * L.pstride + ((long long)w * L.n_tiles + (t0 - L.tile_off)) * 128);
        long long bytes = (long long)(t1 - t0) * kTileBytes;
        while (bytes > 0) {
          const unsigned c = (unsigned)min(bytes, 65536LL);
          l2_prefetch(a, c);
          a += c;
          bytes -= c;
        }
      }
    }
  }
}

// L2 prefetch of slice cta/G of the G^T blocks the op's output feeds.
__device__ __noinline__ void prefetch_feeds_l2(const Prog& P, const ECtl& C, int inst, int n, int cta, int G) {
  if (inst < 0 || C.mode != MODE_DYNAMIC && !C.prime) return;
  const int nt = (n + 31) / 32;
  for (int fi = P.feed_begin[inst] + (int)threadIdx.x; fi < P.feed_begin[inst + 1]; fi += NT) {
    const Feed F = P.feeds[fi];
    if (!F.Gt) continue;
    const long long bytes = (long long)nt * (F.kpad / 64) * (F.f16 ? 4096 : 8192);
    const long long lo = bytes * cta / G / 16 * 16, hi = bytes * (cta + 1) / G / 16 * 16;
    const char* a = reinterpret_cast<const char*>(F.Gt) + lo;
    long long left = hi - lo;
    while (left > 0) {
      const unsigned c = (unsigned)min(left, 65536LL);
      l2_prefetch(a, c);
      a += c;
      left -= c;
    }
  }
}

// ---------------------------------------------------------------------------
// Tile reduction + epilogue (one warp, lane = row of the tile)
// ---------------------------------------------------------------------------
// S of op tile t: sum of the window slots in fixed order.
__device__ __forceinline__ float tile_S(const Prog& P, const Op& O, int t) {
  const int lane = threadIdx.x & 31;
  const size_t row = (size_t)t * 32 + lane;
  float b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f;
  int w = 0;
  for (; w + 3 < O.n_win; w += 4) {
    b0 += __ldcg(P.slot_base + (size_t)w * P.slot_stride + row);
    b1 += __ldcg(P.slot_base + (size_t)(w + 1) * P.slot_stride + row);
    b2 += __ldcg(P.slot_base + (size_t)(w + 2) * P.slot_stride + row);
    b3 += __ldcg(P.slot_base + (size_t)(w + 3) * P.slot_stride + row);
  }
  for (; w < O.n_win; ++w) b0 += __ldcg(P.slot_base + (size_t)w * P.slot_stride + row);
  return (b0 + b1) + (b2 + b3);
}

// y of op tile t (layer li) at the final plane count; valid = row exists.
__device__ __forceinline__ float tile_y(const Prog& P, const Op& O, const Work& W, const Smem& sm, int t,
                                        int& li, int& r, bool& valid) {
  const int lane = threadIdx.x & 31;
  li = layer_of(O, t);
  const Layer& L = O.L[li];
  const int fin = W.fin[li];
  const float S = tile_S(P, O, t);
  r = (t - L.tile_off) * 32 + lane;
  valid = r < L.rows;
  if (!valid) return 0.f;
  const float lo = __ldg(L.lo + r), span = __ldg(L.span + r);
  return sm.scale * (lo * sm.sx + ldexpf(span, -fin) * (S + 0.5f * sm.sx));
}

__device__ __noinline__ void reduce_unit(const Prog& P, const ECtl& C, const Op& O, const Work& W, const Smem& sm, int u) {
  if (O.pair) {
    const int half = O.L[0].n_tiles;
    int li, r, li2, r2;
    bool ok, ok2;
    const float up = tile_y(P, O, W, sm, u, li, r, ok);
    const float gt = tile_y(P, O, W, sm, u + half, li2, r2, ok2);
    const float hv = ok ? up * (gt / (1.0f + expf(-gt))) : 0.f;   // runtime.py:368
    if (ok) O.out[r] = hv;
    if (O.out_inst >= 0) emit_tile(P, C, O.out_inst, u, hv);
  } else {
    int li, r;
    bool ok;
    const float y = tile_y(P, O, W, sm, u, li, r, ok);
    const int o = O.L[li].out_off + r;
    float v = 0.f;
    if (O.add) {
      if (ok) {
        v = __ldcg(O.out + o) + y;                                   // runtime.py:364, 370
        O.out[o] = v;
      }
    } else if (ok) {
      O.out[o] = y;
    }
    if (O.out_inst >= 0) emit_tile(P, C, O.out_inst, (O.L[li].out_off >> 5) + (u - O.L[li].tile_off), v);
  }
}

// Contributions a tile (or pair) receives: one per window.
__device__ __forceinline__ unsigned unit_target(const Op& O, const Work& W, int u) {
  return (unsigned)O.n_win * (O.pair ? 2u : 1u);
}

// ---------------------------------------------------------------------------
// The op stage
// ---------------------------------------------------------------------------
__device__ __forceinline__ int my_groups(const Work& W, int warp) {
  const int n = W.gb - W.ga;
  return n > warp ? (n - warp + NW - 1) / NW : 0;
}

// Append the items of one pass (0: planes [0, nb), 1: planes [nb, fin)) of
// this warp's groups to its shared-memory item list; returns the new length.
// Lane k < mine handles group k (prefix sums by shuffles).
__device__ __forceinline__ int list_pass(const Op& O, const Work& W, Smem& sm, int warp, int mine, int pass,
                                         int n0, int w_first) {
  const int lane = threadIdx.x & 31;
  int cnt = 0, p0 = 0, g = 0, li = 0;
  if (lane < mine) {
    g = W.ga + warp + NW * lane;
    li = layer_of(O, g % O.n_tiles);
    p0 = pass ? W.nb[li] : 0;
    cnt = (pass ? W.fin[li] : W.nb[li]) - p0;
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (lane < mine) {
    const int w = g / O.n_tiles;
    const unsigned lb = (w != w_first) ? 1u : 0u;
    for (int q = 0; q < cnt; ++q) {
      const int idx = n0 + incl - cnt + q;
      sm.ia[warp][idx] = group_plane(O, g, p0 + q);
      sm.im[warp][idx] = (unsigned)lane | (unsigned)(p0 + q) << 8 | (unsigned)pass << 12 |
                         (unsigned)(q + 1 == cnt) << 13 | lb << 14;
    }
  }
  __syncwarp();
  return n0 + total;
}

// Reduction duty of this warp: units u = cta * NW + warp (+ G * NW ...);
// wait until all window contributions arrived, then reduce (fixed order).
__device__ __noinline__ void reduce_duty(const Prog& P, const ECtl& C, const Op& O, const Work& W, const Smem& sm,
                                          int cta, int G) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_units = O.pair ? O.L[0].n_tiles : O.n_tiles;
  for (int u = cta * NW + warp; u < n_units; u += G * NW) {
    const unsigned target = unit_target(O, W, u);
    if (lane == 0) {
      const unsigned* c = P.tile_cnt + u;
      unsigned v;
      const unsigned long long t0 = gclock();
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        if (v >= target) break;
        if (gclock() - t0 > 4000000000ull) hang("tile contributions", u, (long long)v);
      }
      P.tile_cnt[u] = 0u;
    }
    __syncwarp();
    __threadfence();
    reduce_unit(P, C, O, W, sm, u);
  }
}

__device__ __noinline__ void op_stage(const Prog& P, const ECtl& C, const Op& O, Work& W, const Op* On, Work* Wn,
                                         Smem& sm, int cta, int G, unsigned long long wait_target, bool do_wait,
                                         unsigned long long* stamp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cur = C.n_steps_done & 1;
  // ---- base work (decision independent) and first loads, before the barrier
  if (!W.valid) {
    if (warp == 0) build_work_warp(O, C, cta, G, W);
    __syncthreads();
  }
  const int mine = my_groups(W, warp);
  if (mine > kMaxGroups) __trap();        // host sizing guarantees this cannot happen
  const int w_first = W.ga < W.gb ? W.ga / O.n_tiles : 0;
  const int w_last = W.ga < W.gb ? (W.gb - 1) / O.n_tiles : -1;
  int n_items = list_pass(O, W, sm, warp, mine, 0, 0, w_first);   // base planes: decision independent
  // register ring: slot d holds item i + d while item i is consumed (named
  // registers only, so nothing is ever addressed through local memory)
  uint4 a0, a1, a2, a3, b0, b1, b2, b3, c0, c1, c2, c3, e0, e1, e2, e3;
#define ENG_LD(X, IDX)                                    \
  {                                                       \
    const uint4* a_ = sm.ia[warp][IDX] + lane;            \
    X##0 = ld_nc(a_); X##1 = ld_nc(a_ + 32);              \
    X##2 = ld_nc(a_ + 64); X##3 = ld_nc(a_ + 96);         \
  }
  if (0 < n_items) ENG_LD(a, 0)
  if (1 < n_items) ENG_LD(b, 1)
  if (2 < n_items) ENG_LD(c, 2)
  if (3 < n_items) ENG_LD(e, 3)
  const int n_pre = min(n_items, DEPTH);
  if (do_wait) bar_wait(P, wait_target);
  if (stamp && tid == 0) stamp[0] = gclock();

  // ---- prologue: decisions (runtime.py:184-193), input statistics, x windows
  if (warp < O.n_layers) {
    const int li = warp;
    const Layer& L = O.L[li];
    int bit = W.nb[li];
    double est = CUDART_NAN;
    const bool estimating = C.mode == MODE_DYNAMIC && L.sentinel == 0 && L.est != EST_NONE;
    if (estimating) {
      const int slot = (L.src == SRC_PREV_STEP && C.has_prev) ? 2 + C.prev_r : cur;
      const long long* acc = P.acc + (size_t)slot * P.acc_stride + L.acc;
      double q = 0.0;
      for (int kk = lane; kk < L.k; kk += 32) {
        const double g = (double)__ldcg(acc + kk) * L.fbscale;
        q += g * g;
      }
      q = wsum(q);
      const double sq = (double)__ldcg(acc + L.k) * (1.0 / kFxSq);
      const double sc = O.rms ? rsqrt_d(sq / (double)O.cols + (double)P.eps) : 1.0;
      if (L.est == EST_PROJECTION) est = q > 0.0 ? sc * q * rsqrt_d(q) : 0.0;
      else est = L.slope * (sq > 0.0 ? sc * sq * rsqrt_d(sq) : 0.0) + L.intercept;
      if (!C.force) bit = est > L.T ? L.h : L.l;                       // strict > (runtime.py:192)
    }
    if (lane == 0) {
      W.fin[li] = bit;
      if (C.mode == MODE_DYNAMIC && cta == 0 && L.trace >= 0 && P.n_trace > 0 && C.trace_step < P.max_steps) {
        const size_t o = (size_t)C.trace_step * P.n_trace + L.trace;
        P.tr_bits[o] = (signed char)bit;
        P.tr_est[o] = estimating ? (float)est : CUDART_NAN_F;
      }
    }
  } else if (warp == kMaxOpLayers) {
    if (lane == 0) {
      const long long* vs = P.vstat + ((size_t)cur * P.n_inst + O.in_inst) * 2;
      const double s1 = (double)__ldcg(vs) * (1.0 / kFxSum);
      const double s2 = (double)__ldcg(vs + 1) * (1.0 / kFxSq);
      sm.sx = (float)s1;
      sm.scale = O.rms ? (float)rsqrt_d(s2 / (double)O.cols + (double)P.eps) : 1.f;
    }
  } else if (warp == kMaxOpLayers + 1 && On && !Wn->valid) {
    build_work_warp(*On, C, cta, G, *Wn);
  }
  // input windows of this CTA (at most two) -> LUT A / B
  if (w_last > w_first + 1) __trap();     // host sizing guarantees at most two windows per CTA
  for (int q = tid; q < 2 * kWinCols; q += NT) {
    const int which = q / kWinCols, w = w_first + which;
    const int col = w * kWinCols + (q - which * kWinCols);
    sm.xw[which][q - which * kWinCols] = (w <= w_last && col < O.cols) ? __ldcg(O.in + col) : 0.f;
  }
  __syncthreads();
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(&sm);
  build_lut(reinterpret_cast<float*>(reinterpret_cast<char*>(&sm) + (kLutA - sbase)), sm.xw[0]);
  if (w_last > w_first)
    build_lut(reinterpret_cast<float*>(reinterpret_cast<char*>(&sm) + (kLutB - sbase)), sm.xw[1]);
  // zero row 256 of each LUT (= row 0 of LUT B for LUT A)
  if (tid < 64) {
    reinterpret_cast<float*>(reinterpret_cast<char*>(&sm) + (kLutB + 256 * 256 - sbase))[tid] = 0.f;
    if (w_last == w_first) reinterpret_cast<float*>(reinterpret_cast<char*>(&sm) + (kLutB - sbase))[tid] = 0.f;
  }
  __syncthreads();
  if (stamp && tid == 0) stamp[1] = gclock();
  // extra planes of groups whose layer decided high; refill the ring to DEPTH
  n_items = list_pass(O, W, sm, warp, mine, 1, n_items, w_first);
  if (0 >= n_pre && 0 < n_items) ENG_LD(a, 0)
  if (1 >= n_pre && 1 < n_items) ENG_LD(b, 1)
  if (2 >= n_pre && 2 < n_items) ENG_LD(c, 2)
  if (3 >= n_pre && 3 < n_items) ENG_LD(e, 3)
  // ---- stream: item i lives in slot i % 4 (a, b, c, e); after use the slot
  // is refilled with item i + 4. Unrolled by 4 so every slot index is static.
  float S = 0.f;
  auto post = [&](int i, float Pv) {
    const unsigned m = sm.im[warp][i];
    const int k = m & 0xff, p = (m >> 8) & 0xf, pass = (m >> 12) & 1;
    const int g = W.ga + warp + NW * k;
    const int w = g / O.n_tiles, t = g - w * O.n_tiles;
    const int li = layer_of(O, t);
    if (pass == 1 && p == W.nb[li]) S = sm.sbuf[warp][k][lane];
    S = 2.f * S + Pv;                                    // Horner over planes
    if ((m >> 13) & 1u) {                                // end of this group's pass
      if (pass == 0 && W.fin[li] > W.nb[li]) sm.sbuf[warp][k][lane] = S;      // park the base part
      else P.slot_base[(size_t)w * P.slot_stride + (size_t)t * 32 + lane] = S;
      S = 0.f;
    }
  };
#define ENG_STEP(X, J)                                                                    \
  if ((J) < n_items) {                                                                    \
    const unsigned m_ = sm.im[warp][J];                                                   \
    const uint32_t lr_ = ((m_ >> 14) & 1u ? kLutB : kLutA) | ((uint32_t)lane * 4u);       \
    const float Pv_ = plane_sum(X##0, X##1, X##2, X##3, lr_);                             \
    if ((J) + 4 < n_items) ENG_LD(X, (J) + 4)                                             \
    post((J), Pv_);                                                                       \
  }
  for (int i = 0; i < n_items; i += 4) {
    ENG_STEP(a, i)
    ENG_STEP(b, i + 1)
    ENG_STEP(c, i + 2)
    ENG_STEP(e, i + 3)
  }
#undef ENG_STEP
#undef ENG_LD
  if (stamp && tid == 0) stamp[5] = gclock();
  if (On) prefetch_work_l2(*On, *Wn);
  if (warp == NW - 1) prefetch_feeds_l2(P, C, O.out_inst, O.n_tiles * 32, cta, G);
  // ---- publish: one fence per warp, then one arrival per owned group
  __threadfence();
  __syncwarp();
  for (int k = lane; k < mine; k += 32) {
    const int g = W.ga + warp + NW * k;
    const int t = g % O.n_tiles;
    atomicAdd(P.tile_cnt + (O.pair ? (t % O.L[0].n_tiles) : t), 1u);
  }
  reduce_duty(P, C, O, W, sm, cta, G);
  if (stamp && tid == 0) stamp[6] = gclock();
  __syncthreads();
  if (tid == 0) W.valid = 0;
}

// ---------------------------------------------------------------------------
// Attention stage (runtime.py:351-362): RoPE, KV append, causal softmax.
// Unit = (kv head g, position chunk); a unit serves the H/KV query heads of
// its group with an online softmax over 32-position sub-chunks; chunk
// partials are merged by the last unit of the group.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float rope_at(const float* v, int i, int hd, const float* c, const float* s) {
  const int half = hd / 2;
  if (i < half) return __ldcg(v + i) * c[i] - __ldcg(v + i + half) * s[i];
  if (i < 2 * half) return __ldcg(v + i - half) * s[i - half] + __ldcg(v + i) * c[i - half];
  return __ldcg(v + i);
}

__device__ __noinline__ void attn_emit_head(const Prog& P, const ECtl& C, int inst, int h) {
  // emit the hd/32 tiles of head h (warps of this CTA), values already in P.attn
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nt = (P.hd + 31) / 32;
  for (int tt = warp; tt < nt; tt += NW) {
    const int i = tt * 32 + lane;
    const float v = i < P.hd ? __ldcg(P.attn + h * P.hd + i) : 0.f;
    emit_tile(P, C, inst, (h * P.hd) / 32 + tt, v);
  }
}

__device__ __noinline__ void attn_stage(const Prog& P, const ECtl& C, int b, float* sh, int cta, int G, int* s_last) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = C.pos, n = t + 1;
  const int hd = P.hd, KV = P.KV, qh = P.H / P.KV, half = hd / 2;
  int nch = min((n + 15) / 16, max(1, G / KV));
  nch = min(nch, P.attn_max_chunks);
  const int clen = (n + nch - 1) / nch;
  nch = (n + clen - 1) / clen;
  const int units = KV * nch;
  const float scale = 1.0f / sqrtf((float)hd);
  const float* cs = P.cosv + (size_t)t * half;
  const float* sn = P.sinv + (size_t)t * half;
  float* kc = P.kc[b];
  float* vc = P.vc[b];
  // smem: q[qh][hd] kt[hd] vt[hd] K[32][hd] V[32][hd] sc[qh][32] o[qh][hd] m[qh] l[qh] al[qh]
  float* q = sh;
  float* kt = q + qh * hd;
  float* vt = kt + hd;
  float* Ks = vt + hd;
  float* Vs = Ks + 32 * hd;
  float* sc = Vs + 32 * hd;
  float* o = sc + qh * 32;
  float* mm = o + qh * hd;
  float* ll = mm + qh;
  float* al = ll + qh;
  const int inst = 4 * b + 1;
  for (int u = cta; u < units; u += G) {
    const int g = u / nch, ch = u % nch;
    const int s0 = ch * clen, s1 = min(n, s0 + clen);
    __syncthreads();
    for (int idx = tid; idx < qh * hd; idx += NT) {
      const int hq = idx / hd, i = idx - hq * hd;
      q[idx] = rope_at(P.qkv + (g * qh + hq) * hd, i, hd, cs, sn);
      o[idx] = 0.f;
    }
    for (int i = tid; i < hd; i += NT) {
      kt[i] = rope_at(P.qkv + P.d + g * hd, i, hd, cs, sn);
      vt[i] = __ldcg(P.qkv + P.d + P.dkv + g * hd + i);
    }
    if (tid < qh) { mm[tid] = -CUDART_INF_F; ll[tid] = 0.f; }
    __syncthreads();
    if (s1 == n) {       // the unit holding position t appends it to the cache (runtime.py:355-356)
      for (int i = tid; i < hd; i += NT) {
        kc[(size_t)t * P.dkv + g * hd + i] = kt[i];
        vc[(size_t)t * P.dkv + g * hd + i] = vt[i];
      }
    }
    for (int sb = s0; sb < s1; sb += 32) {
      const int ns = min(32, s1 - sb);
      for (int idx = tid; idx < ns * hd; idx += NT) {
        const int sp = idx / hd, i = idx - sp * hd;
        const int s = sb + sp;
        if (s == t) { Ks[idx] = kt[i]; Vs[idx] = vt[i]; }
        else {
          Ks[idx] = __ldcg(kc + (size_t)s * P.dkv + g * hd + i);
          Vs[idx] = __ldcg(vc + (size_t)s * P.dkv + g * hd + i);
        }
      }
      __syncthreads();
      for (int pr = warp; pr < qh * ns; pr += NW) {
        const int hq = pr / ns, sp = pr - hq * ns;
        float a = 0.f;
        for (int i = lane; i < hd; i += 32) a += q[hq * hd + i] * Ks[sp * hd + i];
        a = wsum(a);
        if (lane == 0) sc[hq * 32 + sp] = a * scale;
      }
      __syncthreads();
      if (warp < qh) {
        const int hq = warp;
        const float v = lane < ns ? sc[hq * 32 + lane] : -CUDART_INF_F;
        float mx = v;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        const float mnew = fmaxf(mm[hq], mx);
        const float p = lane < ns ? expf(v - mnew) : 0.f;
        const float ps = wsum(p);
        if (lane < ns) sc[hq * 32 + lane] = p;
        if (lane == 0) {
          const float a = expf(mm[hq] - mnew);
          al[hq] = a;
          ll[hq] = ll[hq] * a + ps;
          mm[hq] = mnew;
        }
      }
      __syncthreads();
      for (int idx = tid; idx < qh * hd; idx += NT) {
        const int hq = idx / hd, i = idx - hq * hd;
        float acc = o[idx] * al[hq];
        for (int sp = 0; sp < ns; ++sp) acc += sc[hq * 32 + sp] * Vs[sp * hd + i];
        o[idx] = acc;
      }
      __syncthreads();
    }
    if (nch == 1) {
      for (int idx = tid; idx < qh * hd; idx += NT) {
        const int hq = idx / hd;
        P.attn[g * qh * hd + idx] = o[idx] / ll[hq];
      }
      __syncthreads();
      if (P.attn_emit) for (int hq = 0; hq < qh; ++hq) attn_emit_head(P, C, inst, g * qh + hq);
      continue;
    }
    for (int idx = tid; idx < qh * hd; idx += NT) {
      const int hq = idx / hd, i = idx - hq * hd;
      P.attn_part[((size_t)(g * qh + hq) * P.attn_max_chunks + ch) * (hd + 2) + i] = o[idx];
    }
    if (tid < qh) {
      float* pp = P.attn_part + ((size_t)(g * qh + tid) * P.attn_max_chunks + ch) * (hd + 2);
      pp[hd] = mm[tid];
      pp[hd + 1] = ll[tid];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) *s_last = atomicAdd(P.attn_cnt + g, 1u) == (unsigned)nch - 1;
    __syncthreads();
    if (!*s_last) continue;
    __threadfence();
    for (int idx = tid; idx < qh * hd; idx += NT) {
      const int hq = idx / hd, i = idx - hq * hd;
      const float* base = P.attn_part + (size_t)(g * qh + hq) * P.attn_max_chunks * (hd + 2);
      float M = -CUDART_INF_F;
      for (int c = 0; c < nch; ++c) M = fmaxf(M, __ldcg(base + c * (hd + 2) + hd));
      float Ls = 0.f, acc = 0.f;
      for (int c = 0; c < nch; ++c) {
        const float e = expf(__ldcg(base + c * (hd + 2) + hd) - M);
        Ls += __ldcg(base + c * (hd + 2) + hd + 1) * e;
        acc += __ldcg(base + c * (hd + 2) + i) * e;
      }
      P.attn[g * qh * hd + idx] = acc / Ls;
    }
    if (tid == 0) P.attn_cnt[g] = 0u;
    __syncthreads();
    if (P.attn_emit) for (int hq = 0; hq < qh; ++hq) attn_emit_head(P, C, inst, g * qh + hq);
  }
}

// EMIT: statistics + feeds of a whole vector (attention output when heads
// are not 32-aligned).
__device__ __noinline__ void emit_stage(const Prog& P, const ECtl& C, const float* v, int n, int inst, int cta, int G) {
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
__device__ __noinline__ void head_stage(const Prog& P, const ECtl& C, Smem& sm, int cta, int G) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cur = C.n_steps_done & 1;
  const int fin_inst = 4 * P.n_blocks;
  const double s2 = (double)__ldcg(P.vstat + ((size_t)cur * P.n_inst + fin_inst) * 2 + 1) * (1.0 / kFxSq);
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
  __syncthreads();
  if (tid == 0) sm.last = atomicAdd(P.head_cnt, 1u) == (unsigned)G - 1;
  __syncthreads();
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
  __syncthreads();
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
__device__ __noinline__ void begin_stage(const Prog& P, const ECtl& C, int cta, int G) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nxt = (C.n_steps_done + 1) & 1;
  {
    long long* a = P.acc + (size_t)nxt * P.acc_stride;
    long long* z = P.acc + (size_t)(2 + C.prev_z) * P.acc_stride;
    long long* vs = P.vstat + (size_t)nxt * P.n_inst * 2;
    for (int i = cta * NT + tid; i < P.acc_stride; i += G * NT) { a[i] = 0; z[i] = 0; }
    for (int i = cta * NT + tid; i < P.n_inst * 2; i += G * NT) vs[i] = 0;
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
extern "C" __global__ void __launch_bounds__(NT, 1) engine_kernel(const Prog Pk, int n_steps) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  if (threadIdx.x == 0) sm.prog = Pk;
  __syncthreads();
  const Prog& P = sm.prog;
  float* lut = reinterpret_cast<float*>(smem_raw + (kLutA - sbase));
  __shared__ int s_last;
  const int cta = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
  if (tid == 0) { sm.work[0].valid = 0; sm.work[1].valid = 0; }
  int wi = 0;
  // barrier epochs continue from previous launches (counter = G x stages so far)
  const unsigned long long e0 = ld_acq64(P.bar) / (unsigned long long)G;   // stages completed before
  unsigned long long k = 0;     // stages completed in this launch
  ECtl& C = sm.ctl;
  __syncthreads();
  for (int step = 0; step < n_steps; ++step) {
    for (int si = 0; si < P.n_stages; ++si) {
      const int2 st = P.stages[si];
      const bool wait = k > 0;
      const unsigned long long target = e0 + k;        // epoch of the previous stage
      if (st.x == ST_OP) {
        // next op stage of this step (ring run-ahead target)
        int nsi = si + 1;
        while (nsi < P.n_stages && P.stages[nsi].x != ST_OP) ++nsi;
        const bool has_next = nsi < P.n_stages;
        // descriptors to shared memory (the current one may already be there)
        {
          const int nw4 = (int)(sizeof(Op) / 16);
          const int4* src = reinterpret_cast<const int4*>(P.ops + st.y);
          int4* dst = reinterpret_cast<int4*>(&sm.op[wi]);
          if (!sm.work[wi].valid)
            for (int q = tid; q < nw4; q += NT) dst[q] = __ldg(src + q);
          if (has_next) {
            const int4* src2 = reinterpret_cast<const int4*>(P.ops + P.stages[nsi].y);
            int4* dst2 = reinterpret_cast<int4*>(&sm.op[wi ^ 1]);
            for (int q = tid; q < nw4; q += NT) dst2[q] = __ldg(src2 + q);
          }
          __syncthreads();
        }
        op_stage(P, C, sm.op[wi], sm.work[wi], has_next ? &sm.op[wi ^ 1] : nullptr, &sm.work[wi ^ 1], sm, cta, G,
                 target, wait, P.dbg ? P.dbg + ((size_t)si * G + cta) * 8 : nullptr);
        wi ^= 1;
      } else {
        if (wait) bar_wait(P, target);
        if (P.dbg && tid == 0) P.dbg[((size_t)si * G + cta) * 8] = gclock();
        if (st.x == ST_BEGIN) {
          read_ctl(P, C);
          begin_stage(P, C, cta, G);
        } else if (st.x == ST_ATTN) {
          attn_stage(P, C, st.y, lut, cta, G, &s_last);
        } else if (st.x == ST_EMIT) {
          emit_stage(P, C, P.attn, P.d, 4 * st.y + 1, cta, G);
        } else {
          head_stage(P, C, sm, cta, G);
        }
      }
      if (P.dbg && tid == 0) P.dbg[((size_t)si * G + cta) * 8 + 7] = gclock();
      bar_arrive(P, e0 + k + 1, G);
      ++k;
    }
  }
}
}  // namespace eng
}  // namespace dpq
