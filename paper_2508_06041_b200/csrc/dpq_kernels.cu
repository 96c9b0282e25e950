// sm_100a kernels for the DP-LLM decode hot path.
//
//  op_kernel        fused precision selector + any-precision bitplane GEMV for
//                   1..3 layers sharing an input vector (q|k|v, up|gate, o,
//                   down). Replaces reference select_precision
//                   (runtime.py:184-193), the estimators (estimator.py:35-73)
//                   and dequantize()@x (quant.py:67-99, runtime.py:348-369).
//  finalize_dual    exact / track_exact epilogue (estimator.py:30-32, 63-73).
//  attention_kernel RoPE + KV append + causal softmax attention for one token
//                   (runtime.py:351-362), split over 64-position chunks.
//  lmhead_kernel    final RMSNorm + lm_head logits + greedy argmax + end-of-step
//                   control (runtime.py:372-380, 405-408).
//  begin_kernel     embedding row (runtime.py:345).
//  repack / quantize / dequant kernels for the store (quant.py:43-80).
#include "dpq_common.cuh"
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <math_constants.h>
#include <cstdio>

namespace dpq {

// ---------------------------------------------------------------------------
// small PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Spin-wait watchdog: a wait that exceeds 2 s reports where it stalled and
// traps, turning a would-be hang into a launch error.
__device__ __noinline__ void dpq_hang(const char* what, int a, int b, unsigned v) {
  printf("dpq watchdog: %s stalled (block %d thread %d, arg %d/%d, value %u)\n", what, blockIdx.x, threadIdx.x,
         a, b, v);
  __trap();
}
#define DPQ_SPIN_UNTIL(cond, what, a, b, v)                                   \
  do {                                                                        \
    const unsigned long long t0_ = gtimer();                                  \
    while (!(cond)) {                                                         \
      __nanosleep(20);                                                        \
      if (gtimer() - t0_ > 2000000000ull) dpq_hang(what, (a), (b), (v));      \
    }                                                                         \
  } while (0)
#define DPQ_STAMP(i) \
  do { if (D.dbg && threadIdx.x == 0) D.dbg[X.cta * 8 + (i)] = gtimer(); } while (0)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide double sum (all threads get the result). red: >= 32 doubles smem.
__device__ double block_sum_d(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += red[i];   // fixed order: deterministic
  __syncthreads();
  return t;
}

// Three block-wide double sums with one barrier round (all threads get them).
__device__ void block_sum3(double& a, double& b, double& c, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  a = warp_sum(a); b = warp_sum(b); c = warp_sum(c);
  __syncthreads();
  if (lane == 0) { red[warp] = a; red[32 + warp] = b; red[64 + warp] = c; }
  __syncthreads();
  double ta = 0.0, tb = 0.0, tc = 0.0;
  for (int i = 0; i < nw; ++i) { ta += red[i]; tb += red[32 + i]; tc += red[64 + i]; }
  a = ta; b = tb; c = tc;
}

// Dot of one 512-column G row slice (window) with xin[512] (smem), one warp,
// vector loads: f32 4x float4 / f16 2x 8 halves / e4m3 1x 16 bytes per lane.
__device__ __forceinline__ float g_dot(const void* Grow, int g_dtype, const float* xin, int lane) {
  float acc = 0.f;
  if (g_dtype == G_F16) {
    const uint4* g = reinterpret_cast<const uint4*>(Grow);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint4 v = __ldg(g + j * 32 + lane);
      const int c0 = (j * 32 + lane) * 8;
      const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __half22float2(h[q]);
        acc += f.x * xin[c0 + 2 * q] + f.y * xin[c0 + 2 * q + 1];
      }
    }
  } else if (g_dtype == G_E4M3) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(Grow) + lane);
    const unsigned char* b = reinterpret_cast<const unsigned char*>(&v);
    const int c0 = lane * 16;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      __nv_fp8_e4m3 e;
      e.__x = b[q];
      acc += float(e) * xin[c0 + q];
    }
  } else {
    const float4* g = reinterpret_cast<const float4*>(Grow);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 v = __ldg(g + j * 32 + lane);
      const int c0 = (j * 32 + lane) * 4;
      acc += v.x * xin[c0] + v.y * xin[c0 + 1] + v.z * xin[c0 + 2] + v.w * xin[c0 + 3];
    }
  }
  return warp_sum(acc);
}

__device__ __forceinline__ long long g_row_bytes(int g_dtype) {
  return g_dtype == G_F16 ? 2 * kWinCols : (g_dtype == G_E4M3 ? kWinCols : 4 * kWinCols);
}

__device__ __forceinline__ float load_g(const void* G, int g_dtype, long long idx) {
  if (g_dtype == G_F16) return __half2float(reinterpret_cast<const __half*>(G)[idx]);
  if (g_dtype == G_E4M3) {
    __nv_fp8_e4m3 v;
    v.__x = reinterpret_cast<const unsigned char*>(G)[idx];
    return float(v);
  }
  return reinterpret_cast<const float*>(G)[idx];
}

// ---------------------------------------------------------------------------
// The hot loop: one (plane, window, 32-row tile) task for one warp.
// Lane l accumulates P_p[row l] = sum_{col in window} plane_p[row][col] * x[col]
// via 64 byte-LUT lookups; 3 SASS ops per 8 weight bits (PRMT, LDS, FADD).
// ---------------------------------------------------------------------------
// lut_addr(W, k) = shared address of LUT row (byte k of W), slot of this lane:
// 0x10000 | e<<8 | 4*lane  (LUT placed at shared address 0x10000, lanereg =
// 0x00010000 | 4*lane), so a single PRMT forms the whole address and the LDS
// adds the step offset 4*s as an immediate.
#define DPQ_LDS(dst, addr, IMM) \
  asm("ld.shared.f32 %0, [%1+%2];" : "=f"(dst) : "r"(addr), "n"(IMM))

__device__ __forceinline__ float plane_task(const uint4 d0, const uint4 d1, const uint4 d2,
                                            const uint4 d3, uint32_t lanereg) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#define DPQ_WORD(W, S0)                                              \
  {                                                                  \
    float v0, v1, v2, v3;                                            \
    DPQ_LDS(v0, __byte_perm((W), lanereg, 0x7604u), 4 * (S0 + 0));   \
    DPQ_LDS(v1, __byte_perm((W), lanereg, 0x7614u), 4 * (S0 + 1));   \
    DPQ_LDS(v2, __byte_perm((W), lanereg, 0x7624u), 4 * (S0 + 2));   \
    DPQ_LDS(v3, __byte_perm((W), lanereg, 0x7634u), 4 * (S0 + 3));   \
    a0 += v0; a1 += v1; a2 += v2; a3 += v3;                          \
  }
  DPQ_WORD(d0.x, 0) DPQ_WORD(d0.y, 4) DPQ_WORD(d0.z, 8) DPQ_WORD(d0.w, 12)
  DPQ_WORD(d1.x, 16) DPQ_WORD(d1.y, 20) DPQ_WORD(d1.z, 24) DPQ_WORD(d1.w, 28)
  DPQ_WORD(d2.x, 32) DPQ_WORD(d2.y, 36) DPQ_WORD(d2.z, 40) DPQ_WORD(d2.w, 44)
  DPQ_WORD(d3.x, 48) DPQ_WORD(d3.y, 52) DPQ_WORD(d3.z, 56) DPQ_WORD(d3.w, 60)
#undef DPQ_WORD
  return (a0 + a1) + (a2 + a3);
}

// Build the byte LUT of one window from x_win[512] (smem). 512 threads:
// thread -> group g = tid & 63, LUT rows [32*(tid>>6), +32).
__device__ __forceinline__ void build_lut(float* lut, const float* xw) {
  const int g = threadIdx.x & 63, rb = threadIdx.x >> 6;
  const float* xg = xw + 8 * g;
  float L[16];
  L[0] = 0.f;
#pragma unroll
  for (int n = 1; n < 16; ++n) {
    const int low = n & (-n);
    const int bit = __ffs(low) - 1;
    L[n] = L[n ^ low] + xg[bit];
  }
  float H[2];
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int m = 2 * rb + hh;
    float s = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (m & (1 << t)) s += xg[4 + t];
    H[hh] = s;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int e = 32 * rb + i;
    lut[e * kGroups + g] = L[i & 15] + H[i >> 4];
  }
  if (rb == 0) lut[256 * kGroups + g] = 0.f;
}

// ---------------------------------------------------------------------------
// op kernel
// ---------------------------------------------------------------------------
struct OpSmem {
  float xw[kWinCols];        // current input window (pre-scale)
  float xp[kWinCols];        // estimator input window when it is not xw
  double red[96];
  int rank;                  // arrival rank of this CTA in its window
  int la[kMaxOpLayers];      // planes streamed before a decision
  int lb[kMaxOpLayers];      // final plane count (-1 = pending decision)
  int is_last;
  unsigned my_gen;
  double xp_scale;           // scale turning xp into the estimator input
  const float* xp_src;       // source vector of xp (nullptr: estimator uses xw)
};

constexpr int kWarpTiles = 8;                 // owned tiles per warp per chunk
constexpr uint32_t kLutShared = 0x10000;     // shared address of the LUT
constexpr int kOpSmemBytes = (int)((sizeof(OpSmem) + 127) / 128 * 128);

// Planes streamed before any decision is known, and the final plane count.
__device__ __forceinline__ void layer_planes(const OpLayer& Ly, int mode, const Control* ctl,
                                             int& a, int& b, int& pending) {
  const DevSel& S = Ly.S;
  pending = 0;
  if (mode == MODE_PREFILL) { a = b = S.prefill_bit; return; }
  if (Ly.dual) { a = b = S.h; return; }                  // both l and h produced
  if (ctl->force && Ly.trace_idx >= 0) { a = b = ctl->forced_bits[Ly.trace_idx]; return; }
  if (S.sentinel == 1) { a = b = S.l; return; }
  if (S.sentinel == 2) { a = b = S.h; return; }
  if (S.sentinel == 3) { a = b = -1; pending = 2; return; }   // bit from decision[] (prior kernel)
  a = S.l; b = S.h; pending = 1;
}

// Per-call context of a fused op: which CTA of how many, readiness flags of
// the producers of the input (persistent step kernel) and of our outputs.
struct StageCtx {
  int cta, G;
  unsigned epoch;
  const unsigned* dep0;     // producer flags covering the input (nullptr: none)
  int dep0_off, dep0_rpf;   // flag index = off + column / rows_per_flag
  const unsigned* dep1;     // second producer (IN_SILU gate half)
  int dep1_off;
  unsigned* out_flags;      // per output tile, set to epoch by the tile reducer
  const OpDesc* next;       // next op: its always-planes are prefetched to L2
};

// Wait until flags f[i0, i1) all equal epoch. Call with a full warp: the
// flags are polled lane-parallel (one L2 round trip per poll, not per flag).
__device__ __forceinline__ void wait_flags_warp(const unsigned* f, int i0, int i1, unsigned epoch) {
  const int lane = threadIdx.x & 31;
  for (int base = i0; base < i1; base += 32) {
    const int i = base + lane;
    const unsigned long long t0 = gtimer();
    while (!__all_sync(0xffffffffu, i >= i1 || ld_acquire(f + i) == epoch)) {
      __nanosleep(20);
      if (gtimer() - t0 > 2000000000ull) dpq_hang("readiness flags", i0, i1, epoch);
    }
  }
}

__device__ __forceinline__ void cta_window(const OpDesc& D, int cta, int G, int& w, int& j, int& m,
                                           int& t_begin, int& t_end) {
  w = cta % D.n_win;
  j = cta / D.n_win;
  m = (G - w + D.n_win - 1) / D.n_win;
  t_begin = (int)((long long)D.total_tiles * j / m);
  t_end = (int)((long long)D.total_tiles * (j + 1) / m);
}

// L2 prefetch of the always-streamed planes of this CTA's share of op D.
__device__ void prefetch_op(const OpDesc& D, const Control* ctl, int cta, int G) {
  if (cta >= G) return;
  int w, j, m, t_begin, t_end;
  cta_window(D, cta, G, w, j, m, t_begin, t_end);
  const int mode = ctl->mode;
  for (int li = 0; li < D.n_layers; ++li) {
    const OpLayer& Ly = D.layer[li];
    int a, b, pend;
    layer_planes(Ly, mode, ctl, a, b, pend);
    if (a <= 0) continue;
    const int lt0 = max(t_begin, Ly.tile_off), lt1 = min(t_end, Ly.tile_off + Ly.L.n_tiles);
    if (lt0 >= lt1) continue;
    for (int p = 0; p < a; ++p) {
      const char* base = reinterpret_cast<const char*>(
          Ly.L.planes + p * Ly.L.plane_stride16 +
          ((long long)w * Ly.L.n_tiles + (lt0 - Ly.tile_off)) * (kTileBytes / 16));
      long long bytes = (long long)(lt1 - lt0) * kTileBytes;
      while (bytes > 0) {
        const unsigned chunk = (unsigned)min(bytes, (long long)65536);
        prefetch_l2_bulk(base, chunk);
        base += chunk;
        bytes -= chunk;
      }
    }
  }
}

constexpr int kGShares = 2;      // CTAs per window computing estimator partials
constexpr int kChunk = 2;        // tiles a warp grabs at a time

// Estimator input of an op (runtime.py:300-309): explicit est_in, the
// previous-step / previous-block snapshot, or nullptr (= the op input).
__device__ __forceinline__ const float* est_input(const OpDesc& D, const Control* ctl, int mode, double& scale) {
  scale = 1.0;
  if (D.est_in) return D.est_in;
  if (mode != MODE_DYNAMIC) return nullptr;
  int need = 0;
  for (int li = 0; li < D.n_layers; ++li) {
    const DevSel& S = D.layer[li].S;
    if (S.prev_residual && S.sentinel == 0 && (S.est_kind == EST_LINEAR || S.est_kind == EST_PROJECTION)) need = 1;
  }
  if (!need) return nullptr;
  int slot = -1, idx = -1;
  if (ctl->async_prev_block) { slot = ctl->snap_w; idx = D.layer[0].snap_in; }
  else if (ctl->has_prev) { slot = ctl->snap_r; idx = D.snap_idx; }
  if (slot < 0 || idx < 0) return nullptr;
  const size_t loc = (size_t)slot * D.n_snap + idx;
  if (D.in_mode == IN_RMS) scale = (double)D.snap_stats[loc * 4 + 2];
  return D.snap + loc * D.snap_stride;
}

// G tile CTAs + the decider finish an op; the last resets the op's counters
// and accumulators for its next execution (nobody can still be using them).
__device__ __forceinline__ void op_done(const OpDesc& D, int G) {
  __threadfence();
  if (atomicAdd(D.ctr + 1, 1u) == (unsigned)G) {
    for (int i = 0; i < 3 + D.n_win; ++i) D.ctr[i] = 0u;
    for (int i = 0; i < kMaxOpLayers * kMaxK; ++i) D.gxa[i] = 0;
    __threadfence();
  }
}

__device__ __forceinline__ int estimator_shares(int G, int n_win) {
  int total = 0;
  for (int ww = 0; ww < n_win; ++ww) total += min(kGShares, (G - ww + n_win - 1) / n_win);
  return total;
}

// Decider of an op, run by warp 0 of the dedicated decider CTA (it owns no
// tiles, so its latency never delays a tile): waits for the estimator shares,
// then op input statistics, estimates, decisions (runtime.py:184-193), trace,
// and the decision-ready release. All loads are issued before any use.
__device__ void decide_warp(const OpDesc& D, const Control* __restrict__ ctl, int G) {
  const int lane = threadIdx.x & 31;
  const int n_win = D.n_win;
  const int mode = ctl->mode;
  const unsigned total = (unsigned)estimator_shares(G, n_win);
  if (lane == 0) DPQ_SPIN_UNTIL(ld_acquire(D.ctr) >= total, "decider shares", (int)total, D.n_win, ld_acquire(D.ctr));
  __syncwarp();
  double xp_scale;
  const float* xp_src = est_input(D, ctl, mode, xp_scale);
  // loads: window stats (2 windows per lane) and projection accumulators
  double a1[2], a2[2], a3[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = lane + 32 * u;
    const bool ok = i < n_win;
    a1[u] = ok ? __ldcg(D.win_stats + 4 * i) : 0.0;
    a2[u] = ok ? __ldcg(D.win_stats + 4 * i + 1) : 0.0;
    a3[u] = ok ? __ldcg(D.win_stats + 4 * i + 2) : 0.0;
  }
  long long gv[kMaxOpLayers][kMaxK / 32];
#pragma unroll
  for (int li = 0; li < kMaxOpLayers; ++li)
#pragma unroll
    for (int u = 0; u < kMaxK / 32; ++u) {
      const int i = lane + 32 * u;
      const bool ok = mode == MODE_DYNAMIC && li < D.n_layers && D.layer[li].S.sentinel == 0 &&
                      D.layer[li].S.est_kind == EST_PROJECTION && i < D.layer[li].S.k;
      gv[li][u] = ok ? __ldcg(D.gxa + li * kMaxK + i) : 0;
    }
  const double t1 = warp_sum(a1[0] + a1[1]);
  const double t2 = warp_sum(a2[0] + a2[1]);
  const double t3 = warp_sum(a3[0] + a3[1]);
  const double inv = 1.0 / sqrt(t2 / (double)D.cols + (double)D.eps);
  const int force = ctl->force, trace_step = ctl->trace_step;
  if (lane == 0) {
    D.op_stats[0] = (float)t1;
    D.op_stats[1] = (float)t2;
    D.op_stats[2] = (float)inv;
    if (D.need_snap) {
      float* st = D.snap_stats + ((size_t)ctl->snap_w * D.n_snap + D.snap_idx) * 4;
      st[0] = (float)t1; st[1] = (float)t2; st[2] = (float)inv; st[3] = 0.f;
    }
  }
  if (mode == MODE_DYNAMIC) {
#pragma unroll
    for (int li = 0; li < kMaxOpLayers; ++li) {
      if (li >= D.n_layers) break;
      const OpLayer& Ly = D.layer[li];
      const DevSel& S = Ly.S;
      double est = CUDART_NAN;
      bool have_est = false;
      const bool prev = xp_src && (S.prev_residual || D.est_in);
      const double in_scale = prev ? xp_scale : (D.in_mode == IN_RMS ? inv : 1.0);
      if (S.sentinel == 0 && S.est_kind == EST_PROJECTION) {
        double q = 0.0;
#pragma unroll
        for (int u = 0; u < kMaxK / 32; ++u) {
          const int i = lane + 32 * u;
          double g = (double)gv[li][u] * 0x1p-40;
          if (S.g_scale && i < S.k) g *= (double)S.g_scale[i];
          q += g * g;
        }
        q = warp_sum(q);
        est = in_scale * sqrt(q);
        have_est = true;
      } else if (S.sentinel == 0 && S.est_kind == EST_LINEAR) {
        const double sq = prev ? t3 : t2;
        est = S.slope * (in_scale * sqrt(sq)) + S.intercept;
        have_est = true;
      }
      if (lane == 0) {
        int bit;
        if (S.sentinel == 3 || (Ly.dual && S.est_kind == EST_EXACT && S.sentinel == 0))
          bit = -1;                                   // finalize / prior kernel decides
        else if (force && Ly.trace_idx >= 0) bit = ctl->forced_bits[Ly.trace_idx];
        else if (S.sentinel == 1) bit = S.l;
        else if (S.sentinel == 2) bit = S.h;
        else if (have_est) bit = (est > S.T) ? S.h : S.l;
        else bit = S.l;
        if (bit >= 0) D.decision[li] = bit;
        if (Ly.trace_idx >= 0 && D.n_trace > 0) {
          const size_t o = (size_t)trace_step * D.n_trace + Ly.trace_idx;
          if (bit >= 0) D.tr_bits[o] = (signed char)bit;
          if (S.sentinel != 3) D.tr_est[o] = have_est ? (float)est : CUDART_NAN_F;
        }
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    st_release(D.ctr + 2, 1u);                // decision ready (reset when the op completes)
    op_done(D, G);
  }
}

__device__ __forceinline__ void op_stage(const OpDesc& D, const Control* __restrict__ ctl, const StageCtx& X,
                                         unsigned char* smem_raw) {
  // Shared layout: [sbase, 0x10000): OpSmem + per-warp S / S_l; [0x10000, +kLutBytes): LUT.
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
  float* lut = reinterpret_cast<float*>(smem_raw + (kLutShared - sbase));
  OpSmem& sm = *reinterpret_cast<OpSmem*>(smem_raw);
  if (kOpSmemBytes + 2 * kThreads * kWarpTiles * 4 > kLutShared - sbase) __trap();

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kW = kThreads / 32;
  const int G = X.G;
  const int n_win = D.n_win;
  const int mode = ctl->mode;
  // static window assignment: CTAs w, w + n_win, ... share window w
  int w, j, m, t_begin, t_end;
  cta_window(D, X.cta, G, w, j, m, t_begin, t_end);
  // op counters: [0] estimator shares done, [1] CTAs done, [2] decision ready, [3 + w] window arrivals
  unsigned* warr = D.ctr + 3;

  // ---- L2 prefetch of our static share of the planes, and of the next op --
  if (tid == 0) {
    prefetch_op(D, ctl, X.cta, G);
    if (X.next) prefetch_op(*X.next, ctl, X.cta, X.G);
  }
  DPQ_STAMP(0);
  pdl_wait();
  unsigned my_rank = 0;
  if (tid == 0) my_rank = atomicAdd(warr + w, 1u);   // arrival rank in the window (used below)
  if (warp == 0 && X.dep0) {
    const int c0 = w * kWinCols, c1 = min(D.cols, c0 + kWinCols);
    wait_flags_warp(X.dep0, X.dep0_off + c0 / X.dep0_rpf, X.dep0_off + (c1 + X.dep0_rpf - 1) / X.dep0_rpf,
                    X.epoch);
    if (X.dep1)
      wait_flags_warp(X.dep1, X.dep1_off + c0 / X.dep0_rpf, X.dep1_off + (c1 + X.dep0_rpf - 1) / X.dep0_rpf,
                      X.epoch);
  }
  DPQ_STAMP(1);

  // ---- estimator-input source ----------------------------------------------
  if (tid == 0) {
    sm.rank = (int)my_rank;
    double scale;
    sm.xp_src = est_input(D, ctl, mode, scale);
    sm.xp_scale = scale;
  }
  __syncthreads();

  // ---- prologue: input window (+ estimator-input window), stats, LUT -------
  const int col0 = w * kWinCols;
  double s1 = 0.0, s2 = 0.0, s3 = 0.0;
  {
    const int c = col0 + tid;
    float v = 0.f, vp = 0.f;
    if (c < D.cols) {
      if (D.in_mode == IN_SILU) {
        const float up = __ldcg(D.in0 + c), gt = __ldcg(D.in1 + c);
        v = up * (gt / (1.0f + expf(-gt)));
      } else {
        v = __ldcg(D.in0 + c);
      }
      if (sm.xp_src) vp = __ldcg(sm.xp_src + c);
    }
    sm.xw[tid] = v;
    sm.xp[tid] = vp;
    s1 = v;
    s2 = (double)v * (double)v;
    s3 = (double)vp * (double)vp;
    if (D.need_snap && sm.rank == 0 && c < D.cols)
      D.snap[((size_t)ctl->snap_w * D.n_snap + D.snap_idx) * D.snap_stride + c] = v;
  }
  __syncthreads();
  build_lut(lut, sm.xw);
  block_sum3(s1, s2, s3, sm.red);
  if (tid == 0) {
    double* ws = D.win_stats + 4 * w;
    ws[0] = s1; ws[1] = s2; ws[2] = s3; ws[3] = 0.0;
  }
  if (tid < D.n_layers) {
    int a, b, pend;
    layer_planes(D.layer[tid], mode, ctl, a, b, pend);
    sm.la[tid] = (pend == 2) ? 0 : a;        // planes streamed before any decision
    sm.lb[tid] = pend ? -1 : b;              // final plane count, -1 = pending
  }
  __syncthreads();
  DPQ_STAMP(2);

  // ---- estimator share: the first min(kGShares, m) CTAs of each window -----
  const int rank = sm.rank;
  const int n_sh = min(kGShares, m);
  if (rank < n_sh) {
    if (mode == MODE_DYNAMIC) {
      int ng_total = 0;
      for (int li = 0; li < D.n_layers; ++li) {
        const DevSel& S = D.layer[li].S;
        if (S.est_kind == EST_PROJECTION && S.sentinel == 0) ng_total += S.k;
      }
      const int r0 = ng_total * rank / n_sh, r1 = ng_total * (rank + 1) / n_sh;
      for (int r = r0 + warp; r < r1; r += kW) {
        int li = 0, i = r;
        while (true) {
          const DevSel& S = D.layer[li].S;
          const int kk = (S.est_kind == EST_PROJECTION && S.sentinel == 0) ? S.k : 0;
          if (i < kk) break;
          i -= kk;
          ++li;
        }
        const DevSel& S = D.layer[li].S;
        const bool use_p = sm.xp_src && (S.prev_residual || D.est_in);
        const char* grow = reinterpret_cast<const char*>(S.G) + ((long long)w * S.k + i) * g_row_bytes(S.g_dtype);
        const float acc = g_dot(grow, S.g_dtype, use_p ? sm.xp : sm.xw, lane);
        if (lane == 0)
          atomicAdd(reinterpret_cast<unsigned long long*>(D.gxa + li * kMaxK + i),
                    (unsigned long long)llrint((double)acc * 0x1p40));
      }
    }
    __threadfence();                          // every issuing thread orders its accumulations
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(D.ctr, 1u);                   // estimator share done (the decider CTA waits for all)
    }
  }
  DPQ_STAMP(3);
  DPQ_STAMP(4);
  if (!X.out_flags) pdl_launch();

  // ---- dynamic tiles: warps grab kChunk tiles of this window at a time -----
  const uint32_t lanereg = kLutShared | ((uint32_t)lane * 4u);
  float* Ssm = reinterpret_cast<float*>(smem_raw + kOpSmemBytes) + warp * (kWarpTiles * 32);
  float* Slsm = reinterpret_cast<float*>(smem_raw + kOpSmemBytes) + (kW + warp) * (kWarpTiles * 32);
  int fb0 = sm.lb[0], fb1 = D.n_layers > 1 ? sm.lb[1] : 0, fb2 = D.n_layers > 2 ? sm.lb[2] : 0;
  bool decided = (fb0 >= 0) && (fb1 >= 0) && (fb2 >= 0);
  auto final_bits = [&](int li) { return li == 0 ? fb0 : (li == 1 ? fb1 : fb2); };
  auto layer_of = [&](int t) {
    int li = 0;
    while (li + 1 < D.n_layers && t >= D.layer[li + 1].tile_off) ++li;
    return li;
  };
  // lane-distributed description of one (chunk, phase) task list over this
  // warp's owned tiles t_begin + warp + kW*(c0 + i), i < nc
  int my_t = -1, my_li = 0, p0 = 0, start = 0x7fffffff, total = 0;
  const int n_ct = t_end - t_begin;
  const int n_my = n_ct > warp ? (n_ct - warp + kW - 1) / kW : 0;
  auto describe = [&](int c0, int phase) {
    const int nc = max(0, min(kWarpTiles, n_my - c0));
    my_t = lane < nc ? t_begin + warp + kW * (c0 + lane) : -1;
    my_li = lane < nc ? layer_of(my_t) : 0;
    int q0 = 0, q1 = 0;
    if (lane < nc) {
      const int la = sm.la[my_li];
      if (phase == 0) { q0 = 0; q1 = la; }
      else { q0 = la; q1 = sm.lb[my_li] < 0 ? final_bits(my_li) : la; }
    }
    p0 = q0;
    const int cnt = q1 > q0 ? q1 - q0 : 0;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    start = lane < nc ? incl - cnt : 0x7fffffff;
    total = __shfl_sync(0xffffffffu, incl, 31);
  };
  auto task_src = [&](int k, int& ti, int& pl) -> const uint4* {
    ti = __popc(__ballot_sync(0xffffffffu, start <= k)) - 1;
    const int t = __shfl_sync(0xffffffffu, my_t, ti);
    const int li = __shfl_sync(0xffffffffu, my_li, ti);
    pl = __shfl_sync(0xffffffffu, p0, ti) + (k - __shfl_sync(0xffffffffu, start, ti));
    const DevLayer& L = D.layer[li].L;
    return L.planes + pl * L.plane_stride16 +
           ((long long)w * L.n_tiles + (t - D.layer[li].tile_off)) * (kTileBytes / 16) + lane;
  };
  uint4 qa0, qa1, qa2, qa3, qb0, qb1, qb2, qb3, qc0, qc1, qc2, qc3;
  int ta = 0, tb = 0, tc = 0, pa = 0, pb = 0, pc = 0;
#define DPQ_LOAD(X_, T, PL, k)                                                        \
  {                                                                                   \
    const uint4* s_ = task_src(k, T, PL);                                             \
    X_##0 = ldg_stream(s_); X_##1 = ldg_stream(s_ + 32);                              \
    X_##2 = ldg_stream(s_ + 64); X_##3 = ldg_stream(s_ + 96);                         \
  }
  auto prime = [&]() {
    if (0 < total) DPQ_LOAD(qa, ta, pa, 0);
    if (1 < total) DPQ_LOAD(qb, tb, pb, 1);
    if (2 < total) DPQ_LOAD(qc, tc, pc, 2);
  };
  // 3-deep register pipeline over the described tasks (tile-major, plane
  // ascending) with Horner accumulation S = 2 S + P_p per tile.
  auto run = [&](int phase) {
    float S = 0.f;
    int cur = -1;
#define DPQ_RUN(X_, T, PL, k)                                                         \
  {                                                                                   \
    const float P_ = plane_task(X_##0, X_##1, X_##2, X_##3, lanereg);                 \
    if ((T) != cur) {                                                                 \
      if (cur >= 0) Ssm[cur * 32 + lane] = S;                                         \
      cur = (T);                                                                      \
      S = (phase == 1) ? Ssm[cur * 32 + lane] : 0.f;                                  \
    }                                                                                 \
    S = 2.f * S + P_;                                                                 \
    {                                                                                 \
      const OpLayer& Ly_ = D.layer[__shfl_sync(0xffffffffu, my_li, T)];              \
      if (Ly_.dual && mode == MODE_DYNAMIC && (PL) == Ly_.S.l - 1) Slsm[(T) * 32 + lane] = S; \
    }                                                                                 \
    if ((k) + 3 < total) DPQ_LOAD(X_, T, PL, (k) + 3);                                \
  }
    for (int k = 0; k < total; k += 3) {
      DPQ_RUN(qa, ta, pa, k);
      if (k + 1 >= total) break;
      DPQ_RUN(qb, tb, pb, k + 1);
      if (k + 2 >= total) break;
      DPQ_RUN(qc, tc, pc, k + 2);
    }
#undef DPQ_RUN
    if (cur >= 0) Ssm[cur * 32 + lane] = S;
    __syncwarp();
  };

  for (int c0 = 0; c0 < n_my; c0 += kWarpTiles) {
    const int nc = min(kWarpTiles, n_my - c0);
    const int c_t = lane < nc ? t_begin + warp + kW * (c0 + lane) : -1;
    const int c_li = lane < nc ? layer_of(c_t) : 0;
    for (int i = 0; i < nc; ++i) Ssm[i * 32 + lane] = 0.f;
    __syncwarp();
    describe(c0, 0);
    prime();
    run(0);
    // planes gated by a pending decision
    bool need = false;
    for (int i = 0; i < nc; ++i)
      if (sm.lb[__shfl_sync(0xffffffffu, c_li, i)] < 0) need = true;
    if (need) {
      if (!decided) {
        DPQ_STAMP(5);
        if (lane == 0) DPQ_SPIN_UNTIL(ld_acquire(D.ctr + 2) != 0u, "decision", D.n_layers, D.n_win, 0u);
        __syncwarp();
        if (fb0 < 0) fb0 = __ldcg(D.decision + 0);
        if (fb1 < 0) fb1 = __ldcg(D.decision + 1);
        if (fb2 < 0) fb2 = __ldcg(D.decision + 2);
        decided = true;
        DPQ_STAMP(6);
      }
      describe(c0, 1);
      prime();
      run(1);
    }

    // ---- publish partial sums; per-tile last arriver reduces over windows --
    const int bsel_i = lane < nc ? final_bits(c_li) : 0;
    for (int i = 0; i < nc; ++i) {
      const int t = __shfl_sync(0xffffffffu, c_t, i);
      const int li = __shfl_sync(0xffffffffu, c_li, i);
      const bool dual = D.layer[li].dual && mode == MODE_DYNAMIC;
      const int row_g = t * 32 + lane;
      D.part[(size_t)w * D.rows_total_pad + row_g] = Ssm[i * 32 + lane];
      if (dual) D.part_lo[(size_t)w * D.rows_total_pad + row_g] = Slsm[i * 32 + lane];
    }
    __threadfence();
    __syncwarp();
    unsigned old = 0;
    if (lane < nc) old = atomicAdd(D.tile_cnt + c_t, 1u);
    const unsigned lastmask = __ballot_sync(0xffffffffu, lane < nc && old == (unsigned)n_win - 1);
    if (lastmask) {
      __threadfence();
      if (lane < nc && ((lastmask >> lane) & 1u)) D.tile_cnt[c_t] = 0u;
      double sx = 0.0, sq = 0.0;
      for (int ii = lane; ii < n_win; ii += 32) {
        sx += __ldcg(D.win_stats + 4 * ii);
        sq += __ldcg(D.win_stats + 4 * ii + 1);
      }
      sx = warp_sum(sx);
      sq = warp_sum(sq);
      const float scale = D.in_mode == IN_RMS ? (float)(1.0 / sqrt(sq / (double)D.cols + (double)D.eps)) : 1.f;
      const float sxf = (float)sx;
      for (unsigned mk = lastmask; mk; mk &= mk - 1) {
        const int i = __ffs(mk) - 1;
        const int t = __shfl_sync(0xffffffffu, c_t, i);
        const int li = __shfl_sync(0xffffffffu, c_li, i);
        const int bsel = __shfl_sync(0xffffffffu, bsel_i, i);
        const OpLayer& Ly = D.layer[li];
        const bool dual = Ly.dual && mode == MODE_DYNAMIC;
        const int row_g = t * 32 + lane;
        float St0 = 0.f, St1 = 0.f, Stl = 0.f;
        int ww = 0;
        for (; ww + 1 < n_win; ww += 2) {
          St0 += __ldcg(D.part + (size_t)ww * D.rows_total_pad + row_g);
          St1 += __ldcg(D.part + (size_t)(ww + 1) * D.rows_total_pad + row_g);
        }
        if (ww < n_win) St0 += __ldcg(D.part + (size_t)ww * D.rows_total_pad + row_g);
        const float St = St0 + St1;
        if (dual)
          for (int w2 = 0; w2 < n_win; ++w2) Stl += __ldcg(D.part_lo + (size_t)w2 * D.rows_total_pad + row_g);
        const int r = row_g - Ly.tile_off * 32;
        if (r < Ly.L.rows) {
          const float lo = __ldg(Ly.L.lo + r), span = __ldg(Ly.L.span + r);
          const int out_row = Ly.out_off + r;
          if (!dual) {
            const float y = scale * (lo * sxf + ldexpf(span, -bsel) * (St + 0.5f * sxf));
            if (D.out_mode == OUT_ADD) D.out[out_row] = __ldcg(D.out + out_row) + y;
            else D.out[out_row] = y;
          } else {
            const float yh = scale * (lo * sxf + ldexpf(span, -Ly.S.h) * (St + 0.5f * sxf));
            const float yl = scale * (lo * sxf + ldexpf(span, -Ly.S.l) * (Stl + 0.5f * sxf));
            D.out_hi[out_row] = yh;
            D.out_lo[out_row] = yl;
            const float dd = yh - yl;
            const double q = warp_sum((double)dd * (double)dd);
            if (lane == 0) D.dual_sq[t] = (float)q;
          }
        } else if (dual) {
          const double q = warp_sum(0.0);
          if (lane == 0) D.dual_sq[t] = (float)q;
        }
        if (X.out_flags) {
          __threadfence();
          __syncwarp();
          if (lane == 0) st_release(X.out_flags + t, X.epoch);
        }
      }
    }
  }
#undef DPQ_LOAD
  // ---- op done: the last CTA resets the op's counters for the next use -----
  __syncthreads();
  if (tid == 0) op_done(D, G);
  DPQ_STAMP(7);
}

extern "C" __global__ void __launch_bounds__(kThreads, 1)
op_kernel(const OpDesc D, Control* __restrict__ ctl) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ Control cs;          // the control block, read once
  pdl_wait();
  if (threadIdx.x == 0) cs = *ctl;
  __syncthreads();
  // the last CTA is the op's decider; the others own the tiles
  if (blockIdx.x == gridDim.x - 1) {
    if (threadIdx.x < 32) decide_warp(D, &cs, gridDim.x - 1);
    return;
  }
  StageCtx X{};
  X.cta = blockIdx.x;
  X.G = gridDim.x - 1;
  op_stage(D, &cs, X, smem_raw);
}

// ---------------------------------------------------------------------------
// Dual (exact / track_exact) epilogue: one CTA per layer of the op.
// exact = ||y_h - y_l|| (estimator.py:30-32 with lo cancelling), decision for
// EXACT estimators, trace, and the selected output (store or residual add).
// ---------------------------------------------------------------------------
extern "C" __global__ void __launch_bounds__(256)
finalize_dual(const OpDesc D, Control* __restrict__ ctl) {
  __shared__ double red[32];
  __shared__ int sbit;
  const int li = blockIdx.x;
  if (li >= D.n_layers) return;
  const OpLayer& Ly = D.layer[li];
  if (!Ly.dual) return;
  pdl_wait();
  if (ctl->mode != MODE_DYNAMIC) return;
  const DevSel& S = Ly.S;
  double q = 0.0;
  for (int t = threadIdx.x; t < Ly.L.n_tiles; t += blockDim.x) q += (double)D.dual_sq[Ly.tile_off + t];
  q = block_sum_d(q, red);
  const double exact = sqrt(q);
  if (threadIdx.x == 0) {
    int bit;
    double est = CUDART_NAN;
    bool have_est = false;
    if (ctl->force && Ly.trace_idx >= 0) bit = ctl->forced_bits[Ly.trace_idx];
    else if (S.sentinel == 1) bit = S.l;
    else if (S.sentinel == 2) bit = S.h;
    else if (S.sentinel == 3) bit = D.decision[li];
    else if (S.est_kind == EST_EXACT) { est = exact; have_est = true; bit = est > S.T ? S.h : S.l; }
    else bit = D.decision[li];
    if (S.est_kind == EST_EXACT && S.sentinel == 0 && !have_est) { est = exact; have_est = true; }
    if (S.sentinel == 1 || S.sentinel == 2) have_est = false;
    sbit = bit;
    if (Ly.trace_idx >= 0 && D.n_trace > 0) {
      const size_t o = (size_t)ctl->trace_step * D.n_trace + Ly.trace_idx;
      D.tr_bits[o] = (signed char)bit;
      if (S.sentinel != 3 && S.est_kind == EST_EXACT) D.tr_est[o] = have_est ? (float)est : CUDART_NAN_F;
      D.tr_exact[o] = (float)exact;
    }
    D.decision[li] = bit;
  }
  __syncthreads();
  const int bit = sbit;
  const float* src = bit == S.h ? D.out_hi : D.out_lo;
  for (int r = threadIdx.x; r < Ly.L.rows; r += blockDim.x) {
    const int o = Ly.out_off + r;
    if (D.out_mode == OUT_ADD) D.out[o] += src[o];
    else D.out[o] = src[o];
  }
}

// Exact estimator over a previous-residual input: dual_sq of an estimation op
// run on the snapshot vector -> estimate + decision for the main op (sentinel 3).
extern "C" __global__ void decide_exact(const OpDesc E, Control* __restrict__ ctl) {
  __shared__ double red[32];
  pdl_wait();
  if (ctl->mode != MODE_DYNAMIC) return;
  for (int li = 0; li < E.n_layers; ++li) {
    const OpLayer& Ly = E.layer[li];
    double q = 0.0;
    for (int t = threadIdx.x; t < Ly.L.n_tiles; t += blockDim.x) q += (double)E.dual_sq[Ly.tile_off + t];
    q = block_sum_d(q, red);
    if (threadIdx.x == 0) {
      const double est = sqrt(q);
      int bit = est > Ly.S.T ? Ly.S.h : Ly.S.l;
      if (ctl->force && Ly.trace_idx >= 0) bit = ctl->forced_bits[Ly.trace_idx];
      E.main_decision[Ly.main_li] = bit;
      if (Ly.trace_idx >= 0 && E.n_trace > 0) {
        const size_t o = (size_t)ctl->trace_step * E.n_trace + Ly.trace_idx;
        E.tr_bits[o] = (signed char)bit;
        E.tr_est[o] = (float)est;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Decode glue
// ---------------------------------------------------------------------------
struct AttnDesc {
  const float* qkv;      // q [d], k [dkv], v [dkv]
  float* kc;             // [seq_cap][dkv] rotated keys
  float* vc;             // [seq_cap][dkv]
  const float* cosv;     // [seq_cap][half]
  const float* sinv;
  float* part;           // [H][n_chunks][hd + 2]
  unsigned* cnt;         // [H]
  float* out;            // [d]
  int H, KV, hd, d, dkv, n_chunks;
  const unsigned* qkv_flags;   // persistent: per 32-row tile of the qkv op output
  unsigned* head_flags;        // persistent: per head, set when attn[h] is final
};

constexpr int kAttnChunk = 64;

__device__ __forceinline__ float rope_elem(const float* v, int i, int hd, const float* c, const float* s) {
  const int half = hd / 2;
  if (i < half) return __ldcg(v + i) * c[i] - __ldcg(v + i + half) * s[i];
  if (i < 2 * half) return __ldcg(v + i - half) * s[i - half] + __ldcg(v + i) * c[i - half];
  return __ldcg(v + i);
}

// One (head, 64-position chunk) unit: RoPE on q and the new k, scores, chunk
// softmax stats and weighted V; the last chunk of a head merges the chunks
// (runtime.py:351-362). smem: (3 hd + kAttnChunk) floats + 1 int.
__device__ void attn_unit(const AttnDesc& A, int h, int ch, int t, float* ash, float* kvs, unsigned epoch) {
  float* q = ash;
  float* kt = q + A.hd;
  float* vt = kt + A.hd;
  float* sc = vt + A.hd;
  int* last = reinterpret_cast<int*>(sc + kAttnChunk);
  const int n_used = t / kAttnChunk + 1;
  const int grp = A.H / A.KV, kvh = h / grp;
  const int half = A.hd / 2;
  const float* cs = A.cosv + (size_t)t * half;
  const float* sn = A.sinv + (size_t)t * half;
  const float* qraw = A.qkv + h * A.hd;
  const float* kraw = A.qkv + A.d + kvh * A.hd;
  const float* vraw = A.qkv + A.d + A.dkv + kvh * A.hd;
  const float scale = 1.0f / sqrtf((float)A.hd);
  if (A.qkv_flags && threadIdx.x < 32) {
    wait_flags_warp(A.qkv_flags, (h * A.hd) / 32, (h * A.hd + A.hd + 31) / 32, epoch);
    wait_flags_warp(A.qkv_flags, (A.d + kvh * A.hd) / 32, (A.d + kvh * A.hd + A.hd + 31) / 32, epoch);
    wait_flags_warp(A.qkv_flags, (A.d + A.dkv + kvh * A.hd) / 32, (A.d + A.dkv + kvh * A.hd + A.hd + 31) / 32,
                    epoch);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < A.hd; i += blockDim.x) {
    q[i] = half ? rope_elem(qraw, i, A.hd, cs, sn) : __ldcg(qraw + i);
    kt[i] = half ? rope_elem(kraw, i, A.hd, cs, sn) : __ldcg(kraw + i);
    vt[i] = __ldcg(vraw + i);
  }
  __syncthreads();
  // the first query head of each kv group appends position t to the cache
  if (h % grp == 0 && ch == n_used - 1) {
    for (int i = threadIdx.x; i < A.hd; i += blockDim.x) {
      A.kc[(size_t)t * A.dkv + kvh * A.hd + i] = kt[i];
      A.vc[(size_t)t * A.dkv + kvh * A.hd + i] = vt[i];
    }
  }
  const int s0 = ch * kAttnChunk, s1 = min(t + 1, s0 + kAttnChunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // stage this chunk's K and V rows in shared memory (one coalesced pass)
  float* Ks = kvs;
  float* Vs = kvs + kAttnChunk * A.hd;
  const int npos = s1 - s0;
  for (int idx = threadIdx.x; idx < npos * A.hd; idx += blockDim.x) {
    const int sp = idx / A.hd, i = idx - sp * A.hd;
    const int s = s0 + sp;
    if (s == t) { Ks[idx] = kt[i]; Vs[idx] = vt[i]; }
    else {
      Ks[idx] = __ldcg(A.kc + (size_t)s * A.dkv + kvh * A.hd + i);
      Vs[idx] = __ldcg(A.vc + (size_t)s * A.dkv + kvh * A.hd + i);
    }
  }
  __syncthreads();
  for (int s = s0 + warp; s < s1; s += nw) {
    const float* kr = Ks + (s - s0) * A.hd;
    float acc = 0.f;
    for (int i = lane; i < A.hd; i += 32) acc += q[i] * kr[i];
    acc = warp_sum(acc);
    if (lane == 0) sc[s - s0] = acc * scale;
  }
  __syncthreads();
  float mx = -CUDART_INF_F;
  for (int s = s0; s < s1; ++s) mx = fmaxf(mx, sc[s - s0]);
  __syncthreads();
  for (int s = s0 + threadIdx.x; s < s1; s += blockDim.x) sc[s - s0] = expf(sc[s - s0] - mx);
  __syncthreads();
  float l = 0.f;
  for (int s = s0; s < s1; ++s) l += sc[s - s0];
  if (n_used == 1) {
    for (int i = threadIdx.x; i < A.hd; i += blockDim.x) {
      float o = 0.f;
      for (int s = 0; s < npos; ++s) o += sc[s] * Vs[s * A.hd + i];
      A.out[h * A.hd + i] = o / l;
    }
    __syncthreads();
    if (threadIdx.x == 0 && A.head_flags) {
      __threadfence();
      st_release(A.head_flags + h, epoch);
    }
    return;
  }
  float* P = A.part + ((size_t)h * A.n_chunks + ch) * (A.hd + 2);
  for (int i = threadIdx.x; i < A.hd; i += blockDim.x) {
    float o = 0.f;
    for (int s = 0; s < npos; ++s) o += sc[s] * Vs[s * A.hd + i];
    P[i] = o;
  }
  if (threadIdx.x == 0) { P[A.hd] = mx; P[A.hd + 1] = l; }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned old = atomicAdd(A.cnt + h, 1u);
    *last = (old == (unsigned)n_used - 1);
  }
  __syncthreads();
  if (!*last) return;
  __threadfence();
  float M = -CUDART_INF_F;
  for (int c = 0; c < n_used; ++c)
    M = fmaxf(M, __ldcg(A.part + ((size_t)h * A.n_chunks + c) * (A.hd + 2) + A.hd));
  float Lsum = 0.f;
  for (int c = 0; c < n_used; ++c) {
    const float* Pc = A.part + ((size_t)h * A.n_chunks + c) * (A.hd + 2);
    Lsum += __ldcg(Pc + A.hd + 1) * expf(__ldcg(Pc + A.hd) - M);
  }
  for (int i = threadIdx.x; i < A.hd; i += blockDim.x) {
    float o = 0.f;
    for (int c = 0; c < n_used; ++c) {
      const float* Pc = A.part + ((size_t)h * A.n_chunks + c) * (A.hd + 2);
      o += __ldcg(Pc + i) * expf(__ldcg(Pc + A.hd) - M);
    }
    A.out[h * A.hd + i] = o / Lsum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    A.cnt[h] = 0u;
    if (A.head_flags) {
      __threadfence();
      st_release(A.head_flags + h, epoch);
    }
  }
}

// grid (H, n_chunks), 128 threads.
extern "C" __global__ void __launch_bounds__(128)
attention_kernel(const AttnDesc A, Control* __restrict__ ctl) {
  extern __shared__ float ash[];
  pdl_wait();
  const int t = ctl->pos;
  if ((int)blockIdx.y >= t / kAttnChunk + 1) return;
  attn_unit(A, blockIdx.x, blockIdx.y, t, ash, ash + 3 * A.hd + kAttnChunk + 4, 0u);
}

struct HeadDesc {
  const float* x;        // residual stream [d]
  const float* lm;       // [vocab][d]
  float* logits;         // [vocab]
  int* tok_log;          // [max_steps] argmax of every step
  unsigned* cnt;         // [1]
  int vocab, d;
  float eps;
  int max_steps;
  const unsigned* x_flags;   // persistent: all d/32 tiles of the last down op
};

// Final RMSNorm + lm_head rows [16 cta, 16 cta + 16) + (last CTA) greedy
// argmax and end-of-step control (runtime.py:372-380). blockDim 512.
__device__ void head_stage(const HeadDesc& Hd, Control* __restrict__ ctl, int cta, int G, float* xs,
                           unsigned epoch) {
  __shared__ double red[32];
  __shared__ int last;
  __shared__ float bv[512];
  __shared__ int bx[512];
  if (Hd.x_flags && threadIdx.x < 32) wait_flags_warp(Hd.x_flags, 0, (Hd.d + 31) / 32, epoch);
  __syncthreads();
  double sq = 0.0;
  for (int i = threadIdx.x; i < Hd.d; i += blockDim.x) { const double v = __ldcg(Hd.x + i); sq += v * v; }
  sq = block_sum_d(sq, red);
  const float inv = (float)(1.0 / sqrt(sq / (double)Hd.d + (double)Hd.eps));
  for (int i = threadIdx.x; i < Hd.d; i += blockDim.x) xs[i] = __ldcg(Hd.x + i) * inv;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int v = cta * 16 + warp; warp < 16 && v < Hd.vocab; v += G * 16) {
    const float* row = Hd.lm + (size_t)v * Hd.d;
    float acc = 0.f;
    for (int i = lane; i < Hd.d; i += 32) acc += row[i] * xs[i];
    acc = warp_sum(acc);
    if (lane == 0) Hd.logits[v] = acc;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(Hd.cnt, 1u) == (unsigned)G - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // greedy argmax (first maximum, like np.argmax)
  float best = -CUDART_INF_F;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < Hd.vocab; i += blockDim.x) {
    const float z = __ldcg(Hd.logits + i);
    if (z > best || (z == best && i < bi)) { best = z; bi = i; }
  }
  bv[threadIdx.x] = best;
  bx[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      const float zb = bv[threadIdx.x + o];
      const int ib = bx[threadIdx.x + o];
      if (zb > bv[threadIdx.x] || (zb == bv[threadIdx.x] && ib < bx[threadIdx.x])) {
        bv[threadIdx.x] = zb;
        bx[threadIdx.x] = ib;
      }
    }
    __syncthreads();
  }
  const int arg = bx[0];
  if (threadIdx.x == 0) {
    Hd.cnt[0] = 0u;
    const int dyn = ctl->mode == MODE_DYNAMIC;
    ctl->token = arg;                 // greedy next token (host may override)
    if (ctl->n_steps_done < Hd.max_steps) Hd.tok_log[ctl->n_steps_done] = arg;
    ctl->pos += 1;
    if (dyn) ctl->trace_step += 1;
    if (dyn || ctl->prime) {          // runtime.py:379-380
      ctl->snap_r = ctl->snap_w;
      ctl->snap_w ^= 1;
      ctl->has_prev = 1;
    }
    __threadfence();
    ctl->n_steps_done += 1;
  }
}

// grid: ceil(vocab / 16) CTAs x 512 threads.
extern "C" __global__ void __launch_bounds__(512)
lmhead_kernel(const HeadDesc Hd, Control* __restrict__ ctl) {
  extern __shared__ float xs[];
  pdl_wait();
  head_stage(Hd, ctl, blockIdx.x, gridDim.x, xs, 0u);
}

// x = embed[ctl->token]  (runtime.py:345)
extern "C" __global__ void begin_kernel(const float* __restrict__ embed, float* __restrict__ x, int d,
                                        Control* __restrict__ ctl) {
  pdl_wait();
  const int tok = ctl->token;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x)
    x[i] = embed[(size_t)tok * d + i];
}

// ---------------------------------------------------------------------------
// Persistent decode step: one CTA per SM runs every stage of one token.
// Stages are linked by epoch-tagged readiness flags (per 32-row output tile of
// an op, per attention head, per embedding tile) instead of kernel
// boundaries: a CTA starts its share of op N+1 as soon as the input window it
// needs is final, and prefetches op N+1's planes into L2 while op N runs.
// ---------------------------------------------------------------------------
enum StageKind : int { ST_BEGIN = 0, ST_OP = 1, ST_ATTN = 2, ST_HEAD = 3 };

struct Stage {
  int kind;
  int idx;                   // op / attention index
  int G;                     // participating CTAs
  int next_op;               // op whose planes to prefetch (-1 none)
  const unsigned* dep0;
  const unsigned* dep1;
  int dep0_off, dep0_rpf, dep1_off, pad_;
  unsigned* out_flags;
};

struct StepDesc {
  int n_stages;
  const Stage* stages;
  const OpDesc* ops;
  const AttnDesc* attn;
  HeadDesc head;
  const float* embed;
  float* x;
  unsigned* x_flags;         // begin stage output flags [d/32]
  int d;
};

extern "C" __global__ void __launch_bounds__(kThreads, 1)
step_kernel(const StepDesc SD, Control* __restrict__ ctl) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ Control cs;          // the control block, read once (constant during a step)
  pdl_wait();
  if (threadIdx.x == 0) cs = *ctl;
  __syncthreads();
  const unsigned epoch = (unsigned)cs.n_steps_done + 1u;
  // scratch region below the LUT: [OpSmem][S arrays 32 KB][OpDesc copy]
  float* aux = reinterpret_cast<float*>(smem_raw + kOpSmemBytes);
  OpDesc* dsm = reinterpret_cast<OpDesc*>(smem_raw + kOpSmemBytes + 2 * kThreads * kWarpTiles * 4);
  const int cta = blockIdx.x;
  // embedding: CTA c writes x tiles c, c+G, ...
  {
    const int tok = cs.token;
    const int n_t = (SD.d + 31) / 32;
    for (int tt = cta; tt < n_t; tt += gridDim.x) {
      const int i = tt * 32 + (threadIdx.x & 31);
      if (threadIdx.x < 32 && i < SD.d) SD.x[i] = SD.embed[(size_t)tok * SD.d + i];
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        st_release(SD.x_flags + tt, epoch);
      }
    }
  }
  for (int si = 0; si < SD.n_stages; ++si) {
    const Stage st = SD.stages[si];
    __syncthreads();
    if (st.kind == ST_OP) {
      if (cta == (int)gridDim.x - 1) {           // the dedicated decider CTA
        if (threadIdx.x < 32) decide_warp(SD.ops[st.idx], &cs, st.G);
        continue;
      }
      if (cta >= st.G) continue;
      const int n = (int)(sizeof(OpDesc) / 4);
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        reinterpret_cast<int*>(dsm)[i] = reinterpret_cast<const int*>(SD.ops + st.idx)[i];
      __syncthreads();
      StageCtx X{};
      X.cta = cta;
      X.G = st.G;
      X.epoch = epoch;
      X.dep0 = st.dep0;
      X.dep0_off = st.dep0_off;
      X.dep0_rpf = st.dep0_rpf;
      X.dep1 = st.dep1;
      X.dep1_off = st.dep1_off;
      X.out_flags = st.out_flags;
      X.next = st.next_op >= 0 ? SD.ops + st.next_op : nullptr;
      op_stage(*dsm, &cs, X, smem_raw);
    } else if (st.kind == ST_ATTN) {
      const AttnDesc& A = SD.attn[st.idx];
      const int t = cs.pos;
      const int n_used = t / kAttnChunk + 1;
      const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
      float* kvs = reinterpret_cast<float*>(smem_raw + (kLutShared - sbase));   // LUT region is free here
      for (int u = cta; u < A.H * n_used; u += gridDim.x - 1) {
        if (cta == (int)gridDim.x - 1) break;
        attn_unit(A, u / n_used, u % n_used, t, aux, kvs, epoch);
        __syncthreads();
      }
    } else if (st.kind == ST_HEAD) {
      if (cta < st.G && cta != (int)gridDim.x - 1) head_stage(SD.head, ctl, cta, st.G, aux, epoch);
    }
  }
}

// ---------------------------------------------------------------------------
// Store construction
// ---------------------------------------------------------------------------

// codes (row-major, uint16 or uint8, or code_bytes == 0: the .dpqs packed
// stream, code-major LSB-first n_bits per code, quant.py:123-126) -> device
// plane layout. One thread per (row, 8-column group); writes one byte per plane.
__device__ __forceinline__ unsigned packed_code(const unsigned char* __restrict__ blob, long long o, int n_bits,
                                                long long nbytes) {
  const long long bit = o * n_bits;
  const long long i = bit >> 3;
  unsigned w = blob[i];
  if (i + 1 < nbytes) w |= (unsigned)blob[i + 1] << 8;        // n_bits <= 8: at most two bytes
  return (w >> (bit & 7)) & ((1u << n_bits) - 1u);
}

extern "C" __global__ void repack_kernel(const void* __restrict__ codes, int code_bytes, int rows,
                                         int cols, int n_bits, int n_win, int n_tiles,
                                         unsigned char* __restrict__ planes) {
  const long long nbytes = ((long long)rows * cols * n_bits + 7) >> 3;   // packed stream size
  const long long n_groups = (long long)n_tiles * 32 * n_win * kGroups;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n_groups;
       idx += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(idx % kGroups);
    const long long rest = idx / kGroups;
    const int w = (int)(rest % n_win);
    const int row = (int)(rest / n_win);
    const int tile = row >> 5, lane = row & 31;
    unsigned c8[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int col = w * kWinCols + 8 * g + t;
      unsigned v = 0;
      if (row < rows && col < cols) {
        const long long o = (long long)row * cols + col;
        v = code_bytes == 2   ? reinterpret_cast<const unsigned short*>(codes)[o]
            : code_bytes == 1 ? reinterpret_cast<const unsigned char*>(codes)[o]
                              : packed_code(reinterpret_cast<const unsigned char*>(codes), o, n_bits, nbytes);
      }
      c8[t] = v;
    }
    const int s = (g - lane + 64) & 63;               // step that lane uses for group g
    const int wrap = (lane + s) >= 64;
    const int c = s >> 4, b16 = s & 15;
    for (int p = 0; p < n_bits; ++p) {
      unsigned e = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) e |= ((c8[t] >> (n_bits - 1 - p)) & 1u) << t;
      e = (e - wrap) & 255u;
      const long long off = (((long long)p * n_win + w) * n_tiles + tile) * kTileBytes + c * 512 + lane * 16 + b16;
      planes[off] = (unsigned char)e;
    }
  }
}

// quant.py:43-64 on the device, float64, without FMA contraction so codes are
// bit-identical to the reference's numpy. One CTA per row.
extern "C" __global__ void quantize_kernel(const float* __restrict__ W, int rows, int cols, int n_bits,
                                           unsigned short* __restrict__ codes, float* __restrict__ lo,
                                           float* __restrict__ hi) {
  __shared__ float rmin[32], rmax[32];
  const int r = blockIdx.x;
  if (r >= rows) return;
  const float* w = W + (size_t)r * cols;
  float mn = CUDART_INF_F, mx = -CUDART_INF_F;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) { mn = fminf(mn, w[c]); mx = fmaxf(mx, w[c]); }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) { rmin[threadIdx.x >> 5] = mn; rmax[threadIdx.x >> 5] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x + 31) / 32; ++i) { mn = fminf(mn, rmin[i]); mx = fmaxf(mx, rmax[i]); }
    rmin[0] = fminf(mn, rmin[0]);
    rmax[0] = fmaxf(mx, rmax[0]);
  }
  __syncthreads();
  const double l = rmin[0], h = rmax[0];
  const double span = __dsub_rn(h, l);
  const int levels = 1 << n_bits;
  const double mul = __ddiv_rn((double)levels, span == 0.0 ? 1.0 : span);
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    double v = floor(__dmul_rn(__dsub_rn((double)w[c], l), mul));
    v = fmin(fmax(v, 0.0), (double)(levels - 1));
    codes[(size_t)r * cols + c] = span == 0.0 ? 0 : (unsigned short)v;
  }
  if (threadIdx.x == 0) { lo[r] = (float)l; hi[r] = (float)h; }
}

// Dequantize from the device planes (quant.py:67-80), float64 output,
// W = lo + (t + 0.5) * span / 2^b with span = hi - lo evaluated in float64.
extern "C" __global__ void dequant_kernel(const DevLayer L, const float* __restrict__ hi, int b,
                                          double* __restrict__ out) {
  const long long n = (long long)L.rows * L.cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(idx / L.cols), col = (int)(idx % L.cols);
    const int tile = row >> 5, lane = row & 31;
    const int w = col / kWinCols, g = (col % kWinCols) >> 3, tb = col & 7;
    const int s = (g - lane + 64) & 63;
    const int wrap = (lane + s) >= 64;
    const int c = s >> 4, b16 = s & 15;
    unsigned t = 0;
    for (int p = 0; p < b; ++p) {
      const unsigned char* base = reinterpret_cast<const unsigned char*>(L.planes + p * L.plane_stride16);
      const long long off = ((long long)w * L.n_tiles + tile) * kTileBytes + c * 512 + lane * 16 + b16;
      const unsigned e = (base[off] + wrap) & 255u;
      t = (t << 1) | ((e >> tb) & 1u);
    }
    const double lo = L.lo[row];
    const double span = __dsub_rn((double)hi[row], lo);
    const double v = __dadd_rn(lo, __ddiv_rn(__dmul_rn(__dadd_rn((double)t, 0.5), span), (double)(1 << b)));
    out[idx] = v;
  }
}

}  // namespace dpq
