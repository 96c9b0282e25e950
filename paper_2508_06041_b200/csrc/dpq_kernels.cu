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
#define DPQ_STAMP(i) \
  do { if (D.dbg && threadIdx.x == 0) D.dbg[blockIdx.x * 8 + (i)] = gtimer(); } while (0)
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
  double lay_q[kMaxOpLayers * 4];
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

extern "C" __global__ void __launch_bounds__(kThreads, 1)
op_kernel(const OpDesc D, Control* __restrict__ ctl) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // Shared layout: [sbase, 0x10000): OpSmem + plane sums; [0x10000, +kLutBytes): LUT.
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
  float* lut = reinterpret_cast<float*>(smem_raw + (kLutShared - sbase));
  OpSmem& sm = *reinterpret_cast<OpSmem*>(smem_raw);
  // below the LUT: OpSmem, then S / S_l per warp-owned tile [2][16 warps][kWarpTiles][32]
  if (kOpSmemBytes + 2 * kThreads * kWarpTiles * 4 > kLutShared - sbase) __trap();

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int n_win = D.n_win;
  const int mode = ctl->mode;

  // ---- CTA -> (window, tile range) --------------------------------------
  // CTAs c = w, w + n_win, w + 2 n_win, ... share window w.
  const int w = blockIdx.x % n_win;
  const int j = blockIdx.x / n_win;
  const int m = (G - w + n_win - 1) / n_win;
  const int t_begin = (int)((long long)D.total_tiles * j / m);
  const int t_end = (int)((long long)D.total_tiles * (j + 1) / m);

  // ---- L2 prefetch of the always-streamed planes (independent of inputs) --
  if (tid == 0) {
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
  DPQ_STAMP(0);
  pdl_wait();
  DPQ_STAMP(1);
  if (tid == 0) sm.my_gen = *reinterpret_cast<volatile unsigned*>(&D.sync->gen);

  // ---- prologue: input window, estimator-input window, window stats --------
  const int col0 = w * kWinCols;
  if (tid == 0) {
    // estimator input for previous-residual estimators (runtime.py:300-309)
    const float* src = nullptr;
    double scale = 1.0;
    if (D.est_in) {
      src = D.est_in;
    } else if (mode == MODE_DYNAMIC) {
      int need = 0;
      for (int li = 0; li < D.n_layers; ++li) {
        const DevSel& S = D.layer[li].S;
        if (S.prev_residual && S.sentinel == 0 && (S.est_kind == EST_LINEAR || S.est_kind == EST_PROJECTION))
          need = 1;
      }
      int slot = -1, idx = -1;
      if (need) {
        if (ctl->async_prev_block) { slot = ctl->snap_w; idx = D.layer[0].snap_in; }
        else if (ctl->has_prev) { slot = ctl->snap_r; idx = D.snap_idx; }
      }
      if (slot >= 0 && idx >= 0) {
        const size_t loc = (size_t)slot * D.n_snap + idx;
        src = D.snap + loc * D.snap_stride;
        if (D.in_mode == IN_RMS) scale = (double)D.snap_stats[loc * 4 + 2];
      }
    }
    sm.xp_src = src;
    sm.xp_scale = scale;
  }
  __syncthreads();
  double s1 = 0.0, s2 = 0.0, s3 = 0.0;
  {
    const int c = col0 + tid;
    float v = 0.f, vp = 0.f;
    if (c < D.cols) {
      if (D.in_mode == IN_SILU) {
        const float up = D.in0[c], gt = D.in1[c];
        v = up * (gt / (1.0f + expf(-gt)));
      } else {
        v = D.in0[c];
      }
      if (sm.xp_src) vp = sm.xp_src[c];
    }
    sm.xw[tid] = v;
    sm.xp[tid] = vp;
    s1 = v;
    s2 = (double)v * (double)v;
    s3 = (double)vp * (double)vp;
    if (D.need_snap && j == 0 && c < D.cols)
      D.snap[((size_t)ctl->snap_w * D.n_snap + D.snap_idx) * D.snap_stride + c] = v;
  }
  __syncthreads();
  build_lut(lut, sm.xw);
  block_sum3(s1, s2, s3, sm.red);
  if (tid == 0) {
    double* ws = D.win_stats + 4 * w;
    ws[0] = s1; ws[1] = s2; ws[2] = s3; ws[3] = 0.0;
  }
  DPQ_STAMP(2);

  // ---- P1: projection-estimator partial dot products (window slice) ------
  if (mode == MODE_DYNAMIC) {
    int ng_total = 0;
    for (int li = 0; li < D.n_layers; ++li) {
      const DevSel& S = D.layer[li].S;
      if (S.est_kind == EST_PROJECTION && S.sentinel == 0) ng_total += S.k;
    }
    if (ng_total > 0) {
      const int r0 = (int)((long long)ng_total * j / m), r1 = (int)((long long)ng_total * (j + 1) / m);
      for (int r = r0 + warp; r < r1; r += kThreads / 32) {
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
        if (lane == 0) D.gx_part[((size_t)li * n_win + w) * kMaxK + i] = acc;
      }
    }
  }

  // ---- op barrier arrive; the last CTA decides -----------------------------
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned old = atomicAdd(&D.sync->arrive, 1u);
    sm.is_last = (old == (unsigned)G - 1);
  }
  __syncthreads();
  DPQ_STAMP(3);
  if (sm.is_last) {
    __threadfence();
    // op input statistics
    double t1 = 0.0, t2 = 0.0, t3 = 0.0;
    for (int i = tid; i < n_win; i += kThreads) {
      t1 += __ldcg(D.win_stats + 4 * i);
      t2 += __ldcg(D.win_stats + 4 * i + 1);
      t3 += __ldcg(D.win_stats + 4 * i + 2);
    }
    block_sum3(t1, t2, t3, sm.red);
    const double inv = 1.0 / sqrt(t2 / (double)D.cols + (double)D.eps);
    if (tid == 0) {
      D.op_stats[0] = (float)t1;
      D.op_stats[1] = (float)t2;
      D.op_stats[2] = (float)inv;
      if (D.need_snap) {
        float* st = D.snap_stats + ((size_t)ctl->snap_w * D.n_snap + D.snap_idx) * 4;
        st[0] = (float)t1; st[1] = (float)t2; st[2] = (float)inv; st[3] = 0.f;
      }
    }
    // projection norms: thread (li, i) sums its window partials; 4 warps per layer
    if (mode == MODE_DYNAMIC) {
      const int li = tid / kMaxK, i = tid % kMaxK;
      double q = 0.0;
      if (li < D.n_layers) {
        const DevSel& S = D.layer[li].S;
        if (S.sentinel == 0 && S.est_kind == EST_PROJECTION && i < S.k) {
          const float* gp = D.gx_part + (size_t)li * n_win * kMaxK + i;
          float g0 = 0.f, g1 = 0.f;
          int ww = 0;
          for (; ww + 1 < n_win; ww += 2) { g0 += __ldcg(gp + (size_t)ww * kMaxK); g1 += __ldcg(gp + (size_t)(ww + 1) * kMaxK); }
          if (ww < n_win) g0 += __ldcg(gp + (size_t)ww * kMaxK);
          float g = g0 + g1;
          if (S.g_scale) g *= S.g_scale[i];
          q = (double)g * (double)g;
        }
      }
      q = warp_sum(q);
      if (lane == 0 && warp < kMaxOpLayers * 4) sm.lay_q[warp] = q;
      __syncthreads();
    }
    for (int li = 0; li < D.n_layers; ++li) {
      const OpLayer& Ly = D.layer[li];
      const DevSel& S = Ly.S;
      if (mode != MODE_DYNAMIC) continue;
      double est = CUDART_NAN;
      bool have_est = false;
      const bool prev = sm.xp_src && (S.prev_residual || D.est_in);
      const double in_scale = prev ? sm.xp_scale : (D.in_mode == IN_RMS ? inv : 1.0);
      if (S.sentinel == 0 && S.est_kind == EST_PROJECTION) {
        const double q = sm.lay_q[4 * li] + sm.lay_q[4 * li + 1] + sm.lay_q[4 * li + 2] + sm.lay_q[4 * li + 3];
        est = in_scale * sqrt(q);
        have_est = true;
      } else if (S.sentinel == 0 && S.est_kind == EST_LINEAR) {
        const double sq = prev ? t3 : t2;
        est = S.slope * (in_scale * sqrt(sq)) + S.intercept;
        have_est = true;
      }
      if (tid == 0) {
        int bit;
        if (S.sentinel == 3 || (Ly.dual && S.est_kind == EST_EXACT && S.sentinel == 0))
          bit = -1;                                         // finalize / prior kernel decides
        else if (ctl->force && Ly.trace_idx >= 0) bit = ctl->forced_bits[Ly.trace_idx];
        else if (S.sentinel == 1) bit = S.l;
        else if (S.sentinel == 2) bit = S.h;
        else if (have_est) bit = (est > S.T) ? S.h : S.l;
        else bit = S.l;
        if (bit >= 0) D.decision[li] = bit;
        if (Ly.trace_idx >= 0 && D.n_trace > 0) {
          const size_t o = (size_t)ctl->trace_step * D.n_trace + Ly.trace_idx;
          if (bit >= 0) D.tr_bits[o] = (signed char)bit;
          if (S.sentinel != 3) D.tr_est[o] = have_est ? (float)est : CUDART_NAN_F;
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      D.sync->arrive = 0u;
      __threadfence();
      st_release(&D.sync->gen, sm.my_gen + 1u);
    }
  }

  DPQ_STAMP(4);
  // ---- per-layer plane counts known to this CTA ----------------------------
  if (tid < D.n_layers) {
    int a, b, pend;
    layer_planes(D.layer[tid], mode, ctl, a, b, pend);
    sm.la[tid] = (pend == 2) ? 0 : a;        // planes streamed before any decision
    sm.lb[tid] = pend ? -1 : b;              // final plane count, -1 = pending
  }
  __syncthreads();
  // Let the next kernel's CTAs start (their L2 prefetch overlaps our stream).
  pdl_launch();

  // ---- warp-owned tiles: tiles t_begin + warp + kW*i, all planes per warp --
  constexpr int kW = kThreads / 32;
  const uint32_t lanereg = kLutShared | ((uint32_t)lane * 4u);
  float* Ssm = reinterpret_cast<float*>(smem_raw + kOpSmemBytes) + warp * (kWarpTiles * 32);
  float* Slsm = reinterpret_cast<float*>(smem_raw + kOpSmemBytes) + (kW + warp) * (kWarpTiles * 32);
  const int n_ct = t_end - t_begin;
  const int n_my = n_ct > warp ? (n_ct - warp + kW - 1) / kW : 0;
  int fb0 = sm.lb[0], fb1 = D.n_layers > 1 ? sm.lb[1] : 0, fb2 = D.n_layers > 2 ? sm.lb[2] : 0;
  bool decided = (fb0 >= 0) && (fb1 >= 0) && (fb2 >= 0);
  auto final_bits = [&](int li) { return li == 0 ? fb0 : (li == 1 ? fb1 : fb2); };
  auto layer_of = [&](int t) {
    int li = 0;
    while (li + 1 < D.n_layers && t >= D.layer[li + 1].tile_off) ++li;
    return li;
  };

  for (int c0 = 0; c0 < n_my; c0 += kWarpTiles) {
    const int nc = min(kWarpTiles, n_my - c0);
    // lane i < nc describes owned tile i of this chunk
    const int my_t = lane < nc ? t_begin + warp + kW * (c0 + lane) : -1;
    const int my_li = lane < nc ? layer_of(my_t) : 0;
    for (int i = 0; i < nc; ++i) Ssm[i * 32 + lane] = 0.f;
    __syncwarp();

    for (int phase = 0; phase < 2; ++phase) {
      if (phase == 1) {
        // decisions of pending layers (one spin per warp, lane 0)
        if (!decided) {
          bool need = false;
          for (int i = 0; i < nc; ++i) {
            const int li = __shfl_sync(0xffffffffu, my_li, i);
            if (final_bits(li) < 0) need = true;
          }
          if (!need) break;
          DPQ_STAMP(5);
          if (lane == 0) {
            while (ld_acquire(&D.sync->gen) == sm.my_gen) __nanosleep(32);
          }
          __syncwarp();
          if (fb0 < 0) fb0 = __ldcg(D.decision + 0);
          if (fb1 < 0) fb1 = __ldcg(D.decision + 1);
          if (fb2 < 0) fb2 = __ldcg(D.decision + 2);
          decided = true;
          DPQ_STAMP(6);
        }
      }
      // per-tile plane range of this phase
      int p0 = 0, p1 = 0;
      if (lane < nc) {
        const int la = sm.la[my_li];
        if (phase == 0) { p0 = 0; p1 = la; }
        else {
          const int fb = final_bits(my_li);
          const bool was_pending = sm.lb[my_li] < 0;
          p0 = la;
          p1 = was_pending ? fb : la;
        }
      }
      // exclusive prefix of task counts across the owned tiles
      const int cnt = p1 > p0 ? p1 - p0 : 0;
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int start = lane < nc ? incl - cnt : 0x7fffffff;
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      if (total == 0) continue;
      auto task_tile = [&](int k) { return __popc(__ballot_sync(0xffffffffu, start <= k)) - 1; };
      auto task_src = [&](int k, int& ti, int& pl) -> const uint4* {
        ti = task_tile(k);
        const int t = __shfl_sync(0xffffffffu, my_t, ti);
        const int li = __shfl_sync(0xffffffffu, my_li, ti);
        pl = __shfl_sync(0xffffffffu, p0, ti) + (k - __shfl_sync(0xffffffffu, start, ti));
        const DevLayer& L = D.layer[li].L;
        return L.planes + pl * L.plane_stride16 +
               ((long long)w * L.n_tiles + (t - D.layer[li].tile_off)) * (kTileBytes / 16) + lane;
      };
      // 3-deep register pipeline over this warp's tasks (tile-major, plane
      // ascending) with Horner accumulation S = 2 S + P_p per owned tile.
      uint4 qa0, qa1, qa2, qa3, qb0, qb1, qb2, qb3, qc0, qc1, qc2, qc3;
      int ta = 0, tb = 0, tc = 0, pa = 0, pb = 0, pc = 0;
      float S = 0.f;
      int cur = -1;
      auto flush_to = [&](int ti) {
        if (cur >= 0) Ssm[cur * 32 + lane] = S;
        cur = ti;
        S = (phase == 1) ? Ssm[ti * 32 + lane] : 0.f;
      };
#define DPQ_LOAD(X, T, PL, k)                                                         \
  {                                                                                   \
    const uint4* s_ = task_src(k, T, PL);                                             \
    X##0 = ldg_stream(s_); X##1 = ldg_stream(s_ + 32);                                \
    X##2 = ldg_stream(s_ + 64); X##3 = ldg_stream(s_ + 96);                           \
  }
#define DPQ_RUN(X, T, PL, k)                                                          \
  {                                                                                   \
    const float P_ = plane_task(X##0, X##1, X##2, X##3, lanereg);                     \
    if ((T) != cur) flush_to(T);                                                      \
    S = 2.f * S + P_;                                                                 \
    {                                                                                 \
      const int lsel_ = D.layer[__shfl_sync(0xffffffffu, my_li, T)].S.l;              \
      const bool dual_ = D.layer[__shfl_sync(0xffffffffu, my_li, T)].dual && mode == MODE_DYNAMIC; \
      if (dual_ && (PL) == lsel_ - 1) Slsm[(T) * 32 + lane] = S;                      \
    }                                                                                 \
    if ((k) + 3 < total) DPQ_LOAD(X, T, PL, (k) + 3);                                 \
  }
      DPQ_LOAD(qa, ta, pa, 0);
      if (1 < total) DPQ_LOAD(qb, tb, pb, 1);
      if (2 < total) DPQ_LOAD(qc, tc, pc, 2);
      for (int k = 0; k < total; k += 3) {
        DPQ_RUN(qa, ta, pa, k);
        if (k + 1 >= total) break;
        DPQ_RUN(qb, tb, pb, k + 1);
        if (k + 2 >= total) break;
        DPQ_RUN(qc, tc, pc, k + 2);
      }
#undef DPQ_RUN
#undef DPQ_LOAD
      if (cur >= 0) Ssm[cur * 32 + lane] = S;
      __syncwarp();
    }

    // ---- publish partial sums of the owned tiles; per-tile last arriver ----
    // reduces over windows and applies the affine epilogue.
    int bsel_i = lane < nc ? final_bits(my_li) : 0;
    for (int i = 0; i < nc; ++i) {
      const int t = __shfl_sync(0xffffffffu, my_t, i);
      const int li = __shfl_sync(0xffffffffu, my_li, i);
      const bool dual = D.layer[li].dual && mode == MODE_DYNAMIC;
      const int row_g = t * 32 + lane;
      D.part[(size_t)w * D.rows_total_pad + row_g] = Ssm[i * 32 + lane];
      if (dual) D.part_lo[(size_t)w * D.rows_total_pad + row_g] = Slsm[i * 32 + lane];
    }
    __threadfence();
    __syncwarp();
    unsigned old = 0;
    if (lane < nc) old = atomicAdd(D.tile_cnt + my_t, 1u);
    const unsigned lastmask = __ballot_sync(0xffffffffu, lane < nc && old == (unsigned)n_win - 1);
    if (lastmask) {
      __threadfence();
      if (lane < nc && ((lastmask >> lane) & 1u)) D.tile_cnt[my_t] = 0u;
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
        const int t = __shfl_sync(0xffffffffu, my_t, i);
        const int li = __shfl_sync(0xffffffffu, my_li, i);
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
            if (D.out_mode == OUT_ADD) D.out[out_row] += y;
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
      }
    }
  }
  DPQ_STAMP(7);
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
};

constexpr int kAttnChunk = 64;

__device__ __forceinline__ float rope_elem(const float* v, int i, int hd, const float* c, const float* s) {
  const int half = hd / 2;
  if (i < half) return v[i] * c[i] - v[i + half] * s[i];
  if (i < 2 * half) return v[i - half] * s[i - half] + v[i] * c[i - half];
  return v[i];
}

// grid (H, n_chunks), 128 threads. Scores for chunk positions, chunk-local
// softmax stats + weighted V; the last chunk CTA of a head merges.
extern "C" __global__ void __launch_bounds__(128)
attention_kernel(const AttnDesc A, Control* __restrict__ ctl) {
  extern __shared__ float ash[];
  float* q = ash;                        // [hd]
  float* kt = q + A.hd;                  // [hd] rotated k at position t
  float* vt = kt + A.hd;                 // [hd]
  float* sc = vt + A.hd;                 // [kAttnChunk]
  __shared__ float red[4];
  __shared__ int last;
  pdl_wait();
  const int h = blockIdx.x, ch = blockIdx.y;
  const int t = ctl->pos;
  const int n_used = t / kAttnChunk + 1;
  if (ch >= n_used) return;
  const int grp = A.H / A.KV, kvh = h / grp;
  const int half = A.hd / 2;
  const float* cs = A.cosv + (size_t)t * half;
  const float* sn = A.sinv + (size_t)t * half;
  const float* qraw = A.qkv + h * A.hd;
  const float* kraw = A.qkv + A.d + kvh * A.hd;
  const float* vraw = A.qkv + A.d + A.dkv + kvh * A.hd;
  const float scale = 1.0f / sqrtf((float)A.hd);
  for (int i = threadIdx.x; i < A.hd; i += blockDim.x) {
    q[i] = half ? rope_elem(qraw, i, A.hd, cs, sn) : qraw[i];
    kt[i] = half ? rope_elem(kraw, i, A.hd, cs, sn) : kraw[i];
    vt[i] = vraw[i];
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
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int s = s0 + warp; s < s1; s += 4) {
    const float* kr = (s == t) ? kt : A.kc + (size_t)s * A.dkv + kvh * A.hd;
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
  float* P = A.part + ((size_t)h * A.n_chunks + ch) * (A.hd + 2);
  for (int i = threadIdx.x; i < A.hd; i += blockDim.x) {
    float o = 0.f;
    for (int s = s0; s < s1; ++s) {
      const float vv = (s == t) ? vt[i] : A.vc[(size_t)s * A.dkv + kvh * A.hd + i];
      o += sc[s - s0] * vv;
    }
    P[i] = o;
  }
  if (threadIdx.x == 0) { P[A.hd] = mx; P[A.hd + 1] = l; }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned old = atomicAdd(A.cnt + h, 1u);
    last = (old == (unsigned)n_used - 1);
  }
  __syncthreads();
  if (!last) return;
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
  if (threadIdx.x == 0) A.cnt[h] = 0u;
  (void)red;
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
};

// grid: ceil(vocab / 16) CTAs x 512 threads (16 warps = 16 logits per CTA).
extern "C" __global__ void __launch_bounds__(512)
lmhead_kernel(const HeadDesc Hd, Control* __restrict__ ctl) {
  extern __shared__ float xs[];          // [d] normalized final residual
  __shared__ double red[32];
  __shared__ int last;
  pdl_wait();
  double sq = 0.0;
  for (int i = threadIdx.x; i < Hd.d; i += blockDim.x) { const double v = Hd.x[i]; sq += v * v; }
  sq = block_sum_d(sq, red);
  const float inv = (float)(1.0 / sqrt(sq / (double)Hd.d + (double)Hd.eps));
  for (int i = threadIdx.x; i < Hd.d; i += blockDim.x) xs[i] = Hd.x[i] * inv;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int v = blockIdx.x * 16 + warp;
  if (v < Hd.vocab) {
    const float* row = Hd.lm + (size_t)v * Hd.d;
    float acc = 0.f;
    for (int i = lane; i < Hd.d; i += 32) acc += row[i] * xs[i];
    acc = warp_sum(acc);
    if (lane == 0) Hd.logits[v] = acc;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(Hd.cnt, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // greedy argmax (first maximum, like np.argmax) + end-of-step control
  float best = -CUDART_INF_F;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < Hd.vocab; i += blockDim.x) {
    const float z = __ldcg(Hd.logits + i);
    if (z > best || (z == best && i < bi)) { best = z; bi = i; }
  }
  __shared__ float bv[512];
  __shared__ int bx[512];
  bv[threadIdx.x] = best;
  bx[threadIdx.x] = bi;
  __syncthreads();
  for (int o = 256; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
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
    ctl->n_steps_done += 1;
  }
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
// Store construction
// ---------------------------------------------------------------------------

// codes (row-major, uint16 or uint8) -> device plane layout. One thread per
// (row, 8-column group); writes one byte per plane.
extern "C" __global__ void repack_kernel(const void* __restrict__ codes, int code_bytes, int rows,
                                         int cols, int n_bits, int n_win, int n_tiles,
                                         unsigned char* __restrict__ planes) {
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
        v = code_bytes == 2 ? reinterpret_cast<const unsigned short*>(codes)[o]
                            : reinterpret_cast<const unsigned char*>(codes)[o];
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
