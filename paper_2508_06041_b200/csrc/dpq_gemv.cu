// Standalone per-layer GEMV and selector+GEMV (dpq_gemv / dpq_select_gemv,
// reference quant.py:95-99 and runtime.py:184-193 + quant.py:95-99): one
// short-lived launch per call, sized for a single layer.
//
// Why a separate kernel: the decode engine is a persistent, multi-stage
// program; a single layer run through it pays its stage hand-offs (BEGIN,
// OP, OUT) on top of the stream. Here every CTA streams a contiguous range of
// the layer's (window, row tile) tasks, so the grid is balanced to one task,
// and the cross-window reduction is a per-tile arrival counter: the CTA that
// completes a tile's last window sums the tile's window partials in fixed
// window order (deterministic) and applies the affine epilogue.
//
// CTA layout: kCW consumer warps (byte-LUT Horner, as the engine) + one TMA
// producer warp. A CTA's task range covers at most two windows (host-checked):
// their byte LUTs sit at shared addresses 0x10000 and 0x20000 (LUT 0's zero
// row 256 is LUT 1's row 0, also zero), so the engine's PRMT-formed lookup
// address (eng::plane_sum) serves both with lanereg = 0x10000 (1 + i) | 4 lane.
//
// Selector (dynamic): the estimator input's G.x is split into (window, G row)
// jobs over all CTAs (64-bit fixed-point red.add, exact and order-free), every
// CTA's producer warp waits for the job counter, takes the same decision from
// the same integers (estimator.py:41-42, 56-57; strict est > T), streams the
// extra planes if high; the last CTA to read the sums resets them.
#pragma once

namespace dpq {
namespace gv {

using eng::u64;
using eng::smem_u32;
using eng::gclock;
using eng::g_diag;

#ifndef DPQ_GV_CW
#define DPQ_GV_CW 16
#endif
#ifndef DPQ_GV_ACQREL
#define DPQ_GV_ACQREL 1
#endif
#ifndef DPQ_GV_GT
#define DPQ_GV_GT 4
#endif
constexpr int kCW = DPQ_GV_CW;              // consumer warps
constexpr int kNC = kCW * 32;               // consumer threads
constexpr int kNT = kNC + 32;               // + the producer warp
constexpr int kGT = DPQ_GV_GT;              // tiles per chunk: one TMA copy = one plane of kGT consecutive tiles
constexpr int kQuads = kCW / kGT;           // warp groups; warp i of a group takes tile i of each chunk
constexpr int kChunk = kGT * 2048;          // 8 KB copies (2 KB copies are TMA-issue bound: tools/ubench_stream.cu)
constexpr int kSlots = 10;                  // ring slots (chunks)
static_assert(kCW % kGT == 0, "consumer warps per chunk group");
constexpr uint32_t kLut0 = 0x10000;         // LUT i at kLut0 (1 + i) - kLut0 ... see header
constexpr int kItem = 2048;

__device__ unsigned long long* g_gv_dbg = nullptr;   // diagnostics: per-CTA timeline (dpq_debug_gemv_stamps)
#ifdef DPQ_GV_STAMPS
#define GV_STAMP(i) do { if (g_gv_dbg) atomicMax(g_gv_dbg + blockIdx.x * 8 + (i), gclock()); } while (0)
// chunk j of CTA b: [0] issued, [1] landed (first reader), [2] released (last reader)
#define GV_CHUNK(j, k) do { if (g_gv_dbg && (j) < 64) g_gv_dbg[gridDim.x * 8 + ((size_t)blockIdx.x * 64 + (j)) * 4 + (k)] = gclock(); } while (0)
#else
#define GV_STAMP(i) do { } while (0)
#define GV_CHUNK(j, k) do { } while (0)
#endif

struct Args {
  const uint4* planes;
  long long pstride16;
  const float* lo;
  const float* span;
  int rows, cols, n_win, n_tiles;
  int l, h;                 // base / high bits (static: l == h)
  int sentinel;             // 0 estimate, 1 low, 2 high (dynamic)
  int est_kind, k, g_dtype;
  const void* G;            // [n_win][k][512]
  const float* g_scale;
  double T, slope, intercept, fbscale, fxscale;
  const float* x;
  float* y;
  int* bit_out;
  float* est_out;
  // scratch (self-resetting)
  float* part;              // [n_win][n_tiles * 32]
  float* sx;                // [n_win] window sums of x
  double* sq;               // [n_win] window sums of x^2
  int* cnt;                 // [n_tiles] window arrivals
  long long* acc;           // [k] G.x fixed point
  int* sync;                // [0] jobs done, [1] CTAs past the decision
  unsigned* err;
};

struct Ctl {
  unsigned long long full[kSlots], empty[kSlots];
  unsigned slot_off[kSlots];
  volatile int seq[kSlots];
  alignas(16) float xw[2][kWinCols];
  volatile int dec_bit;     // -1 until decided
};

// Byte LUT of a window (layout: dpq_common.cuh). Job q = (slot g, row blocks
// 2 mm, 2 mm + 1): the low-nibble subset sums once for both blocks.
__device__ __forceinline__ void lut_build(float* lut, const float* xw, int tid, int nthr) {
  for (int q = tid; q < 512; q += nthr) {
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
    for (int h = 0; h < 2; ++h) {
      const int m = 2 * mm + h;
      float H = 0.f;
      if (m & 1) H += xb.x;
      if (m & 2) H += xb.y;
      if (m & 4) H += xb.z;
      if (m & 8) H += xb.w;
#pragma unroll
      for (int i = 0; i < 16; ++i) lut[(16 * m + i) * kGroups + g] = L[i] + H;
    }
  }
}

#ifndef DPQ_GV_SLEEP
#define DPQ_GV_SLEEP 0
#endif
// consumer waits back off (ns) so that spinning warps leave issue slots to the
// producer warp on their scheduler
#define GV_SPIN(cond, what, a, b)                                                          \
  do {                                                                                     \
    unsigned n_ = 0;                                                                       \
    u64 t0_ = 0;                                                                           \
    while (!(cond)) {                                                                      \
      if (DPQ_GV_SLEEP > 0) __nanosleep(DPQ_GV_SLEEP);                                     \
      if ((++n_ & 255u) == 0) {                                                            \
        const u64 t_ = gclock();                                                           \
        if (t0_ == 0) t0_ = t_;                                                            \
        else if (t_ - t0_ > 4000000000ull) hang(what, a, b);                               \
      }                                                                                    \
    }                                                                                      \
  } while (0)
#define GV_SYNC() asm volatile("bar.sync 1, %0;" :: "n"(dpq::gv::kNC) : "memory")

// Horner over the ring chunks [j0, j0 + n) (one plane each), tile i of each
// (i < nt_chunk; every warp of the group releases the chunk): S = 2 S + P_p.
__device__ __forceinline__ float stream_items(Ctl& c, const unsigned char* dyn0, int j0, int n, int stride, int i,
                                              bool mine, uint32_t lanereg) {
  const int lane = threadIdx.x & 31;
  float S = 0.f;
  for (int q = 0; q < n; ++q) {
    const int j = j0 + q * stride;
    const int sl = j % kSlots;
    if (lane == 0) GV_SPIN(c.seq[sl] == j, "gemv ring sequence", j, c.seq[sl]);
    __syncwarp();
    GV_SPIN(eng::mbar_test(smem_u32(&c.full[sl]), (unsigned)((j / kSlots) & 1)), "gemv ring slot", j, 0);
    if (!mine) {
      __syncwarp();
      if (lane == 0) eng::mbar_arrive_n(&c.empty[sl], 1u);
      continue;
    }
    if (lane == 0 && i == 0) GV_CHUNK(j, 1);
    const uint4* d = reinterpret_cast<const uint4*>(dyn0 + c.slot_off[sl] + i * 2048) + lane;
    const uint4 d0 = d[0], d1 = d[32], d2 = d[64], d3 = d[96];
    __syncwarp();
    if (lane == 0) eng::mbar_arrive_n(&c.empty[sl], 1u);
    if (lane == 0) GV_CHUNK(j, 2);
    S = 2.f * S + eng::plane_sum(d0, d1, d2, d3, lanereg);
  }
  return S;
}

// One estimator job (window w, G row r) per warp: lane l takes columns
// 4 l + 128 q + j. The G row (static) is loaded ahead (gpre_load, before the
// weight stream saturates HBM and before the previous call's x is ready);
// the dot product reads x once the call may.
struct GPre {
  uint4 g[4];
};
__device__ __forceinline__ void gpre_load(const Args& A, int w, int r, GPre& P) {
  const int lane = threadIdx.x & 31;
  const size_t gb = ((size_t)w * A.k + r) * kWinCols + 4 * lane;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (A.g_dtype == G_F16) P.g[q] = eng::ld_nc16_half(reinterpret_cast<const __half*>(A.G) + gb + 128 * q);
    else if (A.g_dtype == G_F32) P.g[q] = eng::ld_nc16(reinterpret_cast<const float*>(A.G) + gb + 128 * q);
    else P.g[q] = make_uint4(eng::ld_nc4(reinterpret_cast<const unsigned char*>(A.G) + gb + 128 * q), 0u, 0u, 0u);
  }
}
__device__ __forceinline__ double g_row_dot(const Args& A, int w, int r, const GPre& P) {
  const int lane = threadIdx.x & 31;
  const float* xw = A.x + (size_t)w * kWinCols;
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c0 = w * kWinCols + 4 * lane + 128 * q;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c0 + 4 <= A.cols) x = __ldg(reinterpret_cast<const float4*>(xw + 4 * lane + 128 * q));
    else
      for (int j = 0; j < 4; ++j)
        if (c0 + j < A.cols) (&x.x)[j] = __ldg(xw + 4 * lane + 128 * q + j);
    float g[4];
    const uint4 t = P.g[q];
    if (A.g_dtype == G_F16) {
      const float2 u = __half22float2(*reinterpret_cast<const __half2*>(&t.x));
      const float2 v = __half22float2(*reinterpret_cast<const __half2*>(&t.y));
      g[0] = u.x; g[1] = u.y; g[2] = v.x; g[3] = v.y;
    } else if (A.g_dtype == G_F32) {
      g[0] = __uint_as_float(t.x); g[1] = __uint_as_float(t.y); g[2] = __uint_as_float(t.z); g[3] = __uint_as_float(t.w);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_fp8_e4m3 e;
        e.__x = (unsigned char)(t.x >> (8 * j));
        g[j] = (float)e;
      }
    }
    s = fmaf(g[0], x.x, s);
    s = fmaf(g[1], x.y, s);
    s = fmaf(g[2], x.z, s);
    s = fmaf(g[3], x.w, s);
  }
  if (A.g_dtype == G_E4M3) s *= __ldg(A.g_scale + r);
  return eng::wsum((double)s);
}

extern "C" __global__ void __launch_bounds__(kNT, 1) bitplane_gemv_kernel(const Args A) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Ctl& c = *reinterpret_cast<Ctl*>(smem_raw);
  const unsigned char* dyn0 = smem_raw;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  const long long T = (long long)A.n_win * A.n_tiles;
  const int t0 = (int)(T * cta / G), t1 = (int)(T * (cta + 1) / G), nt = t1 - t0;
  const bool dyn = A.l != A.h;
  // chunk groups: <= kGT consecutive tiles of one window
  const int w0 = nt > 0 ? t0 / A.n_tiles : 0;
  const int e0 = min(t1, (w0 + 1) * A.n_tiles);
  const int ng0 = (e0 - t0 + kGT - 1) / kGT, ng = ng0 + (t1 - e0 + kGT - 1) / kGT;
  auto group = [&](int g, int& start, int& n) {
    if (g < ng0) { start = t0 + g * kGT; n = min(kGT, e0 - start); }
    else { start = e0 + (g - ng0) * kGT; n = min(kGT, t1 - start); }
  };
  if (tid == 0) GV_STAMP(0);
  if (warp == kCW) {
    // ring slots below LUT 0 (after Ctl) and above LUT 1's zero row; the
    // producer warp's lanes set them up in parallel
    const uint32_t base = smem_u32(smem_raw);
    const uint32_t lo = (base + (uint32_t)sizeof(Ctl) + 127u) & ~127u;
    const int n_lo = lo + kChunk <= kLut0 ? (int)((kLut0 - lo) / kChunk) : 0;
    const uint32_t hi = kLut0 + 0x10000u + kLutBytes;
    uint32_t end;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(end));
    end += base;
    if (n_lo + (int)((end - hi) / kChunk) < kSlots) __trap();
    for (int q = lane; q < kSlots; q += 32) {
      c.slot_off[q] = (q < n_lo ? lo + q * kChunk : hi + (q - n_lo) * kChunk) - base;
      eng::mbar_init(&c.full[q], 1);
      eng::mbar_init(&c.empty[q], kGT);
      c.seq[q] = -1;
    }
    if (lane == 0) c.dec_bit = dyn ? -1 : A.l;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // programmatic dependent launch: the next call's grid may be scheduled now
  // (its CTAs take an SM as this grid's CTAs exit and stream their weights);
  // everything that reads the previous call's results (x, the scratch sums)
  // waits for it below (griddepcontrol.wait)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (tid == 0) GV_STAMP(1);
  if (warp == kCW) {
    // ---- TMA producer (lane 0): base planes 0..l-1 of every group, then (high) l..h-1
    const unsigned long long pol = eng::l2_evict_first_policy();
    // FIFO order: waves of kQuads groups, plane-major inside a wave, so every
    // quad streams its group's planes concurrently (chunk (g, plane p of a
    // phase of np planes) = jb + wave kQuads np + p n_wave + g mod kQuads)
    auto issue = [&](int g, int p, int j) {
      int start, nn;
      group(g, start, nn);
      const int w = start / A.n_tiles, t = start - w * A.n_tiles;
      const unsigned char* src =
          reinterpret_cast<const unsigned char*>(A.planes + ((long long)w * A.n_tiles + t) * (kItem / 16));
      const int sl = j % kSlots;
      if (j >= kSlots)
        SPIN_UNTIL_NS(eng::mbar_test(smem_u32(&c.empty[sl]), (unsigned)(((j / kSlots) - 1) & 1)), "gemv producer",
                      j, 0, 4000000000ull);
      c.seq[sl] = j;
      GV_CHUNK(j, 0);
      eng::mbar_expect_tx(&c.full[sl], (unsigned)(nn * kItem));
      eng::tma_load_1d(const_cast<unsigned char*>(dyn0) + c.slot_off[sl], src + (long long)p * A.pstride16 * 16,
                       (unsigned)(nn * kItem), &c.full[sl], pol);
    };
    // lane l < kSlots issues the chunks j = l (mod kSlots), i.e. owns ring
    // slot j mod kSlots: the lanes refill their slots independently.
    // FIFO layout (chunk index of (group g = wave v, quad qd; plane pp)):
    //   wave 0, base planes:            pp n0 + qd                      (pp < l)
    //   waves v >= 1, all f planes:     B0 + (v - 1) kQuads f + pp nwv + qd
    //   wave 0, extra planes:           B0 + (ng - n0) f + pp n0 + qd   (pp < f - l)
    // with n0 = min(kQuads, ng), B0 = n0 l and f the decided bit (static: l):
    // only wave 0 is streamed before the decision, the extra planes of later
    // waves follow their base planes.
    const int n0 = min(kQuads, ng), B0 = n0 * A.l;
    auto chunk_of = [&](int r, int f, int& g, int& pp) {
      if (r < B0) { pp = r / n0; g = r - pp * n0; return; }
      const int rb = r - B0, nb = (ng - n0) * f;
      if (rb < nb) {
        const int v = 1 + rb / (kQuads * f), rr = rb - (v - 1) * kQuads * f;
        const int nwv = min(kQuads, ng - v * kQuads);
        pp = rr / nwv;
        g = v * kQuads + (rr - pp * nwv);
        return;
      }
      const int re = rb - nb;
      pp = A.l + re / n0;
      g = re - (pp - A.l) * n0;
    };
    auto run = [&](int r0, int r1, int f, bool release) {
      if (lane < kSlots && r0 + lane < r1) {
        int g, pp;
        chunk_of(r0 + lane, f, g, pp);
        issue(g, pp, r0 + lane);
      }
      __syncwarp();
      // the first ring-full is in flight: the consumers' LUT stores may now
      // take the shared-memory pipe (warp-uniform: bar.arrive counts the warp)
      if (release) asm volatile("bar.arrive 2, %0;" :: "n"(kNT) : "memory");
      if (lane < kSlots)
        for (int r = r0 + lane + kSlots; r < r1; r += kSlots) {
          int g, pp;
          chunk_of(r, f, g, pp);
          issue(g, pp, r);
        }
      __syncwarp();
    };
    if (!dyn) {
      run(0, ng * A.l, A.l, true);
      if (lane == 0) GV_STAMP(2);
      return;
    }
    run(0, B0, A.l, true);                 // wave 0's base planes, then the decision
    if (lane == 0) GV_STAMP(2);
    // the decision: every CTA from the same fixed-point sums
    int bit = A.sentinel == 2 ? A.h : A.l;
    double est = CUDART_NAN;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (A.sentinel == 0) {
      const int n_jobs = A.n_win * (A.est_kind == EST_PROJECTION ? A.k : 1);
      if (lane == 0) SPIN_UNTIL(eng::ld_acq_s32(A.sync) >= n_jobs, "gemv estimator", n_jobs, 0);
      __syncwarp();
      double q = 0.0, sq = 0.0;
      if (A.est_kind == EST_PROJECTION)
        for (int r = lane; r < A.k; r += 32) {
          const double gv = (double)__ldcg(A.acc + r) * A.fbscale;
          q += gv * gv;
        }
      for (int w = lane; w < A.n_win; w += 32) sq += __ldcg(A.sq + w);
      q = eng::wsum(q);
      sq = eng::wsum(sq);
      if (A.est_kind == EST_PROJECTION) est = q > 0.0 ? q * eng::rsqrt_d(q) : 0.0;              // estimator.py:56-57
      else est = A.slope * (sq > 0.0 ? sq * eng::rsqrt_d(sq) : 0.0) + A.intercept;           // estimator.py:41-42
      bit = est > A.T ? A.h : A.l;                                                           // runtime.py:192
    }
    if (lane == 0) {                         // the decision first (the consumers wait for it)
      c.dec_bit = bit;
      GV_STAMP(5);
      if (cta == 0) {
        if (A.bit_out) *A.bit_out = bit;
        if (A.est_out) *A.est_out = (float)est;
      }
      // then the last CTA past this point clears the sums for the next call
      // (acq_rel: this CTA's reads of the sums before its count)
      if (A.sentinel == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(A.sync + 1) : "memory");
        if (old == (unsigned)G - 1) {
          for (int r = 0; r < A.k; ++r) A.acc[r] = 0;
          A.sync[0] = 0;
          A.sync[1] = 0;
        }
      }
    }
    __syncwarp();
    run(B0, ng * bit, bit, false);         // the rest: B0 + (ng - n0) f + n0 (f - l) = ng f
    return;
  }
  // ---- consumers
  if (nt <= 0) return;
  const bool jobs = dyn && A.sentinel == 0;
  constexpr int kHalf = kNC / 2;
  constexpr int kPre = 2;                // estimator jobs per warp with the G row loaded ahead
  const int kk = A.est_kind == EST_PROJECTION ? A.k : 1;
  const long long J = (long long)A.n_win * kk;
  const int jj0 = (int)(J * cta / G), jj1 = (int)(J * (cta + 1) / G);
  const int jw = warp - kHalf / 32, nj = kCW - kHalf / 32;
  GPre gpre[kPre];
  if (jobs && tid >= kHalf && A.est_kind == EST_PROJECTION)
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
      const int j = jj0 + jw + u * nj;
      if (j < jj1) gpre_load(A, j / kk, j - (j / kk) * kk, gpre[u]);
    }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int nw = (t1 - 1) / A.n_tiles - w0 + 1;   // <= 2 (host-checked)
  // input windows -> shared memory, window sums of x (and x^2 for the estimator)
  if (tid < 128 * nw) {
    const int i = tid >> 7, w = w0 + i, c0 = w * kWinCols + 4 * (tid & 127);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c0 + 4 <= A.cols) v = __ldg(reinterpret_cast<const float4*>(A.x + c0));
    else
      for (int j = 0; j < 4; ++j)
        if (c0 + j < A.cols) (&v.x)[j] = __ldg(A.x + c0 + j);
    *reinterpret_cast<float4*>(c.xw[i] + 4 * (tid & 127)) = v;
  }
  // The window LUTs and, for a selector, the estimator jobs (w, r) of this
  // CTA (w-major over n_win x k for a projection, one job per window for the
  // linear estimator): jobs on the upper half of the consumer warps, the LUTs
  // on the lower half, which stream as soon as their LUTs are built (bar 3
  // among themselves, bar 4 released to the job warps).
  GV_SYNC();                                   // xw staged
  asm volatile("bar.sync 2, %0;" :: "n"(kNT) : "memory");   // the producer's first ring-full issued
  if (tid == 0) GV_STAMP(3);
  float* lut0 = reinterpret_cast<float*>(smem_raw + (kLut0 - smem_u32(smem_raw)));
  if (!jobs || tid < kHalf) {
    const int nthr = jobs ? kHalf : kNC;
    for (int i = 0; i < nw; ++i) lut_build(lut0 + i * (0x10000 / 4), c.xw[i], tid, nthr);
    if (tid < 32 * nw) {                   // window sums of x (epilogue), identical on every CTA
      const int i = tid >> 5;
      float s = 0.f;
#pragma unroll
      for (int q = 0; q < 16; ++q) s += c.xw[i][lane + 32 * q];
      s = eng::wsum(s);
      if (lane == 0) A.sx[w0 + i] = s;
    }
    if (tid < 64) {                         // zero rows 256 of both LUTs (LUT 0's is LUT 1's row 0)
      lut0[256 * kGroups + tid] = 0.f;
      lut0[256 * kGroups + 0x10000 / 4 + tid] = 0.f;
    }
    if (jobs) {
      asm volatile("bar.sync 3, %0;" :: "n"(kHalf) : "memory");
      asm volatile("bar.arrive 4, %0;" :: "n"(kNC) : "memory");
    } else {
      GV_SYNC();
    }
  } else {
    int mine = 0;
    for (int j = jj0 + jw, u = 0; j < jj1; j += nj, ++u) {
      const int w = j / kk, r = j - w * kk;
      if (A.est_kind == EST_PROJECTION) {
        GPre gp;
        if (u == 0) gp = gpre[0];
        else if (u == 1) gp = gpre[1];
        else gpre_load(A, w, r, gp);
        const double v = g_row_dot(A, w, r, gp) * A.fxscale;
        if (lane == 0) {
          long long f = 0;
          if (fabs(v) < 4.5e15) f = llrint(v);
          else atomicOr(A.err, 1u);
          atomicAdd(reinterpret_cast<unsigned long long*>(A.acc + r), (unsigned long long)f);
        }
      }
      if (r == 0) {                        // the window's sum x^2 (the linear estimator's ||x||)
        double q = 0.0;
        for (int cc = lane; cc < kWinCols; cc += 32) {
          const int col = w * kWinCols + cc;
          const double xv = col < A.cols ? (double)__ldg(A.x + col) : 0.0;
          q += xv * xv;
        }
        q = eng::wsum(q);
        if (lane == 0) A.sq[w] = q;
      }
      ++mine;
    }
    if (mine && lane == 0)           // release: this lane's acc red.adds before the count
      asm volatile("red.release.gpu.global.add.s32 [%0], %1;" :: "l"(A.sync), "r"(mine) : "memory");
    asm volatile("bar.sync 4, %0;" :: "n"(kNC) : "memory");   // the LUTs are built
  }
  if (tid == 0) GV_STAMP(4);
  const int rpad = A.n_tiles * 32;
  // a tile's window partial is final: count it; the tile's last window applies
  // the epilogue (quant.py:74-78) over the window partials in window order
  auto arrive = [&](int t, int bit) {
    __syncwarp();
    int last = 0;
#if DPQ_GV_ACQREL
    if (lane == 0) {           // one acq_rel atomic: the warp's partials before the count, and
      int old;                 // (last window) the other windows' partials after it
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(A.cnt + t) : "memory");
      last = old == A.n_win - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __syncwarp();
#else
    if (lane == 0) {
      __threadfence();
      last = atomicAdd(A.cnt + t, 1) == A.n_win - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();
#endif
    double Sd = 0.0, sx = 0.0;
    for (int v = 0; v < A.n_win; ++v) {
      Sd += (double)__ldcg(A.part + (size_t)v * rpad + t * 32 + lane);
      sx += (double)__ldcg(A.sx + v);
    }
    const int r = t * 32 + lane;
    if (r < A.rows) {
      const float lo = __ldg(A.lo + r), sp = __ldg(A.span + r);
      A.y[r] = (float)((double)lo * sx + ldexp((double)sp, -bit) * (Sd + 0.5 * sx));
    }
    if (lane == 0) A.cnt[t] = 0;
    if (lane == 0) GV_STAMP(7);
  };
  // warp i of quad q: tile i of the groups q, q + kQuads, ... (FIFO layout:
  // see the producer). Wave 0: the base planes (the decision may be pending);
  // later waves: all decided planes in one Horner pass; then wave 0's extras.
  const int q = warp / kGT, i = warp % kGT;
  const int n0 = min(kQuads, ng), B0 = n0 * A.l;
  int bit = A.l;
  for (int g = q; g < ng; g += kQuads) {
    int start, n;
    group(g, start, n);
    const int w = start / A.n_tiles, t = start - w * A.n_tiles + i;
    const uint32_t lanereg = (kLut0 << (w - w0)) | ((uint32_t)lane * 4u);
    const int v = g / kQuads, nwv = min(kQuads, ng - v * kQuads);
    float S;
    if (v == 0) {
      S = stream_items(c, dyn0, g, A.l, n0, i, i < n, lanereg);
    } else {
      if (dyn && v == 1) {                 // (first later wave of this quad) the decision
        if (lane == 0) SPIN_UNTIL(c.dec_bit >= 0, "gemv decision", 0, 0);
        __syncwarp();
        bit = c.dec_bit;
      }
      S = stream_items(c, dyn0, B0 + (v - 1) * kQuads * bit + (g - v * kQuads), bit, nwv, i, i < n, lanereg);
    }
    if (i < n) {
      A.part[(size_t)w * rpad + t * 32 + lane] = S;
      if (!dyn || v > 0) arrive(t, bit);
    }
  }
  if (lane == 0) GV_STAMP(6);
  if (!dyn || q >= n0) return;
  // wave 0 (group q): its extra planes, then the tile's partial is final
  if (lane == 0) SPIN_UNTIL(c.dec_bit >= 0, "gemv decision", 0, 0);
  __syncwarp();
  bit = c.dec_bit;
  int start, n;
  group(q, start, n);
  const int w = start / A.n_tiles, t = start - w * A.n_tiles + i;
  if (bit > A.l) {                         // S_h = 2^(h-l) S_l + the extra planes' Horner sum
    const uint32_t lanereg = (kLut0 << (w - w0)) | ((uint32_t)lane * 4u);
    const int ne = bit - A.l;
    const float Sx = stream_items(c, dyn0, B0 + (ng - n0) * bit + q, ne, n0, i, i < n, lanereg);
    if (i < n) {
      float* pp = A.part + (size_t)w * rpad + t * 32 + lane;
      *pp = ldexpf(*pp, ne) + Sx;
    }
  }
  if (i < n) arrive(t, bit);
}

}  // namespace gv
}  // namespace dpq
