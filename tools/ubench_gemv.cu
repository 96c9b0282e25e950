// Microbenchmark of the bitplane byte-LUT GEMV core on one B200 (no
// reduction, no selector): how close does the inner loop get to HBM peak?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o ubench tools/ubench_gemv.cu
//   ./ubench
//
// Layout (same as the library): plane p, window w (512 cols), tile t (32
// rows) = 2 KB = [chunk c][lane l][16 B]; lane l's 64 bytes are the 64 steps.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int kWin = 512, kGroups = 64, kTileBytes = 2048;
constexpr uint32_t kLutShared = 0x10000;
constexpr int kLutBytes = 257 * 64 * 4;

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
#define LDS(dst, addr, IMM) asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(dst) : "r"(addr), "n"(IMM))

__device__ __forceinline__ float plane_task(const uint4 d0, const uint4 d1, const uint4 d2, const uint4 d3,
                                            uint32_t lanereg) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#define WORD(W, S0)                                             \
  {                                                             \
    float v0, v1, v2, v3;                                       \
    LDS(v0, __byte_perm((W), lanereg, 0x7604u), 4 * (S0 + 0));  \
    LDS(v1, __byte_perm((W), lanereg, 0x7614u), 4 * (S0 + 1));  \
    LDS(v2, __byte_perm((W), lanereg, 0x7624u), 4 * (S0 + 2));  \
    LDS(v3, __byte_perm((W), lanereg, 0x7634u), 4 * (S0 + 3));  \
    a0 += v0; a1 += v1; a2 += v2; a3 += v3;                     \
  }
  WORD(d0.x, 0) WORD(d0.y, 4) WORD(d0.z, 8) WORD(d0.w, 12)
  WORD(d1.x, 16) WORD(d1.y, 20) WORD(d1.z, 24) WORD(d1.w, 28)
  WORD(d2.x, 32) WORD(d2.y, 36) WORD(d2.z, 40) WORD(d2.w, 44)
  WORD(d3.x, 48) WORD(d3.y, 52) WORD(d3.z, 56) WORD(d3.w, 60)
#undef WORD
  return (a0 + a1) + (a2 + a3);
}

template <int NT>
__device__ __forceinline__ void build_lut(float* lut, const float* xw) {
  // thread -> group g = tid & 63, rows blocks of 256 / (NT / 64)
  constexpr int RB = NT / 64;
  constexpr int ROWS = 256 / RB;
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
  float xh[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) xh[t] = xg[4 + t];
#pragma unroll
  for (int hh = 0; hh < ROWS / 16; ++hh) {
    const int m = (ROWS / 16) * rb + hh;
    float H = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) if (m & (1 << t)) H += xh[t];
#pragma unroll
    for (int i = 0; i < 16; ++i) lut[(16 * m + i) * kGroups + g] = L[i] + H;
  }
  if (rb == 0) lut[256 * kGroups + g] = 0.f;
}

// Each CTA: balanced contiguous range of groups (window-major), all b planes.
template <int NT, int DEPTH, int MODE = 0>
__global__ void __launch_bounds__(NT, 1)
core_kernel(const uint4* __restrict__ planes, long long plane_stride16, int n_win, int n_tiles, int b,
            const float* __restrict__ x, float* __restrict__ slots) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ float xw[kWin];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  float* lut = reinterpret_cast<float*>(smem + (kLutShared - sbase));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const long long N = (long long)n_win * n_tiles;
  const long long g0 = N * blockIdx.x / gridDim.x, g1 = N * (blockIdx.x + 1) / gridDim.x;
  const uint32_t lanereg = kLutShared | ((uint32_t)lane * 4u);
  long long g = g0;
  while (g < g1) {
    const int w = (int)(g / n_tiles);
    const long long seg_end = min(g1, (long long)(w + 1) * n_tiles);
    __syncthreads();
    for (int i = tid; i < kWin; i += NT) xw[i] = x[w * kWin + i];
    __syncthreads();
    build_lut<NT>(lut, xw);
    __syncthreads();
    // warp items: groups g + warp + NW*j, planes 0..b-1
    const int t0 = (int)(g - (long long)w * n_tiles);
    const int nseg = (int)(seg_end - g);
    const int my_groups = nseg > warp ? (nseg - warp + NW - 1) / NW : 0;
    const int n_items = my_groups * b;
    uint4 buf[DEPTH][4];
    auto src = [&](int it) {
      const int j = it / b, p = it - j * b;
      const int t = t0 + warp + NW * j;
      return planes + p * plane_stride16 + ((long long)w * n_tiles + t) * (kTileBytes / 16) + lane;
    };
#pragma unroll
    for (int d = 0; d < DEPTH; ++d)
      if (d < n_items) {
        const uint4* s = src(d);
        buf[d][0] = ldg_stream(s); buf[d][1] = ldg_stream(s + 32);
        buf[d][2] = ldg_stream(s + 64); buf[d][3] = ldg_stream(s + 96);
      }
    float S = 0.f;
    for (int it0 = 0; it0 < n_items; it0 += DEPTH) {
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) {
        const int it = it0 + d;
        if (it < n_items) {
          float P;
          if (MODE == 1) {
            const unsigned xx = buf[d][0].x ^ buf[d][1].y ^ buf[d][2].z ^ buf[d][3].w ^ buf[d][0].y ^ buf[d][1].z;
            P = __uint_as_float(xx & 0x3f800000u);
          } else {
            P = plane_task(buf[d][0], buf[d][1], buf[d][2], buf[d][3], lanereg);
          }
          const int j = it / b, p = it - j * b;
          S = 2.f * S + P;
          if (p == b - 1) {
            const int t = t0 + warp + NW * j;
            slots[(long long)w * n_tiles * 32 + t * 32 + lane] = S;
            S = 0.f;
          }
          if (it + DEPTH < n_items) {
            if (MODE == 2) {
              buf[d][0].x += 0x01010101u; buf[d][1].y += 0x01010101u; buf[d][2].z ^= 0x03030303u; buf[d][3].w ^= (unsigned)it;
            } else {
              const uint4* s = src(it + DEPTH);
              buf[d][0] = ldg_stream(s); buf[d][1] = ldg_stream(s + 32);
              buf[d][2] = ldg_stream(s + 64); buf[d][3] = ldg_stream(s + 96);
            }
          }
        }
      }
    }
    g = seg_end;
  }
}

__global__ void stream_kernel(const uint4* __restrict__ p, long long n16, unsigned* out) {
  unsigned acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = ldg_stream(p + i), b2 = ldg_stream(p + i + stride), c = ldg_stream(p + i + 2 * stride),
          d = ldg_stream(p + i + 3 * stride);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b2.x ^ b2.y ^ b2.z ^ b2.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
  }
  for (; i < n16; i += stride) { uint4 a = ldg_stream(p + i); acc ^= a.x ^ a.y ^ a.z ^ a.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int NT, int DEPTH, int MODE = 0>
void run_core(const char* name, int rows, int cols, int b, int n_bits, int ncopy, int grid, int reps) {
  const int n_win = cols / kWin, n_tiles = rows / 32;
  const long long plane_bytes = (long long)n_win * n_tiles * kTileBytes;
  const long long layer_bytes = plane_bytes * n_bits;
  std::vector<uint4*> P(ncopy);
  for (int i = 0; i < ncopy; ++i) {
    CK(cudaMalloc(&P[i], layer_bytes));
    CK(cudaMemset(P[i], 0x5a + i, layer_bytes));
  }
  float *x, *slots;
  CK(cudaMalloc(&x, cols * 4));
  CK(cudaMemset(x, 0, cols * 4));
  CK(cudaMalloc(&slots, (size_t)n_win * rows * 4));
  const int smem = (int)kLutShared + kLutBytes;
  CK(cudaFuncSetAttribute(core_kernel<NT, DEPTH, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 3 * ncopy; ++i)
    core_kernel<NT, DEPTH, MODE><<<grid, NT, smem>>>(P[i % ncopy], plane_bytes / 16, n_win, n_tiles, b, x, slots);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i)
    core_kernel<NT, DEPTH, MODE><<<grid, NT, smem>>>(P[i % ncopy], plane_bytes / 16, n_win, n_tiles, b, x, slots);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double t = ms / reps * 1e-3;
  const double bytes = (double)plane_bytes * b;
  printf("%-10s M%d NT=%4d D=%d grid=%4d %6dx%-6d b=%d  %8.2f us  %7.1f GB/s\n", name, MODE, NT, DEPTH, grid, rows, cols, b,
         t * 1e6, bytes / t / 1e9);
  for (auto p : P) cudaFree(p);
  cudaFree(x);
  cudaFree(slots);
}


// ---- TMA variant: warp 0 lane 0 streams items (group, plane) with 1D bulk
// copies into a STAGES-deep shared-memory ring (mbarrier full / empty);
// consumer warps own groups and read their 64 B per lane with LDS.128.
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned ok = 0;
  long long t0 = clock64();
  while (!ok) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(a), "r"(phase) : "memory");
    if (clock64() - t0 > 4000000000LL) { printf("mbar timeout block %d thread %d phase %u\n", blockIdx.x, threadIdx.x, phase); __trap(); }
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                  "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

template <int NT, int STAGES>
__global__ void __launch_bounds__(NT, 1)
core_tma_kernel(const uint4* __restrict__ planes, long long plane_stride16, int n_win, int n_tiles, int b,
                const float* __restrict__ x, float* __restrict__ slots) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ float xw[kWin];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  __shared__ volatile int seq[STAGES];      // item index armed in each slot (disambiguates phase parity)
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  float* lut = reinterpret_cast<float*>(smem + (kLutShared - sbase));
  unsigned char* ring = smem + (kLutShared - sbase) + kLutBytes;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32, NC = NW - 1;
  const long long N = (long long)n_win * n_tiles;
  const long long g0 = N * blockIdx.x / gridDim.x, g1 = N * (blockIdx.x + 1) / gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); seq[s] = -1; }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int n_items_all = (int)(g1 - g0) * b;
  if (warp == 0) {
    // producer: items in (group, plane) order; single window assumed per CTA segment
    if (lane == 0) {
      for (int j = 0; j < n_items_all; ++j) {
        const int s = j % STAGES;
        if (j >= STAGES) mbar_wait(&empty[s], ((j / STAGES) - 1) & 1);
        const long long g = g0 + j / b;
        const int p = j % b;
        const int w = (int)(g / n_tiles), t = (int)(g - (long long)w * n_tiles);
        seq[s] = j;
        mbar_expect_tx(&full[s], kTileBytes);
        tma_load_1d(ring + s * kTileBytes, planes + p * plane_stride16 + ((long long)w * n_tiles + t) * (kTileBytes / 16),
                    kTileBytes, &full[s]);
      }
    }
    return;
  }
  // consumers: LUT of the first window (benchmark: ranges rarely span two)
  const int w0 = (int)(g0 / n_tiles);
  for (int i = tid - 32; i < kWin; i += NT - 32) xw[i] = x[w0 * kWin + i];
  asm volatile("bar.sync 1, %0;" :: "r"(NT - 32));
  for (int u = tid - 32; u < 512; u += NT - 32) {
    const int g = u & 63, rb = u >> 6;
    const float* xg = xw + 8 * g;
    float L[16];
    L[0] = 0.f;
#pragma unroll
    for (int n = 1; n < 16; ++n) { const int low = n & (-n); L[n] = L[n ^ low] + xg[__ffs(low) - 1]; }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int m = 2 * rb + hh;
      float H = 0.f;
      for (int t2 = 0; t2 < 4; ++t2) if (m & (1 << t2)) H += xg[4 + t2];
#pragma unroll
      for (int i = 0; i < 16; ++i) lut[(16 * m + i) * kGroups + g] = L[i] + H;
    }
    if (rb == 0) lut[256 * kGroups + g] = 0.f;
  }
  asm volatile("bar.sync 1, %0;" :: "r"(NT - 32));
  const uint32_t lanereg = kLutShared | ((uint32_t)lane * 4u);
  const int cw = warp - 1;
  for (long long g = g0 + cw; g < g1; g += NC) {
    float S = 0.f;
    const int jg = (int)(g - g0) * b;
    for (int p = 0; p < b; ++p) {
      const int j = jg + p, s = j % STAGES;
      while (seq[s] != j) {}
      mbar_wait(&full[s], (j / STAGES) & 1);
      const uint4* q = reinterpret_cast<const uint4*>(ring + s * kTileBytes) + lane;
      const uint4 d0 = q[0], d1 = q[32], d2 = q[64], d3 = q[96];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      S = 2.f * S + plane_task(d0, d1, d2, d3, lanereg);
    }
    const int w = (int)(g / n_tiles), t = (int)(g - (long long)w * n_tiles);
    slots[(long long)w * n_tiles * 32 + t * 32 + lane] = S;
  }
}

// ---- TMA v2: producer streams (8-tile chunk, plane) items of up to 16 KB
// (contiguous tiles of one plane) into an NSLOT ring; consumer warp (c*8+i) % NC
// handles tile i of chunk c over all b planes (Horner in registers).
template <int NT, int NSLOT>
__global__ void __launch_bounds__(NT, 1)
core_tma2_kernel(const uint4* __restrict__ planes, long long plane_stride16, int n_win, int n_tiles, int b,
                 const float* __restrict__ x, float* __restrict__ slots) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ float xw[kWin];
  __shared__ uint64_t full[NSLOT], empty[NSLOT];
  __shared__ volatile int seq[NSLOT];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  // LUT at 0x20000, ring below it (from the dynamic base) and above it
  float* lut = reinterpret_cast<float*>(smem + (0x20000u - sbase));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32, NC = NW - 1;
  const long long N = (long long)n_win * n_tiles;
  const long long g0 = N * blockIdx.x / gridDim.x, g1 = N * (blockIdx.x + 1) / gridDim.x;
  const int ng = (int)(g1 - g0);
  const int n_chunks = (ng + 7) / 8;
  auto slot_ptr = [&](int s) -> unsigned char* {
    const uint32_t lo_room = (0x20000u - sbase) / 16384u;   // slots below the LUT
    if ((uint32_t)s < lo_room) return smem + s * 16384;
    return smem + (0x20000u - sbase) + 257 * 256 + (s - lo_room) * 16384;
  };
  if (tid == 0) {
    for (int q = 0; q < NSLOT; ++q) { mbar_init(&full[q], 1); mbar_init(&empty[q], 8); seq[q] = -1; }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      int j = 0;
      for (int c = 0; c < n_chunks; ++c) {
        const long long ga = g0 + 8 * c;
        const int nt = (int)min(8LL, g1 - ga);
        const int w = (int)(ga / n_tiles), t = (int)(ga - (long long)w * n_tiles);
        for (int p = 0; p < b; ++p, ++j) {
          const int q = j % NSLOT;
          if (j >= NSLOT) mbar_wait(&empty[q], ((j / NSLOT) - 1) & 1);
          seq[q] = j;
          mbar_expect_tx(&full[q], nt * kTileBytes);
          tma_load_1d(slot_ptr(q), planes + p * plane_stride16 + ((long long)w * n_tiles + t) * (kTileBytes / 16),
                      nt * kTileBytes, &full[q]);
        }
      }
    }
    return;
  }
  const int w0 = (int)(g0 / n_tiles);
  for (int i = tid - 32; i < kWin; i += NT - 32) xw[i] = x[w0 * kWin + i];
  asm volatile("bar.sync 1, %0;" :: "r"(NT - 32));
  for (int u = tid - 32; u < 512; u += NT - 32) {
    const int g = u & 63, rb = u >> 6;
    const float* xg = xw + 8 * g;
    float L[16];
    L[0] = 0.f;
#pragma unroll
    for (int n = 1; n < 16; ++n) { const int low = n & (-n); L[n] = L[n ^ low] + xg[__ffs(low) - 1]; }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int m = 2 * rb + hh;
      float H = 0.f;
      for (int t2 = 0; t2 < 4; ++t2) if (m & (1 << t2)) H += xg[4 + t2];
#pragma unroll
      for (int i = 0; i < 16; ++i) lut[(16 * m + i) * kGroups + g] = L[i] + H;
    }
    if (rb == 0) lut[256 * kGroups + g] = 0.f;
  }
  asm volatile("bar.sync 1, %0;" :: "r"(NT - 32));
  const uint32_t lanereg = 0x20000u | ((uint32_t)lane * 4u);
  const int cw = warp - 1;
  // my (chunk, tile) pairs: k = c*8 + i with k % NC == cw
  for (int k = cw; k < ng; k += NC) {
    const int c = k >> 3, i = k & 7;
    const int nt = min(8, ng - 8 * c);
    float S = 0.f;
    for (int p = 0; p < b; ++p) {
      const int j = c * b + p, q = j % NSLOT;
      while (seq[q] != j) {}
      mbar_wait(&full[q], (j / NSLOT) & 1);
      const uint4* d = reinterpret_cast<const uint4*>(slot_ptr(q) + i * kTileBytes) + lane;
      const uint4 d0 = d[0], d1 = d[32], d2 = d[64], d3 = d[96];
      __syncwarp();
      // 8 arrivals free the slot: one per tile, the last tile of a partial chunk adds the rest
      if (lane == 0) {
        const unsigned cnt = (i == nt - 1) ? (unsigned)(9 - nt) : 1u;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&empty[q])), "r"(cnt) : "memory");
      }
      S = 2.f * S + plane_task(d0, d1, d2, d3, lanereg);
    }
    const long long g = g0 + k;
    const int w = (int)(g / n_tiles), t = (int)(g - (long long)w * n_tiles);
    slots[(long long)w * n_tiles * 32 + t * 32 + lane] = S;
  }
}

template <int NT, int STAGES, int V2 = 0>
void run_tma(const char* name, int rows, int cols, int b, int n_bits, int ncopy, int reps) {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int n_win = cols / kWin, n_tiles = rows / 32;
  const long long plane_bytes = (long long)n_win * n_tiles * kTileBytes;
  const long long layer_bytes = plane_bytes * n_bits;
  std::vector<uint4*> P(ncopy);
  for (int i = 0; i < ncopy; ++i) {
    CK(cudaMalloc(&P[i], layer_bytes));
    CK(cudaMemset(P[i], 0x5a + i, layer_bytes));
  }
  float *x, *slots;
  CK(cudaMalloc(&x, cols * 4));
  CK(cudaMemset(x, 0, cols * 4));
  CK(cudaMalloc(&slots, (size_t)n_win * rows * 4));
  const int smem = V2 ? 232448 - 4096 : (int)kLutShared + kLutBytes + STAGES * kTileBytes;
  auto kern = V2 ? core_tma2_kernel<NT, STAGES> : core_tma_kernel<NT, STAGES>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 3 * ncopy; ++i)
    kern<<<nsm, NT, smem>>>(P[i % ncopy], plane_bytes / 16, n_win, n_tiles, b, x, slots);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i)
    kern<<<nsm, NT, smem>>>(P[i % ncopy], plane_bytes / 16, n_win, n_tiles, b, x, slots);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double t = ms / reps * 1e-3;
  printf("%-10s TMA%d NT=%4d STAGES=%d %6dx%-6d b=%d copies=%d  %8.2f us  %7.1f GB/s\n", name, V2 + 1, NT, STAGES, rows, cols, b,
         ncopy, t * 1e6, (double)plane_bytes * b / t / 1e9);
  for (auto p : P) cudaFree(p);
  cudaFree(x);
  cudaFree(slots);
}


int main() {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  // pure streaming reference
  {
    const long long bytes = 1LL << 30;
    uint4* p;
    unsigned* o;
    CK(cudaMalloc(&p, bytes));
    CK(cudaMemset(p, 1, bytes));
    CK(cudaMalloc(&o, 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int grid : {nsm, 2 * nsm, 4 * nsm}) {
      stream_kernel<<<grid, 512>>>(p, bytes / 16, o);
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) stream_kernel<<<grid, 512>>>(p, bytes / 16, o);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("stream grid=%d: %.1f GB/s\n", grid, bytes * 10 / (ms * 1e-3) / 1e9);
    }
    cudaFree(p);
  }
  const int reps = 20;
  // large shapes: steady-state streaming rate (startup amortised)
  run_core<512, 4, 0>("big", 229376, 4096, 3, 4, 1, nsm, reps);
  run_core<512, 4, 1>("big", 229376, 4096, 3, 4, 1, nsm, reps);
  run_tma<384, 9, 1>("big", 229376, 4096, 3, 4, 1, reps);
  run_tma<448, 9, 1>("big", 229376, 4096, 3, 4, 1, reps);
  run_tma<544, 9, 1>("big", 229376, 4096, 3, 4, 1, reps);
  run_tma<672, 9, 1>("big", 229376, 4096, 3, 4, 1, reps);
  run_tma<800, 9, 1>("big", 229376, 4096, 3, 4, 1, reps);
  // one up|gate-sized op (2 x 14336 rows, 3 planes) and a down-sized one, 8 copies (cold in L2)
  run_tma<384, 9, 1>("upgate", 28672, 4096, 3, 4, 8, reps);
  run_tma<544, 9, 1>("upgate", 28672, 4096, 3, 4, 8, reps);
  run_tma<384, 9, 1>("down", 4096, 14336, 3, 4, 8, reps);
  run_tma<544, 9, 1>("down", 4096, 14336, 3, 4, 8, reps);
  return 0;
}
