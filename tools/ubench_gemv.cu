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
template <int NT, int DEPTH>
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
          const float P = plane_task(buf[d][0], buf[d][1], buf[d][2], buf[d][3], lanereg);
          const int j = it / b, p = it - j * b;
          S = 2.f * S + P;
          if (p == b - 1) {
            const int t = t0 + warp + NW * j;
            slots[(long long)w * n_tiles * 32 + t * 32 + lane] = S;
            S = 0.f;
          }
          if (it + DEPTH < n_items) {
            const uint4* s = src(it + DEPTH);
            buf[d][0] = ldg_stream(s); buf[d][1] = ldg_stream(s + 32);
            buf[d][2] = ldg_stream(s + 64); buf[d][3] = ldg_stream(s + 96);
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

template <int NT, int DEPTH>
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
  CK(cudaFuncSetAttribute(core_kernel<NT, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 3 * ncopy; ++i)
    core_kernel<NT, DEPTH><<<grid, NT, smem>>>(P[i % ncopy], plane_bytes / 16, n_win, n_tiles, b, x, slots);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i)
    core_kernel<NT, DEPTH><<<grid, NT, smem>>>(P[i % ncopy], plane_bytes / 16, n_win, n_tiles, b, x, slots);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double t = ms / reps * 1e-3;
  const double bytes = (double)plane_bytes * b;
  printf("%-10s NT=%4d D=%d grid=%4d %6dx%-6d b=%d  %8.2f us  %7.1f GB/s\n", name, NT, DEPTH, grid, rows, cols, b,
         t * 1e6, bytes / t / 1e9);
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
  const int reps = 200;
  // big op shapes: upgate (28672x4096), down (4096x14336), qkv (6144x4096), o (4096x4096)
  struct Sh { const char* n; int r, c, nc; } shapes[] = {
      {"upgate", 28672, 4096, 6}, {"down", 4096, 14336, 10}, {"qkv", 6144, 4096, 24}, {"o", 4096, 4096, 32}};
  for (auto& s : shapes) {
    for (int b : {3, 4}) {
      run_core<512, 2>(s.n, s.r, s.c, b, 4, s.nc, nsm, reps);
      run_core<512, 3>(s.n, s.r, s.c, b, 4, s.nc, nsm, reps);
      run_core<512, 4>(s.n, s.r, s.c, b, 4, s.nc, nsm, reps);
      run_core<1024, 2>(s.n, s.r, s.c, b, 4, s.nc, nsm, reps);
    }
  }
  return 0;
}
