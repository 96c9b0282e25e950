// Byte-LUT lookup throughput on one B200 SM (no global traffic): how many
// conflict-free LDS.32 lookups per clock per SM does the hot loop sustain?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ubench_lut tools/ubench_lut.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
constexpr uint32_t kLutShared = 0x10000;
constexpr int kLutBytes = 257 * 64 * 4;
#define LDS(dst, addr, IMM) asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(dst) : "r"(addr), "n"(IMM))
#define LDSNV(dst, addr, IMM) asm("ld.shared.f32 %0, [%1+%2];" : "=f"(dst) : "r"(addr), "n"(IMM))

template <bool VOL>
__device__ __forceinline__ float plane_task(const uint4 d0, const uint4 d1, const uint4 d2, const uint4 d3,
                                            uint32_t lanereg) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#define WORD(W, S0)                                                            \
  {                                                                            \
    float v0, v1, v2, v3;                                                      \
    if (VOL) {                                                                 \
      LDS(v0, __byte_perm((W), lanereg, 0x7604u), 4 * (S0 + 0));               \
      LDS(v1, __byte_perm((W), lanereg, 0x7614u), 4 * (S0 + 1));               \
      LDS(v2, __byte_perm((W), lanereg, 0x7624u), 4 * (S0 + 2));               \
      LDS(v3, __byte_perm((W), lanereg, 0x7634u), 4 * (S0 + 3));               \
    } else {                                                                   \
      LDSNV(v0, __byte_perm((W), lanereg, 0x7604u), 4 * (S0 + 0));             \
      LDSNV(v1, __byte_perm((W), lanereg, 0x7614u), 4 * (S0 + 1));             \
      LDSNV(v2, __byte_perm((W), lanereg, 0x7624u), 4 * (S0 + 2));             \
      LDSNV(v3, __byte_perm((W), lanereg, 0x7634u), 4 * (S0 + 3));             \
    }                                                                          \
    a0 += v0; a1 += v1; a2 += v2; a3 += v3;                                    \
  }
  WORD(d0.x, 0) WORD(d0.y, 4) WORD(d0.z, 8) WORD(d0.w, 12)
  WORD(d1.x, 16) WORD(d1.y, 20) WORD(d1.z, 24) WORD(d1.w, 28)
  WORD(d2.x, 32) WORD(d2.y, 36) WORD(d2.z, 40) WORD(d2.w, 44)
  WORD(d3.x, 48) WORD(d3.y, 52) WORD(d3.z, 56) WORD(d3.w, 60)
#undef WORD
  return (a0 + a1) + (a2 + a3);
}

template <bool VOL>
__global__ void lut_kernel(int iters, const uint4* seed, float* out, long long* clk) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  float* lut = reinterpret_cast<float*>(smem + (kLutShared - sbase));
  for (int i = threadIdx.x; i < 257 * 64; i += blockDim.x) lut[i] = (float)(i & 1023) * 1e-3f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t lanereg = kLutShared | ((uint32_t)lane * 4u);
  uint4 d0 = seed[(threadIdx.x * 4 + 0) & 255], d1 = seed[(threadIdx.x * 4 + 1) & 255];
  uint4 d2 = seed[(threadIdx.x * 4 + 2) & 255], d3 = seed[(threadIdx.x * 4 + 3) & 255];
  float acc = 0.f;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    acc += plane_task<VOL>(d0, d1, d2, d3, lanereg);
    const uint32_t m = 0x01010101u * (uint32_t)(i & 7);
    d0.x ^= m; d0.y ^= m; d0.z ^= m; d0.w ^= m; d1.x ^= m; d1.y ^= m; d1.z ^= m; d1.w ^= m;
    d2.x ^= m; d2.y ^= m; d2.z ^= m; d2.w ^= m; d3.x ^= m; d3.y ^= m; d3.z ^= m; d3.w ^= m;
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  uint4* seed;
  CK(cudaMalloc(&seed, 256 * 16));
  uint4 h[256];
  for (int i = 0; i < 256; ++i) h[i] = make_uint4(rand(), rand(), rand(), rand());
  CK(cudaMemcpy(seed, h, sizeof h, cudaMemcpyHostToDevice));
  float* out;
  long long* clk;
  CK(cudaMalloc(&out, nsm * 1024 * 4));
  CK(cudaMalloc(&clk, nsm * 8));
  const int smem = (int)kLutShared + kLutBytes;
  CK(cudaFuncSetAttribute(lut_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(lut_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 2000;
  for (int vol = 0; vol < 2; ++vol)
    for (int nt : {128, 256, 512, 1024}) {
      if (vol) lut_kernel<true><<<nsm, nt, smem>>>(iters, seed, out, clk);
      else lut_kernel<false><<<nsm, nt, smem>>>(iters, seed, out, clk);
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (vol) lut_kernel<true><<<nsm, nt, smem>>>(iters, seed, out, clk);
      else lut_kernel<false><<<nsm, nt, smem>>>(iters, seed, out, clk);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double c = ms * 1e-3 * 1.965e9;
      const double lookups = (double)iters * 64 * nt;   // per SM
      printf("vol=%d nt=%4d: %.2f lookups/clk/SM  (%.1f B/clk plane data, %.2f TB/s chip @1.965GHz)\n", vol, nt,
             lookups / c, lookups / c, lookups / c * nsm * 1.965e9 / 1e12);
    }
  return 0;
}
