// HBM read-bandwidth ceiling on one B200 by load mechanism: LDG.128 with
// varying loads in flight, and 1D TMA bulk copies (cp.async.bulk) into a
// shared-memory ring with mbarriers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ubench_stream tools/ubench_stream.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// Each CTA streams a contiguous slice; each warp reads U x 512 B per round.
template <int U>
__global__ void ldg_kernel(const uint4* __restrict__ p, long long n16, unsigned* out) {
  const long long per = n16 / gridDim.x;
  const uint4* base = p + per * blockIdx.x;
  unsigned acc = 0;
  const int nt = blockDim.x;
  for (long long i = threadIdx.x; i + (U - 1) * nt < per; i += (long long)U * nt) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_stream(base + i + u * nt);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" :: "r"(a), "r"(phase) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                  "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

// Warp 0 lane 0 = producer; the other warps consume (LDS.128 xor) each stage.
template <int STAGES, int CHUNK>
__global__ void tma_kernel(const unsigned char* __restrict__ p, long long nbytes, unsigned* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const long long per = nbytes / gridDim.x / CHUNK * CHUNK;
  const unsigned char* base = p + per * blockIdx.x;
  const int n_chunks = (int)(per / CHUNK);
  const int nw = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nw); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      for (int c = 0; c < n_chunks; ++c) {
        const int s = c % STAGES;
        if (c >= STAGES) mbar_wait(&empty[s], ((c / STAGES) - 1) & 1);
        mbar_expect_tx(&full[s], CHUNK);
        tma_load_1d(smem + s * CHUNK, base + (long long)c * CHUNK, CHUNK, &full[s]);
      }
    }
    return;
  }
  unsigned acc = 0;
  const int cw = warp - 1;
  for (int c = 0; c < n_chunks; ++c) {
    const int s = c % STAGES;
    mbar_wait(&full[s], (c / STAGES) & 1);
    const uint4* q = reinterpret_cast<const uint4*>(smem + s * CHUNK);
    for (int i = cw * 32 + lane; i < CHUNK / 16; i += nw * 32) { uint4 v = q[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const long long bytes = 2LL << 30;
  unsigned char* p;
  unsigned* o;
  CK(cudaMalloc(&p, bytes));
  CK(cudaMemset(p, 1, bytes));
  CK(cudaMalloc(&o, 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %8.1f GB/s\n", name, bytes * 10.0 / (ms * 1e-3) / 1e9);
  };
  char nm[128];
  for (int nt : {256, 512, 1024}) {
    for (int g : {1, 2}) {
      snprintf(nm, sizeof nm, "ldg U=4  nt=%d grid=%dx", nt, g);
      timeit(nm, [&] { ldg_kernel<4><<<g * nsm, nt>>>((const uint4*)p, bytes / 16, o); });
      snprintf(nm, sizeof nm, "ldg U=8  nt=%d grid=%dx", nt, g);
      timeit(nm, [&] { ldg_kernel<8><<<g * nsm, nt>>>((const uint4*)p, bytes / 16, o); });
      snprintf(nm, sizeof nm, "ldg U=16 nt=%d grid=%dx", nt, g);
      timeit(nm, [&] { ldg_kernel<16><<<g * nsm, nt>>>((const uint4*)p, bytes / 16, o); });
    }
  }
  {
    auto k1 = tma_kernel<4, 16384>;
    CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384));
    timeit("tma 4x16KB nt=288", [&] { k1<<<nsm, 288, 4 * 16384>>>(p, bytes, o); });
    auto k2 = tma_kernel<8, 16384>;
    CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384));
    timeit("tma 8x16KB nt=288", [&] { k2<<<nsm, 288, 8 * 16384>>>(p, bytes, o); });
    timeit("tma 8x16KB nt=544", [&] { k2<<<nsm, 544, 8 * 16384>>>(p, bytes, o); });
    auto k3 = tma_kernel<12, 16384>;
    CK(cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384));
    timeit("tma 12x16KB nt=544", [&] { k3<<<nsm, 544, 12 * 16384>>>(p, bytes, o); });
    auto k4 = tma_kernel<6, 32768>;
    CK(cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768));
    timeit("tma 6x32KB nt=544", [&] { k4<<<nsm, 544, 6 * 32768>>>(p, bytes, o); });
  }
  return 0;
}
