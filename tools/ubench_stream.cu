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


// The bitplane GEMV's access pattern: 8 KB chunks, plane-strided sources
// (chunk c -> plane c % NP at offset (c / NP) * CHUNK of that plane's region),
// consumed by quads of 4 warps (warp i of quad q reads 2 KB of the chunks
// c = q, q + NQ, ...; empty barrier count 4).
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                                 unsigned long long pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                  "r"((unsigned)__cvta_generic_to_shared(bar)), "l"(pol) : "memory");
}
template <int STAGES, int NP, int HINT = 0>
__global__ void ring_kernel(const unsigned char* __restrict__ p, long long nbytes, unsigned* out) {
  constexpr int CHUNK = 8192;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  __shared__ volatile int seq[STAGES];
  const long long plane = nbytes / NP;
  const long long per = plane / gridDim.x / CHUNK * CHUNK;
  const int n_chunks = (int)(per / CHUNK) * NP;
  const int nw = blockDim.x / 32 - 1, nq = nw / 4;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); seq[s] = -1; }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      for (int c = 0; c < n_chunks; ++c) {
        const int s = c % STAGES;
        if (c >= STAGES) mbar_wait(&empty[s], ((c / STAGES) - 1) & 1);
        seq[s] = c;
        mbar_expect_tx(&full[s], CHUNK);
        const unsigned char* src = p + (long long)(c % NP) * plane + per * blockIdx.x + (long long)(c / NP) * CHUNK;
        if (HINT) {
          unsigned long long pol;
          asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
          tma_load_1d_hint(smem + s * CHUNK, src, CHUNK, &full[s], pol);
        } else {
          tma_load_1d(smem + s * CHUNK, src, CHUNK, &full[s]);
        }
      }
    }
    return;
  }
  unsigned acc = 0;
  const int cw = warp - 1, q = cw / 4, i = cw % 4;
  for (int c = q; c < n_chunks; c += nq) {
    const int s = c % STAGES;
    while (seq[s] != c) {}
    mbar_wait(&full[s], (c / STAGES) & 1);
    const uint4* d = reinterpret_cast<const uint4*>(smem + s * CHUNK + i * 2048) + lane;
    const uint4 a = d[0], b = d[32], e = d[64], f = d[96];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    acc ^= a.x ^ b.y ^ e.z ^ f.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// 2 KB items issued by L producer lanes in parallel (lane l: items c = l mod L,
// slot c mod STAGES), consumed by all consumer warps round-robin (one warp per item).
template <int STAGES, int L>
__global__ void lanes_kernel(const unsigned char* __restrict__ p, long long nbytes, unsigned* out) {
  constexpr int CHUNK = 2048;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  __shared__ volatile int seq[STAGES];
  const long long per = nbytes / gridDim.x / CHUNK * CHUNK;
  const unsigned char* base = p + per * blockIdx.x;
  const int n_chunks = (int)(per / CHUNK);
  const int nw = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); seq[s] = -1; }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane < L)
      for (int c = lane; c < n_chunks; c += L) {
        const int s = c % STAGES;
        if (c >= STAGES) mbar_wait(&empty[s], ((c / STAGES) - 1) & 1);
        seq[s] = c;
        mbar_expect_tx(&full[s], CHUNK);
        tma_load_1d(smem + s * CHUNK, base + (long long)c * CHUNK, CHUNK, &full[s]);
      }
    return;
  }
  unsigned acc = 0;
  for (int c = warp - 1; c < n_chunks; c += nw) {
    const int s = c % STAGES;
    while (seq[s] != c) {}
    mbar_wait(&full[s], (c / STAGES) & 1);
    const uint4* d = reinterpret_cast<const uint4*>(smem + s * CHUNK) + lane;
    const uint4 a = d[0], b = d[32], e = d[64], f = d[96];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    acc ^= a.x ^ b.y ^ e.z ^ f.w;
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
    // small items (the GEMV's 2 KB (plane, tile) items): issue-rate bound?
    auto k5 = tma_kernel<64, 2048>;
    CK(cudaFuncSetAttribute(k5, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 2048));
    timeit("tma 64x2KB nt=544", [&] { k5<<<nsm, 544, 64 * 2048>>>(p, bytes, o); });
    auto k6 = tma_kernel<32, 4096>;
    CK(cudaFuncSetAttribute(k6, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 4096));
    timeit("tma 32x4KB nt=544", [&] { k6<<<nsm, 544, 32 * 4096>>>(p, bytes, o); });
    auto k7 = tma_kernel<16, 8192>;
    CK(cudaFuncSetAttribute(k7, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 8192));
    timeit("tma 16x8KB nt=544", [&] { k7<<<nsm, 544, 16 * 8192>>>(p, bytes, o); });
    auto r1 = ring_kernel<10, 8>;
    CK(cudaFuncSetAttribute(r1, cudaFuncAttributeMaxDynamicSharedMemorySize, 10 * 8192));
    timeit("ring 10x8KB quads 8 planes nt=544", [&] { r1<<<nsm, 544, 10 * 8192>>>(p, bytes, o); });
    auto r2 = ring_kernel<10, 1>;
    CK(cudaFuncSetAttribute(r2, cudaFuncAttributeMaxDynamicSharedMemorySize, 10 * 8192));
    timeit("ring 10x8KB quads 1 plane nt=544", [&] { r2<<<nsm, 544, 10 * 8192>>>(p, bytes, o); });
    auto r4 = ring_kernel<10, 8, 1>;
    CK(cudaFuncSetAttribute(r4, cudaFuncAttributeMaxDynamicSharedMemorySize, 10 * 8192));
    timeit("ring 10x8KB quads 8 planes evict_first", [&] { r4<<<nsm, 544, 10 * 8192>>>(p, bytes, o); });
    for (long long small : {58720256LL, 22020096LL, 6291456LL}) {
      // a single layer's bytes per launch, 30 copies round-robin (HBM, not L2)
      float best = 0.f;
      cudaEventRecord(e0);
      for (int it = 0; it < 60; ++it)
        r1<<<nsm, 544, 10 * 8192>>>(p + (long long)(it % 30) * small, small, o);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&best, e0, e1);
      printf("ring 10x8KB 8 planes, %lld B per launch: %.2f us/launch, %.1f GB/s\n", small, best * 1e3 / 60,
             small * 60 / (best * 1e-3) / 1e9);
    }
    {
      auto l1 = lanes_kernel<64, 1>;
      CK(cudaFuncSetAttribute(l1, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 2048));
      timeit("2KB items 64 slots 1 lane", [&] { l1<<<nsm, 544, 64 * 2048>>>(p, bytes, o); });
      auto l8 = lanes_kernel<64, 8>;
      CK(cudaFuncSetAttribute(l8, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 2048));
      timeit("2KB items 64 slots 8 lanes", [&] { l8<<<nsm, 544, 64 * 2048>>>(p, bytes, o); });
      auto l16 = lanes_kernel<64, 16>;
      CK(cudaFuncSetAttribute(l16, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 2048));
      timeit("2KB items 64 slots 16 lanes", [&] { l16<<<nsm, 544, 64 * 2048>>>(p, bytes, o); });
      auto l32 = lanes_kernel<64, 32>;
      CK(cudaFuncSetAttribute(l32, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 2048));
      timeit("2KB items 64 slots 32 lanes", [&] { l32<<<nsm, 544, 64 * 2048>>>(p, bytes, o); });
    }
    auto r3 = ring_kernel<20, 8>;
    CK(cudaFuncSetAttribute(r3, cudaFuncAttributeMaxDynamicSharedMemorySize, 20 * 8192));
    timeit("ring 20x8KB quads 8 planes nt=544", [&] { r3<<<nsm, 544, 20 * 8192>>>(p, bytes, o); });
    auto k8 = tma_kernel<100, 2048>;
    CK(cudaFuncSetAttribute(k8, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 2048));
    timeit("tma 100x2KB nt=544", [&] { k8<<<nsm, 544, 100 * 2048>>>(p, bytes, o); });
  }
  return 0;
}
