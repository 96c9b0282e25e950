// Grid-barrier latency on one B200 (148 co-resident CTAs): cost per barrier of
// several software implementations, and of cooperative_groups grid.sync().
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ubench_barrier tools/ubench_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// mode 0: red.release counter, poll counter acquire
// mode 1: red counter (after fence), poll counter relaxed, fence after
// mode 2: atom counter, last writes 8 flags, poll own flag relaxed
// mode 3: like 2 with 1 flag
// mode 4: atom counter, last writes one flag per CTA (148 lines), poll own
__global__ void bar_kernel(unsigned long long* bar, int iters, int mode, long long* out) {
  const int G = gridDim.x;
  const unsigned long long e0 = bar[0] / G;
  const long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    const unsigned long long ep = e0 + it;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (mode == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" :: "l"(bar) : "memory");
        while (ld_acq(bar) < ep * G) {}
      } else if (mode == 1) {
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" :: "l"(bar) : "memory");
        while (ld_rlx(bar) < ep * G) {}
        __threadfence();
      } else {
        const unsigned long long old = atomicAdd(bar, 1ull);
        const int nf = mode == 2 ? 8 : (mode == 3 ? 1 : G);
        if (old + 1 == ep * G) {
          for (int i = 0; i < nf; ++i)
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(bar + 16 * (1 + i)), "l"(ep) : "memory");
        }
        const unsigned long long* f = bar + 16 * (1 + (blockIdx.x % nf));
        while (ld_rlx(f) < ep) {}
        __threadfence();
      }
    }
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

__global__ void cg_kernel(int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) g.sync();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* bar;
  CK(cudaMalloc(&bar, 16 * (2 + 160) * 8));
  long long* out;
  CK(cudaMalloc(&out, nsm * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int mode = 0; mode < 5; ++mode) {
    CK(cudaMemset(bar, 0, 16 * (2 + 160) * 8));
    void* args[] = {&bar, (void*)&iters, &mode, &out};
    CK(cudaLaunchCooperativeKernel((void*)bar_kernel, nsm, 512, args, 0, 0));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)bar_kernel, nsm, 512, args, 0, 0));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("mode %d: %.3f us per barrier\n", mode, ms * 1e3 / iters);
  }
  {
    void* args[] = {(void*)&iters, &out};
    CK(cudaLaunchCooperativeKernel((void*)cg_kernel, nsm, 512, args, 0, 0));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)cg_kernel, nsm, 512, args, 0, 0));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cg grid.sync: %.3f us per barrier\n", ms * 1e3 / iters);
  }
  return 0;
}
