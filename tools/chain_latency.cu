// Kernel-to-kernel hand-off cost of a chain of persistent one-CTA-per-SM grids (the decode
// step's launch shape: #SMs CTAs x 704 threads, ~222 KB shared memory), three ways:
//   0  plain stream order (no PDL)
//   1  programmatic dependent launch, griddepcontrol.wait at the top (the library's default)
//   2  programmatic dependent launch, no griddepcontrol.wait: every CTA adds to a grid-wide
//      counter (red.release.gpu) after its work; the next grid's CTAs poll it (ld.acquire.gpu)
// Each CTA busy-waits `work_ns` (globaltimer) with a per-CTA skew of up to `skew_ns`, like
// the step's end spread. Prints us per kernel above the work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/chain tools/chain_latency.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(704, 1) step(int mode, unsigned long long* ctr, unsigned long long seq,
                                               unsigned work_ns, unsigned skew_ns) {
  extern __shared__ uint8_t sm[];
  if (mode == 1) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (mode == 2 && threadIdx.x == 0) {
    const unsigned long long want = seq * gridDim.x;
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
    } while (v < want);
  }
  __syncthreads();
  if (mode != 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    sm[0] = 1;
    const unsigned long long t0 = gt();
    const unsigned long long w = work_ns + (skew_ns ? (blockIdx.x * 2654435761u) % skew_ns : 0);
    while (gt() - t0 < w) {
    }
  }
  __syncthreads();
  if (mode == 2 && threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
}

int main(int argc, char** argv) {
  const unsigned work = argc > 1 ? atoi(argv[1]) : 20000;
  const unsigned skew = argc > 2 ? atoi(argv[2]) : 0;
  const int iters = 2000;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 222 * 1024;
  cudaFuncSetAttribute(step, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* ctr;
  cudaMalloc(&ctr, 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      cudaMemset(ctr, 0, 8);
      cudaDeviceSynchronize();
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(sms);
      cfg.blockDim = dim3(704);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = mode ? 1 : 0;
      unsigned long long seq = 0;
      for (int i = 0; i < 50; ++i) cudaLaunchKernelEx(&cfg, step, mode, ctr, seq++, work, skew);
      cudaEventRecord(e0, s);
      for (int i = 0; i < iters; ++i) cudaLaunchKernelEx(&cfg, step, mode, ctr, seq++, work, skew);
      cudaEventRecord(e1, s);
      cudaError_t e = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"mode\": %d, \"work_ns\": %u, \"skew_ns\": %u, \"us_per_kernel\": %.3f, \"overhead_us\": %.3f, \"err\": \"%s\"}\n",
             mode, work, skew, ms * 1000.f / iters, ms * 1000.f / iters - work / 1000.f, cudaGetErrorString(e));
    }
  return 0;
}
