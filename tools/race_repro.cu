// race_repro.cu — minimal reproduction of the pattern the fused decode kernel uses on a miss
// (a slot written DURING the kernel by other CTAs, read with a bulk async copy after an
// acquire), to tell a kernel bug from a compute-sanitizer racecheck artefact.
//
//   launch i:  CTAs 1..G-1 write buf[] = i (plain st.global), then red.release.gpu on a counter;
//              CTA 0 acquires the counter (ld.acquire.gpu), fence.proxy.async.global, then
//              cp.async.bulk global -> shared of buf and checks every word == i.
// The buffer holds the previous launch's values when CTA 0 last read it, so a reader that is
// served stale data shows up as mismatches.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o race_repro tools/race_repro.cu
//   ./race_repro ; compute-sanitizer --tool racecheck ./race_repro
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kWords = 4096;  // 16 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void repro(uint32_t* buf, unsigned long long* ctr, unsigned long long target, uint32_t val, int* bad) {
  __shared__ __align__(128) uint32_t s[kWords];
  __shared__ __align__(8) uint64_t bar;
  const int G = gridDim.x, b = blockIdx.x;
  if (b > 0) {
    // writers: CTA b owns words [lo, hi)
    const int lo = (int)((long long)kWords * (b - 1) / (G - 1)), hi = (int)((long long)kWords * b / (G - 1));
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) buf[i] = val;
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    return;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned long long v, t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {  // (10 s cap: a tool that does not co-schedule the CTAs would otherwise hang)
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (v < target && t - t0 < 10000000000ull);
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(kWords * 4)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(s)),
        "l"(buf), "r"(kWords * 4), "r"(smem_u32(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            smem_u32(&bar))
        : "memory");
  }
  __syncthreads();
  int nb = 0;
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) nb += s[i] != val;
  if (nb) atomicAdd(bad, nb);
}

int main() {
  uint32_t* buf;
  unsigned long long* ctr;
  int* bad;
  cudaMalloc(&buf, kWords * 4);
  cudaMalloc(&ctr, 8);
  cudaMallocManaged(&bad, 4);
  cudaMemset(buf, 0, kWords * 4);
  cudaMemset(ctr, 0, 8);
  *bad = 0;
  const int G = 16, iters = 50;
  int total = 0;
  for (int it = 1; it <= iters; ++it) {
    repro<<<G, 256>>>(buf, ctr, (unsigned long long)it * (G - 1), (uint32_t)it, bad);
    cudaDeviceSynchronize();
    total += *bad;
    *bad = 0;
  }
  const cudaError_t e = cudaGetLastError();
  printf("race_repro: %d launches, mismatching words read through the bulk copy: %d (%s)\n", iters, total,
         cudaGetErrorString(e));
  return total != 0;
}
