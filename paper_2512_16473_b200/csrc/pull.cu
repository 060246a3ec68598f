// pull.cu — MOE_MISS_PULL for the split decode path and the prefill path: one kernel, run
// in stream order between the kernel that decided the misses (router / prefill plan) and
// the expert kernels that read the slots. Every CTA copies a 1/grid share of each listed
// blob from the pinned host backing store into its slot (pull.cuh); the last CTA to finish
// publishes ready[slot] = gen for each (the expert kernels' readiness check), then resets
// the completion counter for the next launch.
#include "moe_internal.cuh"
#include "pull.cuh"

namespace moe {
namespace {

constexpr int kPullThreads = 512;

__global__ void __launch_bounds__(kPullThreads) pull_kernel(const PullJob j) {
  __shared__ bool last;
  const int cnt = *j.count;
  for (int i = 0; i < cnt; ++i) {
    if (!j.flag[i] || (j.only && j.only[i] != j.only_val)) continue;
    long long u0, u1;
    pull_share(j.slot_bytes, blockIdx.x, gridDim.x, &u0, &u1);
    pull_copy(j.pool + (long long)j.slot[i] * j.slot_bytes, j.hblob[j.expert[i]], u0, u1, threadIdx.x, kPullThreads);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(j.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = threadIdx.x; i < cnt; i += kPullThreads)
    if (j.flag[i] && (!j.only || j.only[i] == j.only_val)) *((volatile uint32_t*)(j.ready + j.slot[i])) = j.gen[i];
  if (threadIdx.x == 0) *j.done = 0u;
}

}  // namespace

cudaError_t preload_pull_kernels() {
  cudaFuncAttributes fa;
  return cudaFuncGetAttributes(&fa, pull_kernel);
}

cudaError_t launch_pull(const PullJob& j, int grid, cudaStream_t s) {
  pull_kernel<<<grid, kPullThreads, 0, s>>>(j);
  return cudaGetLastError();
}

}  // namespace moe
