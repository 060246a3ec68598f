// Cost of a gpu-scope release inside an HBM-streaming kernel (the decode step's h
// publication): one CTA per SM streams 705 MB through a bulk-copy ring; every 8th stage a
// consumer warp's lane 0 publishes to a global counter in one of these ways, timed with
// globaltimer around the publication:
//   0  st.global (an h value) ; red.release.gpu.add      (the kernel's pattern)
//   1  red.release.gpu.add with no store of its own since the last publication
//   2  st.global ; red.relaxed.gpu.add                     (no fence: not a valid publication)
//   3  st.global ; fence.acq_rel.gpu ; red.relaxed.gpu.add
//   4  st.global ; (next stage) red.release.gpu.add        (release one stage later)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fence_cost tools/fence_cost.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(704, 1) stream_pub(const uint8_t* p, long long bytes, int NS, int SB, int mode,
                                                     unsigned long long* ctr, float* hbuf, unsigned long long* acc_ns,
                                                     unsigned long long* acc_n) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)NS * SB);
  uint64_t* empty = full + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long b0 = bytes * blockIdx.x / gridDim.x / 16 * 16, b1 = bytes * (blockIdx.x + 1) / gridDim.x / 16 * 16;
  const int nparts = (int)((b1 - b0 + SB - 1) / SB);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(full + s)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(empty + s)), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      for (int t = 0; t < nparts; ++t) {
        const int s = t % NS;
        const uint32_t par = ((t / NS) & 1) ^ 1;
        asm volatile("{\n.reg .pred q;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W%=;\n}" ::"r"(
                         sa(empty + s)),
                     "r"(par));
        const long long off = b0 + (long long)t * SB;
        const uint32_t nb = (uint32_t)((b1 - off) < SB ? (b1 - off) : SB);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(nb));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                sa(sm + (size_t)s * SB)),
            "l"(p + off), "r"(nb), "r"(sa(full + s)), "l"(pol)
            : "memory");
      }
    }
    return;
  }
  const int cw = warp - 1;
  if (cw >= NS) return;
  int acc = 0;
  unsigned long long tsum = 0, tn = 0;
  bool pending = false;
  for (int t = cw; t < nparts; t += NS) {
    asm volatile("{\n.reg .pred q;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W%=;\n}" ::"r"(
                     sa(full + cw)),
                 "r"((t / NS) & 1));
    acc ^= ((int*)(sm + (size_t)cw * SB))[lane];
    __syncwarp();
    if (lane == 0) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + cw)));
      float* hp = hbuf + (blockIdx.x * 32 + cw) * 64 + ((t / NS) & 63);
      if (mode == 4 && pending) {
        const unsigned long long t0 = gt();
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        tsum += gt() - t0;
        ++tn;
        pending = false;
      }
      if (((t / NS) & 7) == 7) {
        if (mode != 1) *(volatile float*)hp = (float)acc;
        const unsigned long long t0 = gt();
        if (mode == 0 || mode == 1) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        if (mode == 2) asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        if (mode == 3) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        }
        if (mode == 4) pending = true;
        if (mode != 4) {
          tsum += gt() - t0;
          ++tn;
        }
      }
    }
  }
  if (lane == 0 && tn) {
    atomicAdd(acc_ns, tsum);
    atomicAdd(acc_n, tn);
  }
}

int main() {
  const long long bytes = 705ll * 1000000 / 4096 * 4096;
  const long long buf = 6ll << 30;
  uint8_t* p;
  cudaMalloc(&p, buf);
  cudaMemset(p, 1, buf);
  unsigned long long *ctr, *acc;
  float* hbuf;
  cudaMalloc(&ctr, 8);
  cudaMalloc(&acc, 16);
  cudaMalloc(&hbuf, 148 * 32 * 64 * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int NS = 10, SB = 16384;
  const size_t smem = (size_t)NS * SB + 2 * NS * 8;
  cudaFuncSetAttribute(stream_pub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int slots = (int)(buf / bytes);
  for (int mode = 0; mode < 5; ++mode) {
    for (int i = 0; i < 5; ++i)
      stream_pub<<<sms, 704, smem>>>(p + (i % slots) * bytes, bytes, NS, SB, mode, ctr, hbuf, acc, acc + 1);
    cudaMemset(acc, 0, 16);
    cudaEventRecord(e0);
    const int iters = 50;
    for (int i = 0; i < iters; ++i)
      stream_pub<<<sms, 704, smem>>>(p + (i % slots) * bytes, bytes, NS, SB, mode, ctr, hbuf, acc, acc + 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2];
    cudaMemcpy(h, acc, 16, cudaMemcpyDeviceToHost);
    printf("{\"mode\": %d, \"us_per_kernel\": %.2f, \"publications\": %llu, \"publish_ns_mean\": %.1f, \"err\": \"%s\"}\n", mode,
           ms * 1000 / iters, h[1], h[1] ? (double)h[0] / h[1] : 0.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
