// Floor of the decode step's structure: a chain of one-CTA-per-SM kernels (programmatic
// dependent launch, griddepcontrol.wait at the top) that each only STREAM `bytes` of HBM
// through a bulk-copy ring (one producer lane, NS x SB stages, consumer warps releasing them),
// every CTA a contiguous equal share, consecutive launches reading different bytes (no L2
// reuse). What this chain takes above bytes / bandwidth is the cost of the kernel boundary,
// the first-byte latency and the end drain with NO routing, h exchange or stolen tail: the
// fixed cost an ideal one-kernel step could not avoid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/chain_stream tools/chain_stream.cu
//   tools/chain_stream [SB NS]
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(704, 1) stream_step(const uint8_t* p, long long bytes, int NS, int SB, int early,
                                                      int* out) {
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
  if (early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
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
  for (int t = cw; t < nparts; t += NS) {
    asm volatile("{\n.reg .pred q;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W%=;\n}" ::"r"(
                     sa(full + cw)),
                 "r"((t / NS) & 1));
    acc ^= ((int*)(sm + (size_t)cw * SB))[lane];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + cw)));
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main(int argc, char** argv) {
  const int SB = argc > 1 ? atoi(argv[1]) : 24576, NS = argc > 2 ? atoi(argv[2]) : 8;
  const long long buf = 6ll << 30;
  uint8_t* p;
  int* out;
  cudaMalloc(&p, buf);
  cudaMalloc(&out, 4);
  cudaMemset(p, 1, buf);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = (size_t)NS * SB + 2 * NS * 8;
  cudaFuncSetAttribute(stream_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (long long mb : {1ll, 20ll, 151ll, 315ll, 705ll}) {
    const long long bytes = mb * 1000000ll / 4096 * 4096;
    const int slots = (int)(buf / bytes);
    for (int early = 0; early < 2; ++early) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(sms);
      cfg.blockDim = dim3(704);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const int iters = mb > 300 ? 500 : 2000;
      for (int i = 0; i < 20; ++i) cudaLaunchKernelEx(&cfg, stream_step, (const uint8_t*)(p + (i % slots) * bytes), bytes, NS, SB, early, out);
      cudaEventRecord(e0, s);
      for (int i = 0; i < iters; ++i)
        cudaLaunchKernelEx(&cfg, stream_step, (const uint8_t*)(p + (i % slots) * bytes), bytes, NS, SB, early, out);
      cudaEventRecord(e1, s);
      const cudaError_t e = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1000.0 / iters;
      printf("{\"MB\": %lld, \"SB\": %d, \"NS\": %d, \"early_trigger\": %d, \"us_per_kernel\": %.3f, \"GBs\": %.1f, \"err\": \"%s\"}\n", mb,
             SB, NS, early, us, bytes / (us * 1e-6) / 1e9, cudaGetErrorString(e));
    }
  }
  return 0;
}
