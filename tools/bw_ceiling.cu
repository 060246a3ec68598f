// Read-bandwidth ceilings on this B200: LDG streaming vs bulk-copy (TMA linear) ring.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int U>
__global__ void ldg_read(const int4* __restrict__ p, long long n16, int* out) {
  int acc = 0;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n16; i += stride * U) {
    int4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      long long j = i + k * stride;
      if (j < n16) asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(p + j));
      else v[k] = make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

// 1 CTA per SM: lane 0 of warp 0 streams [begin,end) of this CTA's share in SB chunks
// into NS stages; NS consumer warps each own a stage and just release it (touching one word).
__global__ void bulk_ring(const uint8_t* p, long long bytes, int NS, int SB, int* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)NS * SB);
  uint64_t* empty = full + NS;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long b0 = bytes * blockIdx.x / gridDim.x / 16 * 16, b1 = bytes * (blockIdx.x + 1) / gridDim.x / 16 * 16;
  int nparts = (int)((b1 - b0 + SB - 1) / SB);
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
        int s = t % NS;
        uint32_t par = ((t / NS) & 1) ^ 1;
        asm volatile("{\n.reg .pred q;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W%=;\n}" ::"r"(sa(empty + s)), "r"(par));
        long long off = b0 + (long long)t * SB;
        uint32_t nb = (uint32_t)((b1 - off) < SB ? (b1 - off) : SB);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(nb));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(sa(sm + (size_t)s * SB)), "l"(p + off), "r"(nb), "r"(sa(full + s)), "l"(pol) : "memory");
      }
    }
    return;
  }
  int cw = warp - 1;
  if (cw >= NS) return;
  int acc = 0;
  for (int t = cw; t < nparts; t += NS) {
    asm volatile("{\n.reg .pred q;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W%=;\n}" ::"r"(sa(full + cw)), "r"((t / NS) & 1));
    acc ^= ((int*)(sm + (size_t)cw * SB))[lane];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + cw)));
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  const long long bytes = 2ll << 30;  // 2 GiB
  uint8_t* p; int* out;
  cudaMalloc(&p, bytes); cudaMalloc(&out, 4);
  cudaMemset(p, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto fn, const char* name) {
    for (int i = 0; i < 3; ++i) fn();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) fn();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %8.1f GB/s  (%s)\n", name, bytes * 10 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int blocks : {1, 2, 4, 8}) {
    for (int thr : {256, 512}) {
      char nm[64]; snprintf(nm, 64, "ldg U=8 grid=%dx%d thr=%d", sms, blocks, thr);
      timeit([&] { ldg_read<8><<<sms * blocks, thr>>>((const int4*)p, bytes / 16, out); }, nm);
    }
  }
  cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int SB : {8192, 16384, 32768}) {
    for (int NS : {4, 6, 8, 10, 12, 16}) {
      size_t smem = (size_t)NS * SB + 2 * NS * 8;
      if (smem > 227 * 1024 || NS > 16) continue;
      char nm[64]; snprintf(nm, 64, "bulk ring SB=%d NS=%d (%zu KB)", SB, NS, smem / 1024);
      timeit([&] { bulk_ring<<<sms, 32 * 17, smem>>>(p, bytes, NS, SB, out); }, nm);
    }
  }
  return 0;
}
