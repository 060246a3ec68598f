// pull.cuh — MOE_MISS_PULL (moe.h): a missed expert's blob is copied from the pinned host
// backing store (device-accessible through UVA) into its HBM slot by the SMs themselves.
//
// P:200 fetches a missed expert "to update the cache"; P:226 does it on a copy stream driven
// by the host. Here the copy is part of the call's own kernel(s): each participating CTA
// moves a contiguous 1/G share of the blob with 16-B loads over PCIe (several independent
// loads in flight per thread, so ~100 KB are outstanding grid-wide — the PCIe Gen5
// bandwidth-latency product) and plain stores into the slot. Ordering towards the readers
// (bulk async copies, possibly in other CTAs) is the caller's: a release after the copy, an
// acquire + fence.proxy.async before the first bulk read of the slot.
#pragma once
#include <stdint.h>

namespace moe {

// 16-B load that bypasses L1 (host memory, read once)
__device__ __forceinline__ int4 ld_nc_na_v4(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Share [lo, hi) of a blob of `bytes` bytes (bytes % 16 == 0) for part `b` of `G`, 16-B units.
__device__ __forceinline__ void pull_share(long long bytes, int b, int G, long long* lo, long long* hi) {
  const long long units = bytes >> 4;
  *lo = units * b / G;
  *hi = units * (b + 1) / G;
}

// dst[i] = src[i] for 16-B units i in [u0, u1), threads tid = 0 .. nthr-1 of the caller.
__device__ __forceinline__ void pull_copy(uint8_t* dst, const uint8_t* src, long long u0, long long u1, int tid,
                                          int nthr) {
#ifndef MOE_PULL_U
#define MOE_PULL_U 4
#endif
  constexpr int U = MOE_PULL_U;  // independent loads in flight per thread
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  for (long long i = u0 + tid; i < u1; i += (long long)U * nthr) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long k = i + (long long)u * nthr;
      if (k < u1) v[u] = ld_nc_na_v4(s + k);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long k = i + (long long)u * nthr;
      if (k < u1) d[k] = v[u];
    }
  }
}

}  // namespace moe
