// expert_fused.cu — K23: the whole expert FFN of one decode step in ONE persistent kernel
// (sm_100a): SwiGLU gate/up GEMVs -> barrier -> down GEMV + gate-weighted combine.
//
//   phase A  h_r[j] = silu(W1_r[j,:] x) * (W3_r[j,:] x)              (R4)
//   phase B  y[c]  += w_r * (W2_r[c,:] h_r)
//
// Decode batch 1 makes every expert matrix a GEMV (~1 FLOP/byte): an HBM stream, not a
// tensor-core contraction. Design for B200:
//  - one CTA per SM (grid = #SMs, cooperative => co-resident). The CTAs are split into K
//    groups, group r serving routed expert r only: its phase A rows j and its phase B
//    rows c — 88% in static contiguous blocks, the tail claimed in small chunks from a
//    per-expert counter (per-SM HBM bandwidth varies by ~10%; stealing evens it out). The
//    barrier between the phases is per expert (the CTAs that produce h_r), and a CTA needs
//    only ONE expert's h in shared memory, which leaves room for a large weight ring;
//  - warp 0 / lane 0 is a producer streaming weight rows with bulk async copies
//    (cp.async.bulk — the TMA engine's linear path, SASS UBLKCP) into an NS-stage shared
//    memory ring guarded by full/empty mbarriers (L2 evict-first). Bytes in flight per SM
//    = the ring (~160 KB at Mixtral shapes), independent of how many consumer warps are
//    still busy. W2 rows do not depend on h, so the producer streams through the barrier;
//  - one consumer warp per ring stage: x (bf16) and then h_r (fp32, stored by phase A in
//    a 2-plane layout and pulled in with ONE bulk copy) live in shared memory; fp32 FMAs,
//    warp-shuffle reductions;
//  - combine: y (zeroed by the router kernel) += w_r * o_r[c] with fire-and-forget fp32
//    reductions. K <= 2 only: two addends onto 0 commute exactly, so y is bit-identical
//    to the oracle's rank-ordered sum; other K take the split path.
#include <math.h>

#include "moe_internal.cuh"
#include "ptx.cuh"

namespace moe {
namespace {

using namespace ptx;

constexpr int kMaxNS = 10;                 // ring stages (phase B pairs them: NS even)
constexpr int kWarpsPerStage = 2;          // consumer warps sharing one stage
constexpr int kThreadsF = 32 * (1 + kWarpsPerStage * kMaxNS);

// Packed fp32 FMA (sm_100: FFMA2): acc.{x,y} += a.{x,y} * b.{x,y}
__device__ __forceinline__ float2 ffma2(const float2 a, const float2 b, const float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
        "l"(*reinterpret_cast<const unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}

// bf16 pair (one 32-bit word) -> (lo, hi) fp32, exact
__device__ __forceinline__ float2 bf2(uint32_t v) { return make_float2(bf_lo(v), bf_hi(v)); }

// acc += w(8 bf16) . x(8 fp32)
__device__ __forceinline__ float2 dot8(const int4 w, const float4 a, const float4 b, float2 acc) {
  acc = ffma2(bf2(w.x), make_float2(a.x, a.y), acc);
  acc = ffma2(bf2(w.y), make_float2(a.z, a.w), acc);
  acc = ffma2(bf2(w.z), make_float2(b.x, b.y), acc);
  acc = ffma2(bf2(w.w), make_float2(b.z, b.w), acc);
  return acc;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// h_r[j] lives at plane (j%8)/4, chunk j/8, lane j%4: a consumer lane reading the 8 h
// values of one 16-B weight chunk issues two conflict-free 16-B shared loads.
__device__ __forceinline__ int h_plane_index(int j, int ffr) {
  return ((j >> 2) & 1) * (ffr >> 1) + ((j >> 3) << 2) + (j & 3);
}

__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

__device__ __forceinline__ void red_release_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr int kChunkA = 2;     // phase A rows per tail claim
constexpr int kChunkB = 1;     // phase B rows per tail claim
constexpr int kStaticPct = 88; // share of each phase's rows assigned statically (no atomics)

// Static-then-steal schedule over `total` rows for CTA li of a group of gsz CTAs: the first
// kStaticPct% of the rows are split into equal contiguous blocks, the tail is claimed in
// chunks from a per-expert counter, so every CTA of the group ends each phase within about
// one chunk of the others, whatever its share of HBM bandwidth.
struct RowSched {
  int s0, s1;    // this CTA's static block
  int tail0;     // first tail row
};
__device__ __forceinline__ RowSched make_sched(int total, int li, int gsz) {
  RowSched rs;
  const int sb = (int)((long long)total * kStaticPct / 100 / gsz);
  rs.s0 = li * sb;
  rs.s1 = rs.s0 + sb;
  rs.tail0 = gsz * sb;
  return rs;
}

// Shared memory: ring[NS][SB] | xh | full[NS] empty[NS] hbar | meta[NS] | part[NS][2] |
//                parB[NS/2]
//  - phase A: stage s (16 KB) = one W1 row + one W3 row, consumed by warps 2s, 2s+1 (one
//    half of the row each); x lives in xh as fp32.
//  - phase B: stages (2u, 2u+1) form one super-stage holding a whole W2 row (<= 2*SB),
//    guarded by full[2u]/empty[2u] and consumed by the 4 warps of stages 2u, 2u+1 (a
//    quarter of the row each); h_r lives in xh as fp32 in the 2-plane layout.
//  - partial sums of a stage's warps are combined in a fixed order after a named barrier
//    (deterministic, no atomics). Every consumer warp waits on one mbarrier per phase, and
//    its next wait is always one phase ahead of the part it just released: parity waits
//    cannot alias.
__global__ void __launch_bounds__(kThreadsF, 1) expert_fused_kernel(const FusedArgs f) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ const uint8_t* sbase;
  __shared__ float swgt;
  __shared__ int swait, shost, sslot;
  __shared__ uint32_t sgen;
  const ExpertArgs& a = f.e;
  const int NS = f.NS, SB = f.SB, NSB = NS >> 1;
  uint8_t* ring = smem;
  uint8_t* xh = smem + (size_t)NS * SB;
  uint64_t* full = reinterpret_cast<uint64_t*>(xh + f.xh_bytes);
  uint64_t* empty = full + NS;
  uint64_t* hbar = empty + NS;
  volatile int* meta = reinterpret_cast<volatile int*>(hbar + 1);
  volatile float* part = reinterpret_cast<volatile float*>(meta + NS);   // [NS][4]
  volatile uint32_t* parB = reinterpret_cast<volatile uint32_t*>(part + 4 * NS);  // full[2u] parity at phase B start

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.K, d = a.d, ffr = a.ffr;
  const int G = gridDim.x, b = blockIdx.x;
  // expert group of this CTA: group r serves routed expert r (phase A rows j and phase B
  // rows c of that expert)
  const int r = (int)((long long)b * K / G);
  const int gb0 = (int)(((long long)r * G + K - 1) / K);
  const int gb1 = (int)(((long long)(r + 1) * G + K - 1) / K);
  const int gsz = gb1 - gb0, li = b - gb0;
  const int rowA = 4 * d;                       // bytes of one W1 row + one W3 row
  const int rowB = ffr * 2;                     // bytes of one W2 row (<= 2*SB)
  const long long w2off = 2ll * ffr * d * 2;    // W2 offset in a slot

  if (f.ts && threadIdx.x == 0) {
    f.ts[b * 8 + 0] = globaltimer();
    f.ts[b * 8 + 6] = 0;
    f.ts[b * 8 + 7] = 0;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(hbar, 1);
    fence_mbar_init();
  }
  // The router kernel publishes its route (release) before it completes: acquire it here
  // instead of waiting for the router grid's completion and memory flush (PDL launch).
  if (threadIdx.x == 0) {
    if (a.route_flag) {
      while (ld_acquire_u64(a.route_flag) != a.seq) {
      }
    }
  }
  if (!a.route_flag) griddep_wait();
  __syncthreads();
  if (f.ts && threadIdx.x == 0) f.ts[b * 8 + 1] = globaltimer();
  if (threadIdx.x == 0) {
    const int slot = a.route->slot[r];
    sslot = slot;
    sgen = a.route->gen[r];
    swait = a.route->wait[r];
    shost = a.route->host[r];
    sbase = a.pool + (long long)slot * a.slot_bytes;
    swgt = a.route->w[r];
  }
  for (int i = threadIdx.x; i < (d >> 2); i += kThreadsF) {  // x -> fp32 in shared memory
    const uint2 v = reinterpret_cast<const uint2*>(a.x)[i];
    reinterpret_cast<float4*>(xh)[i] = make_float4(bf_lo(v.x), bf_hi(v.x), bf_lo(v.y), bf_hi(v.y));
  }
  __syncthreads();
  const uint8_t* base = sbase;

  if (shost) {
    // ---------------------------------------------------------------- host-computed expert
    // (MOE_MISS_HOST_COMPUTE): wait for the host's result on the activation stream
    // and add w_r * o_r over this CTA's share of y; keep the group barrier count in step.
    if (threadIdx.x == 0) {
      red_release_add_u64(f.bar + 16 * r, 1ull);
      const uint32_t want = (uint32_t)a.seq;
      const unsigned long long t0 = globaltimer();
      unsigned ns = 256;
      while (ld_acquire_u32(a.host_flag + r) != want) {
        __nanosleep(ns);
        if (ns < 8192) ns <<= 1;
        if (globaltimer() - t0 > 60ull * 1000000000ull) __trap();
      }
    }
    __syncthreads();
    const int c0 = (int)((long long)d * li / gsz), c1 = (int)((long long)d * (li + 1) / gsz);
    const float w = swgt;
    const float* o = a.host_out + (size_t)r * d;
    for (int c = c0 + (int)threadIdx.x; c < c1; c += kThreadsF) {
      const float v = w * __ldcg(o + c);
      if (K == 1) a.y[c] = v;
      else red_add_f32(a.y + c, v);  // K == 2: 0 + a + b is order-independent
    }
    if (b == 0 && threadIdx.x == 0) *a.last_seq = a.seq;
    griddep_launch_dependents();
    return;
  }

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      if (swait) wait_ready(a.ready, sslot, sgen);  // fill of this slot still in flight
      unsigned* ctrA = f.ctr + r;
      unsigned* ctrB = f.ctr + kMaxK + r;
      uint32_t use = 0;                               // per-stage use-count parity bits
      auto acquire = [&](int s) {                     // wait until stage s is free
        mbar_wait(empty + s, ((use >> s) & 1) ^ 1);
        use ^= 1u << s;
      };
      int t = 0;
      auto issue_a = [&](int j) {
        const int s = t % NS;
        acquire(s);
        const uint8_t* w1 = base + (long long)j * d * 2;
        const uint8_t* w3 = w1 + (long long)ffr * d * 2;
        meta[s] = j;
        mbar_arrive_expect_tx(full + s, (uint32_t)rowA);
        bulk_g2s(ring + (size_t)s * SB, w1, 2u * d, full + s, pol);
        bulk_g2s(ring + (size_t)s * SB + 2 * d, w3, 2u * d, full + s, pol);
        ++t;
      };
      // phase A: static block, then tail claims (two claims in flight hide the atomic latency)
      const RowSched sa = make_sched(ffr, li, gsz);
      unsigned c1 = atomicAdd(ctrA, (unsigned)kChunkA);
      for (int j = sa.s0; j < sa.s1; ++j) issue_a(j);
      unsigned c2 = atomicAdd(ctrA, (unsigned)kChunkA);
      while (sa.tail0 + (int)c1 < ffr) {
        const int j0 = sa.tail0 + (int)c1, j1 = min(j0 + kChunkA, ffr);
        c1 = c2;
        if (sa.tail0 + (int)c1 < ffr) c2 = atomicAdd(ctrA, (unsigned)kChunkA);
        for (int j = j0; j < j1; ++j) issue_a(j);
      }
      for (int k = 0; k < NS; ++k, ++t) {  // one end-of-phase marker per stage
        const int s = t % NS;
        acquire(s);
        meta[s] = -1;
        mbar_arrive(full + s);
      }
      // phase B: whole W2 rows into super-stages (2u, 2u+1); W2 does not depend on h, so
      // these loads stream while the consumers finish phase A and cross the barrier
      int tb = 0;
      auto issue_b = [&](int c) {
        const int u = tb % NSB, s = 2 * u;
        acquire(s);
        meta[s] = c;
        mbar_arrive_expect_tx(full + s, (uint32_t)rowB);
        bulk_g2s(ring + (size_t)s * SB, base + w2off + (long long)c * rowB, (uint32_t)rowB, full + s, pol);
        ++tb;
      };
      const RowSched sbk = make_sched(d, li, gsz);
      c1 = atomicAdd(ctrB, (unsigned)kChunkB);
      for (int c = sbk.s0; c < sbk.s1; ++c) issue_b(c);
      c2 = atomicAdd(ctrB, (unsigned)kChunkB);
      while (sbk.tail0 + (int)c1 < d) {
        const int r0 = sbk.tail0 + (int)c1, r1 = min(r0 + kChunkB, d);
        c1 = c2;
        if (sbk.tail0 + (int)c1 < d) c2 = atomicAdd(ctrB, (unsigned)kChunkB);
        for (int c = r0; c < r1; ++c) issue_b(c);
      }
      for (int k = 0; k < NSB; ++k, ++tb) {
        const int s = 2 * (tb % NSB);
        acquire(s);
        meta[s] = -1;
        mbar_arrive(full + s);
      }
      // publish the call's progress to the host fetch thread (PCIe write overlaps the tail)
      if (b == 0) *a.last_seq = a.seq;
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  const int cw = warp - 1;                 // consumer warp 0 .. 2*NS-1
  if (cw >= kWarpsPerStage * NS) return;
  const int nthr = kWarpsPerStage * NS * 32;
  const int sA = cw >> 1, half = cw & 1;   // phase A: stage and half of the row
  float* hglob = a.h + (long long)r * ffr;
  uint32_t ph = 0;                         // parity of the barrier this warp waits on
  {
    const int nchA = d >> 3;               // 16-B chunks per W1 (or W3) row
    const int c0 = half * (nchA >> 1), c1 = half ? nchA : (nchA >> 1);
    const float4* xv = reinterpret_cast<const float4*>(xh);
    const int4* w1 = reinterpret_cast<const int4*>(ring + (size_t)sA * SB);
    const int4* w3 = reinterpret_cast<const int4*>(ring + (size_t)sA * SB + 2 * d);
    bool first = true;
    while (true) {
      mbar_wait(full + sA, ph);
      ph ^= 1;
      const int j = meta[sA];
      if (j < 0) break;
      if (f.ts && first && cw == 0 && lane == 0) f.ts[b * 8 + 2] = globaltimer();
      first = false;
      const unsigned long long tp0 = (f.ts && cw == 0) ? globaltimer() : 0ull;
      float2 g = make_float2(0.f, 0.f), u = make_float2(0.f, 0.f);
#pragma unroll 4
      for (int c = c0 + lane; c < c1; c += 32) {
        const float4 xa = xv[2 * c], xb = xv[2 * c + 1];
        g = dot8(w1[c], xa, xb, g);
        u = dot8(w3[c], xa, xb, u);
      }
      const float gs = warp_sum(g.x + g.y);
      const float us = warp_sum(u.x + u.y);
      if (lane == 0) {
        part[4 * sA + 2 * half] = gs;
        part[4 * sA + 2 * half + 1] = us;
      }
      named_bar_sync(2 + sA, 64);          // both halves of stage sA done (reads + partials)
      if (half == 0 && lane == 0) {
        mbar_arrive(empty + sA);
        const float gg = part[4 * sA + 0] + part[4 * sA + 2];   // fixed order: half 0 + half 1
        const float uu = part[4 * sA + 1] + part[4 * sA + 3];
        hglob[h_plane_index(j, ffr)] = gg / (1.0f + expf(-gg)) * uu;
        if (f.ts && cw == 0) f.ts[b * 8 + 6] += globaltimer() - tp0;
      }
    }
    named_bar_sync(2 + sA, 64);
    if (half == 0 && lane == 0) mbar_arrive(empty + sA);  // release the end marker's stage
    if (half == 0 && lane == 0 && (sA & 1) == 0) parB[sA >> 1] = ph;  // full[sA] parity for phase B
  }
  named_bar_sync(1, nthr);
  if (f.ts && cw == 0 && lane == 0) f.ts[b * 8 + 3] = globaltimer();
  if (f.ts && cw == 0 && lane == 0) f.ts[b * 8 + 7] = 0;
  // Per-expert barrier: all h_r rows (written by the gsz CTAs of this group) are visible
  // before any of them is read. Release-RED arrival, acquire spin (PTX memory model:
  // bar.sync + release at gpu scope publishes the whole CTA's writes).
  if (cw == 0 && lane == 0) {
    unsigned long long* bar = f.bar + 16 * r;   // one 128-B line per expert group
    const unsigned long long target = (f.calls + 1) * (unsigned long long)gsz;
    if (f.barmode == 1) {          // experiment: fence + relaxed atomic, relaxed spin + fence
      __threadfence();
      atomicAdd(bar, 1ull);
      while (*((volatile unsigned long long*)bar) < target) __nanosleep(40);
      __threadfence();
    } else if (f.barmode == 2) {   // experiment: release RED, acquire spin without backoff
      red_release_add_u64(bar, 1ull);
      while (ld_acquire_u64(bar) < target) {
      }
    } else {
      red_release_add_u64(bar, 1ull);
      while (ld_acquire_u64(bar) < target) __nanosleep(40);
    }
    if (f.ts) f.ts[b * 8 + 4] = globaltimer();
    // h_r -> shared memory with one bulk copy (the async proxy reads global memory written
    // through the generic proxy by other CTAs: fence the proxies first)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_arrive_expect_tx(hbar, (uint32_t)ffr * 4u);
    bulk_g2s(xh, hglob, (uint32_t)ffr * 4u, hbar, policy_evict_first());
  }
  mbar_wait(hbar, 0);
  {
    const int u = cw >> 2, q = cw & 3;     // super-stage and quarter of the W2 row
    if (u >= NSB) return;                  // (NS odd: the last stage's warps sit out phase B)
    const int s = 2 * u;
    ph = parB[u];
    const int nck = rowB >> 4;
    const int k0 = (nck * q) >> 2, k1 = (nck * (q + 1)) >> 2;
    const float4* hp0 = reinterpret_cast<const float4*>(xh);   // h[8c .. 8c+3]
    const float4* hp1 = hp0 + (ffr >> 3);                      // h[8c+4 .. 8c+7]
    const int4* wv = reinterpret_cast<const int4*>(ring + (size_t)s * SB);
    const float w = swgt;
    while (true) {
      mbar_wait(full + s, ph);
      ph ^= 1;
      const int c = meta[s];
      if (c < 0) break;
      const unsigned long long tp0 = (f.ts && cw == 0) ? globaltimer() : 0ull;
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll 4
      for (int cc = k0 + lane; cc < k1; cc += 32) acc = dot8(wv[cc], hp0[cc], hp1[cc], acc);
      const float sum = warp_sum(acc.x + acc.y);
      if (lane == 0) part[4 * u + q] = sum;
      named_bar_sync(2 + u, 128);          // the 4 quarters of this row are done
      if (q == 0 && lane == 0) {
        mbar_arrive(empty + s);
        const float o = ((part[4 * u] + part[4 * u + 1]) + part[4 * u + 2]) + part[4 * u + 3];
        if (K == 1) a.y[c] = w * o;
        else red_add_f32(a.y + c, w * o);  // K == 2: 0 + a + b is order-independent
        if (f.ts && cw == 0) f.ts[b * 8 + 7] += globaltimer() - tp0;
      }
      named_bar_sync(2 + u, 128);          // partials consumed before they are overwritten
    }
  }
  if (f.ts && cw == 0 && lane == 0) f.ts[b * 8 + 5] = globaltimer();
  griddep_launch_dependents();
}

}  // namespace

cudaError_t preload_fused_kernels() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, expert_fused_kernel);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(expert_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kFusedMaxDynSmem);
}

bool plan_fused(int d, int ffr, int K, int grid, FusedPlan* p) {
  if (K > 2 || grid < K) return false;          // deterministic combine needs K <= 2
  const int SB = max(16384, 4 * d);              // one W1+W3 row pair per stage
  if (2 * ffr > 2 * SB) return false;            // a W2 row fits one super-stage (2 stages)
  const int xh = ((max(4 * d, ffr * 4) + 127) / 128) * 128;   // x (fp32) | one expert's h (fp32)
  const int tail = 2 * kMaxNS * 8 + 8 + kMaxNS * 4 + kMaxNS * 16 + kMaxNS * 4 + 64;
  int NS = (kFusedMaxDynSmem - xh - tail) / SB;
  if (NS > kMaxNS) NS = kMaxNS;
  NS &= ~1;                                      // stages pair into super-stages in phase B
  if (NS < 4) return false;
  p->SB = SB;
  p->NS = NS;
  p->xh_bytes = xh;
  p->ypart_bytes = 0;
  p->smem = (size_t)NS * SB + xh + tail;
  p->threads = kThreadsF;
  p->partB = 2 * ffr;
  p->copiesB = 1;
  return p->smem <= (size_t)kFusedMaxDynSmem;
}

cudaError_t launch_expert_fused(const FusedArgs& f, const FusedPlan& p, int grid, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(p.threads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeCooperative;
  at[na].val.cooperative = 1;
  ++na;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, expert_fused_kernel, f);
}

}  // namespace moe
