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
//    rows c, in balanced contiguous ranges. The barrier between the phases is therefore
//    per expert (the CTAs that produce h_r), and a CTA needs only ONE expert's h in
//    shared memory, which leaves room for a large weight ring;
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

constexpr int kMaxNC = 16;              // consumer warps (one per ring stage; NS <= kMaxNC)
constexpr int kThreadsF = 32 * (kMaxNC + 1);

__device__ __forceinline__ float dot8_bb(const int4 w, const int4 x, float s) {
  s = fmaf(bf_lo(w.x), bf_lo(x.x), s);
  s = fmaf(bf_hi(w.x), bf_hi(x.x), s);
  s = fmaf(bf_lo(w.y), bf_lo(x.y), s);
  s = fmaf(bf_hi(w.y), bf_hi(x.y), s);
  s = fmaf(bf_lo(w.z), bf_lo(x.z), s);
  s = fmaf(bf_hi(w.z), bf_hi(x.z), s);
  s = fmaf(bf_lo(w.w), bf_lo(x.w), s);
  s = fmaf(bf_hi(w.w), bf_hi(x.w), s);
  return s;
}

__device__ __forceinline__ float dot8_bf(const int4 w, const float4 a, const float4 b, float s) {
  s = fmaf(bf_lo(w.x), a.x, s);
  s = fmaf(bf_hi(w.x), a.y, s);
  s = fmaf(bf_lo(w.y), a.z, s);
  s = fmaf(bf_hi(w.y), a.w, s);
  s = fmaf(bf_lo(w.z), b.x, s);
  s = fmaf(bf_hi(w.z), b.y, s);
  s = fmaf(bf_lo(w.w), b.z, s);
  s = fmaf(bf_hi(w.w), b.w, s);
  return s;
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

// Shared-memory plan (bytes):  ring[NS][SB] | xh | ypart | full[NS] empty[NS] hbar
//   xh = x (bf16) in phase A, then this group's h_r (fp32, 2-plane layout) in phase B.
__global__ void __launch_bounds__(kThreadsF, 1) expert_fused_kernel(const FusedArgs f) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ const uint8_t* sbase;
  __shared__ float swgt;
  __shared__ int smiss, sslot;
  __shared__ uint32_t sgen;
  const ExpertArgs& a = f.e;
  const int NS = f.NS, SB = f.SB;
  uint8_t* ring = smem;
  uint8_t* xh = smem + (size_t)NS * SB;
  float* ypart = reinterpret_cast<float*>(xh + f.xh_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(ypart) + f.ypart_bytes);
  uint64_t* empty = full + NS;
  uint64_t* hbar = empty + NS;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.K, d = a.d, ffr = a.ffr;
  const int G = gridDim.x, b = blockIdx.x;
  // expert group of this CTA and its balanced ranges
  const int r = (int)((long long)b * K / G);
  const int gb0 = (int)(((long long)r * G + K - 1) / K);        // first CTA of group r
  const int gb1 = (int)(((long long)(r + 1) * G + K - 1) / K);  // one past the last
  const int gsz = gb1 - gb0, li = b - gb0;
  const int ja = (int)((long long)ffr * li / gsz), jb = (int)((long long)ffr * (li + 1) / gsz);
  const int nA = jb - ja;                       // phase A rows of expert r
  const int c0 = (int)((long long)d * li / gsz), c1 = (int)((long long)d * (li + 1) / gsz);
  const int nB = c1 - c0;                       // phase B rows of expert r
  const int rowB = ffr * 2;                     // bytes of one W2 row
  const int npB = (rowB + SB - 1) / SB;         // ring parts per phase B row
  const long long w2off = 2ll * ffr * d * 2;    // W2 offset in a slot

  if (f.ts && threadIdx.x == 0) f.ts[b * 8 + 0] = globaltimer();
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(hbar, 1);
    fence_mbar_init();
  }
  griddep_wait();  // route record / zeroed y (router kernel) and x (caller) are visible now
  if (f.ts && threadIdx.x == 0) f.ts[b * 8 + 1] = globaltimer();
  if (threadIdx.x == 0) {
    const int slot = a.route->slot[r];
    sslot = slot;
    sgen = a.route->gen[r];
    smiss = a.route->miss[r];
    sbase = a.pool + (long long)slot * a.slot_bytes;
    swgt = a.route->w[r];
  }
  for (int i = threadIdx.x; i < (d >> 3); i += kThreadsF)
    reinterpret_cast<int4*>(xh)[i] = reinterpret_cast<const int4*>(a.x)[i];
  __syncthreads();
  const uint8_t* base = sbase;

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      if (smiss) wait_ready(a.ready, sslot, sgen);  // a hit's fill landed in an earlier call
      int t = 0;
      for (int j = ja; j < jb; ++j, ++t) {
        const int s = t % NS;
        mbar_wait(empty + s, ((t / NS) & 1) ^ 1);
        const uint8_t* w1 = base + (long long)j * d * 2;
        const uint8_t* w3 = w1 + (long long)ffr * d * 2;
        mbar_arrive_expect_tx(full + s, 4u * d);
        bulk_g2s(ring + (size_t)s * SB, w1, 2u * d, full + s, pol);
        bulk_g2s(ring + (size_t)s * SB + 2 * d, w3, 2u * d, full + s, pol);
      }
      for (int i = 0; i < nB; ++i) {  // W2 rows do not depend on h: stream through the barrier
        const uint8_t* row = base + w2off + (long long)(c0 + i) * rowB;
        for (int p = 0; p < npB; ++p, ++t) {
          const int s = t % NS;
          const uint32_t bytes = (uint32_t)min(SB, rowB - p * SB);
          mbar_wait(empty + s, ((t / NS) & 1) ^ 1);
          mbar_arrive_expect_tx(full + s, bytes);
          bulk_g2s(ring + (size_t)s * SB, row + (long long)p * SB, bytes, full + s, pol);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  // Ring part t (phase A row t, then phase B part t - nA) lives in stage t % NS and is
  // consumed by warp t % NS: each consumer warp owns one stage, so its next wait is always
  // exactly one mbarrier phase ahead of the part it just released (parity waits cannot
  // alias) and the producer refills a stage as soon as its owner is done with it.
  const int cw = warp - 1;
  if (cw >= NS) return;
  const int nthr = NS * 32;
  float* hglob = a.h + (long long)r * ffr;
  {
    const int nchA = d >> 3;
    const int4* xv = reinterpret_cast<const int4*>(xh);
    const int4* w1 = reinterpret_cast<const int4*>(ring + (size_t)cw * SB);
    const int4* w3 = reinterpret_cast<const int4*>(ring + (size_t)cw * SB + 2 * d);
    for (int t = cw; t < nA; t += NS) {
      mbar_wait(full + cw, (t / NS) & 1);
      if (f.ts && t == 0 && lane == 0) f.ts[b * 8 + 2] = globaltimer();
      float g0 = 0.f, g1 = 0.f, u0 = 0.f, u1 = 0.f;
#pragma unroll 2
      for (int c = lane; c < nchA; c += 64) {
        const int4 xa = xv[c];
        g0 = dot8_bb(w1[c], xa, g0);
        u0 = dot8_bb(w3[c], xa, u0);
        if (c + 32 < nchA) {
          const int4 xb = xv[c + 32];
          g1 = dot8_bb(w1[c + 32], xb, g1);
          u1 = dot8_bb(w3[c + 32], xb, u1);
        }
      }
      const float g = warp_sum(g0 + g1);
      const float u = warp_sum(u0 + u1);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty + cw);
        hglob[h_plane_index(ja + t, ffr)] = g / (1.0f + expf(-g)) * u;
      }
    }
  }
  named_bar_sync(1, nthr);
  if (f.ts && cw == 0 && lane == 0) f.ts[b * 8 + 3] = globaltimer();
  // Per-expert barrier: all h_r rows (written by the gsz CTAs of this group) are visible
  // before any of them is read. Release-RED arrival, acquire spin (PTX memory model:
  // bar.sync + release at gpu scope publishes the whole CTA's writes).
  if (cw == 0 && lane == 0) {
    unsigned long long* bar = f.bar + r;
    const unsigned long long target = (f.calls + 1) * (unsigned long long)gsz;
    red_release_add_u64(bar, 1ull);
    while (ld_acquire_u64(bar) < target) {
    }
    if (f.ts) f.ts[b * 8 + 4] = globaltimer();
    // h_r -> shared memory with one bulk copy (the async proxy reads global memory written
    // through the generic proxy by other CTAs: fence the proxies first)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_arrive_expect_tx(hbar, (uint32_t)ffr * 4u);
    bulk_g2s(xh, hglob, (uint32_t)ffr * 4u, hbar, policy_evict_first());
  }
  mbar_wait(hbar, 0);
  const float4* hp0 = reinterpret_cast<const float4*>(xh);   // h[8c .. 8c+3]
  const float4* hp1 = hp0 + (ffr >> 3);                      // h[8c+4 .. 8c+7]
  {
    const int4* wv = reinterpret_cast<const int4*>(ring + (size_t)cw * SB);
    const int totB = nB * npB;
    int t = nA + ((cw - nA % NS) % NS + NS) % NS;  // first t >= nA with t % NS == cw
    for (; t < nA + totB; t += NS) {
      const int k = t - nA;
      const int p = k % npB;
      const int nck = min(SB, rowB - p * SB) >> 4;
      const int cb = (p * SB) >> 4;
      mbar_wait(full + cw, (t / NS) & 1);
      float acc0 = 0.f, acc1 = 0.f;
#pragma unroll 2
      for (int cc = lane; cc < nck; cc += 64) {
        acc0 = dot8_bf(wv[cc], hp0[cb + cc], hp1[cb + cc], acc0);
        if (cc + 32 < nck) acc1 = dot8_bf(wv[cc + 32], hp0[cb + cc + 32], hp1[cb + cc + 32], acc1);
      }
      const float acc = warp_sum(acc0 + acc1);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty + cw);
        ypart[k] = acc;
      }
    }
  }
  named_bar_sync(1, nthr);
  if (f.ts && cw == 0 && lane == 0) f.ts[b * 8 + 5] = globaltimer();
  griddep_launch_dependents();
  const float w = swgt;
  for (int i = cw * 32 + lane; i < nB; i += nthr) {
    float o = 0.f;
    for (int p = 0; p < npB; ++p) o += ypart[i * npB + p];
    if (K == 1) a.y[c0 + i] = w * o;
    else red_add_f32(a.y + c0 + i, w * o);  // K == 2: 0 + a + b is order-independent
  }
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
  const int SB = max(16384, 4 * d);
  const int xh = ((max(2 * d, ffr * 4) + 127) / 128) * 128;   // x (bf16) | one expert's h (fp32)
  const int gmin = grid / K;                                  // smallest group
  const int cmax = (d + gmin - 1) / gmin + 1;
  const int npB = (ffr * 2 + SB - 1) / SB;
  const int ypart = ((cmax * npB * 4 + 15) / 16) * 16;
  const int fixed = xh + ypart + 16;
  int NS = (kFusedMaxDynSmem - fixed) / (SB + 16);
  if (NS > kMaxNC) NS = kMaxNC;  // one consumer warp per stage
  if (NS < 3) return false;
  p->SB = SB;
  p->NS = NS;
  p->xh_bytes = xh;
  p->ypart_bytes = ypart;
  p->smem = (size_t)NS * SB + xh + ypart + 2 * NS * 8 + 8;
  p->threads = kThreadsF;
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
