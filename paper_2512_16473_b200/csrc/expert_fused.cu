// expert_fused.cu — K23: the whole expert FFN of one decode step in ONE persistent kernel
// (sm_100a): SwiGLU gate/up GEMVs -> grid barrier -> down GEMV + gate-weighted combine.
//
//   phase A  h_r[j] = silu(W1_r[j,:] x) * (W3_r[j,:] x)              (R4)
//   phase B  y[c]   = sum_r w_r * (W2_r[c,:] h_r)   (rank order)
//
// Decode batch 1 makes every expert matrix a GEMV (~1 FLOP/byte), so this is an HBM
// stream, not a tensor-core contraction. Design for B200:
//  - one CTA per SM (grid = #SMs, cooperative => co-resident), balanced contiguous work
//    ranges: phase A rows (r, j) and phase B output rows c (all K experts of c in one CTA,
//    so the combine is CTA-local and deterministic — no atomics);
//  - warp 0 / lane 0 is a producer that streams weight rows with bulk async copies
//    (cp.async.bulk, the TMA engine's linear path; SASS UBLKCP) into an NS-stage shared
//    memory ring guarded by full/empty mbarriers, L2 evict-first; bytes in flight per SM =
//    the ring (~96 KB), independent of how many consumer warps are still busy, so partial
//    rounds at the end of a range do not starve HBM;
//  - W2 rows do not depend on h, so the producer runs into phase B while the consumers
//    are still in phase A / the grid barrier: the barrier is covered by in-flight W2;
//  - 8 consumer warps: x (bf16) and then h (fp32) live in shared memory; fp32 FMAs,
//    warp-shuffle reductions.
#include <math.h>

#include "moe_internal.cuh"
#include "ptx.cuh"

namespace moe {
namespace {

using namespace ptx;

constexpr int kNC = 8;                  // consumer warps
constexpr int kThreadsF = 32 * (kNC + 1);

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

__global__ void __launch_bounds__(kThreadsF, 1) expert_fused_kernel(const FusedArgs f) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ const uint8_t* base[kMaxK];
  __shared__ float wgt[kMaxK];
  const ExpertArgs& a = f.e;
  const int NS = f.NS, SB = f.SB;
  uint8_t* ring = smem;
  uint8_t* xh = smem + (size_t)NS * SB;                       // x (bf16) in A, h (fp32) in B
  float* ypart = reinterpret_cast<float*>(xh + f.xh_bytes);   // [c1-c0][K]
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(ypart) + f.ypart_bytes);
  uint64_t* empty = full + NS;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.K, d = a.d, ffr = a.ffr;
  const int G = gridDim.x, b = blockIdx.x;
  const long long UA = (long long)K * ffr;
  const long long qa0 = UA * b / G, qa1 = UA * (b + 1) / G;
  const int nA = (int)(qa1 - qa0);
  const int c0 = (int)((long long)d * b / G), c1 = (int)((long long)d * (b + 1) / G);
  const int nc = c1 - c0;
  const int nB = nc * K;                        // phase B items, expert-major: i -> (r = i / nc, c = c0 + i % nc)
  const int rowB = ffr * 2;                     // bytes of one W2 row
  const int npB = (rowB + SB - 1) / SB;         // ring parts per phase B item
  const long long w2off = 2ll * ffr * d * 2;    // W2 offset in a slot

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    fence_mbar_init();
  }
  griddep_wait();  // route record (router kernel) and x (caller) are visible from here on
  if (f.dbg && threadIdx.x == 0) atomicAdd_system(f.dbg + 0, 1u);
  if (threadIdx.x < K) {
    base[threadIdx.x] = a.pool + (long long)a.route->slot[threadIdx.x] * a.slot_bytes;
    wgt[threadIdx.x] = a.route->w[threadIdx.x];
  }
  for (int i = threadIdx.x; i < (d >> 3); i += kThreadsF)
    reinterpret_cast<int4*>(xh)[i] = reinterpret_cast<const int4*>(a.x)[i];
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int r = 0; r < K; ++r) wait_ready(a.ready, a.route->slot[r], a.route->gen[r]);
      int t = 0;
      for (long long q = qa0; q < qa1; ++q, ++t) {
        const int s = t % NS;
        mbar_wait(empty + s, ((t / NS) & 1) ^ 1);
        const int r = (int)(q / ffr), j = (int)(q - (long long)r * ffr);
        const uint8_t* w1 = base[r] + (long long)j * d * 2;
        const uint8_t* w3 = w1 + (long long)ffr * d * 2;
        mbar_arrive_expect_tx(full + s, 4u * d);
        bulk_g2s(ring + (size_t)s * SB, w1, 2u * d, full + s, pol);
        bulk_g2s(ring + (size_t)s * SB + 2 * d, w3, 2u * d, full + s, pol);
      }
      if (f.dbg) atomicAdd_system(f.dbg + 1, 1u);
      for (int i = 0; i < nB; ++i) {
        const int r = i / nc, c = c0 + i % nc;
        const uint8_t* row = base[r] + w2off + (long long)c * rowB;
        for (int p = 0; p < npB; ++p, ++t) {
          const int s = t % NS;
          const uint32_t bytes = (uint32_t)min(SB, rowB - p * SB);
          mbar_wait(empty + s, ((t / NS) & 1) ^ 1);
          mbar_arrive_expect_tx(full + s, bytes);
          bulk_g2s(ring + (size_t)s * SB, row + (long long)p * SB, bytes, full + s, pol);
        }
      }
      if (f.dbg) atomicAdd_system(f.dbg + 2, 1u);
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  // Ring part t (phase A item t, then phase B part t - nA) lives in stage t % NS and is
  // consumed by warp t % NS: each consumer warp owns one stage, so its next wait is always
  // exactly one mbarrier phase ahead of the part it just released (parity waits cannot
  // alias) and the producer refills a stage as soon as its owner is done with it.
  const int cw = warp - 1;
  if (cw >= NS) return;
  const int nchA = d >> 3;
  const int4* xv = reinterpret_cast<const int4*>(xh);
  {
    const int4* w1 = reinterpret_cast<const int4*>(ring + (size_t)cw * SB);
    const int4* w3 = reinterpret_cast<const int4*>(ring + (size_t)cw * SB + 2 * d);
    for (int t = cw; t < nA; t += NS) {
      mbar_wait(full + cw, (t / NS) & 1);
      float g = 0.f, u = 0.f;
#pragma unroll 4
      for (int c = lane; c < nchA; c += 32) {
        const int4 xx = xv[c];
        g = dot8_bb(w1[c], xx, g);
        u = dot8_bb(w3[c], xx, u);
      }
      g = warp_sum(g);
      u = warp_sum(u);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty + cw);
        a.h[qa0 + t] = g / (1.0f + expf(-g)) * u;
      }
    }
  }
  const int nthr = NS * 32;
  named_bar_sync(1, nthr);
  // grid-wide barrier: every h_r[j] is written before any CTA reads h
  if (cw == 0 && lane == 0) {
    if (f.dbg) atomicAdd_system(f.dbg + 3, 1u);
    __threadfence();
    atomicAdd(f.bar, 1ull);
    while (ld_acquire_u64(f.bar) < f.bar_target) __nanosleep(32);
    __threadfence();
  }
  named_bar_sync(1, nthr);
  {
    const float4* hg = reinterpret_cast<const float4*>(a.h);
    float4* hs4 = reinterpret_cast<float4*>(xh);
    for (int i = cw * 32 + lane; i < (K * ffr) >> 2; i += nthr) hs4[i] = __ldcg(hg + i);
  }
  named_bar_sync(1, nthr);
  const float* hs = reinterpret_cast<const float*>(xh);
  const int totB = nB * npB;
  {
    const int4* wv = reinterpret_cast<const int4*>(ring + (size_t)cw * SB);
    int t = nA + ((cw - nA % NS) % NS + NS) % NS;   // first t >= nA with t % NS == cw
    for (; t < nA + totB; t += NS) {
      const int k = t - nA;
      const int i = k / npB, p = k - i * npB;
      const int r = i / nc;
      const int nck = min(SB, rowB - p * SB) >> 4;
      const int cb = (p * SB) >> 4;
      const float4* h4 = reinterpret_cast<const float4*>(hs + (long long)r * ffr) + 2 * cb;
      mbar_wait(full + cw, (t / NS) & 1);
      float acc = 0.f;
#pragma unroll 4
      for (int cc = lane; cc < nck; cc += 32) acc = dot8_bf(wv[cc], h4[2 * cc], h4[2 * cc + 1], acc);
      acc = warp_sum(acc);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty + cw);
        ypart[k] = acc;
      }
    }
  }
  named_bar_sync(1, nthr);
  if (f.dbg && cw == 0 && lane == 0) atomicAdd_system(f.dbg + 4, 1u);
  griddep_launch_dependents();
  for (int cl = cw * 32 + lane; cl < nc; cl += nthr) {
    float y = 0.f;
    for (int r = 0; r < K; ++r) {  // o_r = sum of its parts (fixed order); rank-ordered combine
      const float* pr = ypart + (size_t)(r * nc + cl) * npB;
      float o = 0.f;
      for (int p = 0; p < npB; ++p) o += pr[p];
      y += wgt[r] * o;
    }
    a.y[c0 + cl] = y;
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
  const int SB = max(16384, 4 * d);
  const int xh = max(2 * d, K * ffr * 4);
  const int cmax = (d + grid - 1) / grid;
  const int npB = (ffr * 2 + SB - 1) / SB;
  const int ypart = ((cmax * K * npB * 4 + 15) / 16) * 16;
  const int fixed = xh + ypart;
  int NS = (kFusedMaxDynSmem - fixed) / (SB + 16);
  if (NS > kNC) NS = kNC;  // one consumer warp per stage
  if (NS < 3) return false;
  p->SB = SB;
  p->NS = NS;
  p->xh_bytes = ((xh + 15) / 16) * 16;
  p->ypart_bytes = ypart;
  p->smem = (size_t)NS * SB + p->xh_bytes + ypart + 2 * NS * 8;
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
