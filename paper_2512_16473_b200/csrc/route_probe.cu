// route_probe.cu — K1: fused router + cache probe + on-device LRU update (sm_100a).
//
// One CTA per call. Warps compute the gate GEMV z = Wg x (16-byte loads, fp32
// accumulation, warp-shuffle reduction). Warp 0 then does, with one lane per expert
// and one lane per way:
//   top-K by (z desc, index asc) and softmax over the K           (R1, R2)
//   step 1 cache check of set `layer` against the pre-access state (R10)
//   LRU restamp of hits, then victim/insert of misses in rank order,
//   never evicting a way that holds an expert of this access       (R10)
//   layers >= N: coverage misses into staging slots, no insertion   (R13)
// and writes the route record (for the expert kernels), the access trace, the
// per-layer counters and the miss mailbox (host-mapped; P:200's post-fetch is issued
// by the runtime's fetch thread from it).
#include <math.h>

#include "moe_internal.cuh"
#include "ptx.cuh"

namespace moe {
namespace {

using ptx::griddep_launch_dependents;
using ptx::griddep_wait;

__device__ __forceinline__ float bf_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

__device__ __forceinline__ float dot8_bf16(const int4 a, const int4 b) {
  float s = bf_lo(a.x) * bf_lo(b.x);
  s = fmaf(bf_hi(a.x), bf_hi(b.x), s);
  s = fmaf(bf_lo(a.y), bf_lo(b.y), s);
  s = fmaf(bf_hi(a.y), bf_hi(b.y), s);
  s = fmaf(bf_lo(a.z), bf_lo(b.z), s);
  s = fmaf(bf_hi(a.z), bf_hi(b.z), s);
  s = fmaf(bf_lo(a.w), bf_lo(b.w), s);
  s = fmaf(bf_hi(a.w), bf_hi(b.w), s);
  return s;
}

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kPF = 8;  // gate chunks per lane prefetched into registers before the PDL wait

__global__ void __launch_bounds__(kThreads) route_probe_kernel(const RouteArgs a) {
  __shared__ float part[MOE_MAX_EXPERTS][kWarps + 1];
  __shared__ int sS[kMaxK];
  __shared__ float sZ[kMaxK], sW[kMaxK];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- gate GEMV z = Wg x: G = 32/n warps per expert row, lane-strided 16-B chunks.
  // The gate rows do not depend on x, so they are loaded BEFORE griddepcontrol.wait and
  // overlap the tail of the preceding kernel (programmatic dependent launch).
  const int n = a.n;
  const int G = kWarps / n;                 // n <= 32 -> G >= 1
  const int e = warp / G, g = warp - e * G;
  const bool active = e < n;
  const int nchunk = a.d >> 3;
  const int stride = 32 * G;
  const int c0 = g * 32 + lane;
  const int4* wr = reinterpret_cast<const int4*>(a.Wg + (size_t)(active ? e : 0) * a.d);
  int4 wv[kPF];
#pragma unroll
  for (int k = 0; k < kPF; ++k) {
    const int c = c0 + k * stride;
    if (active && c < nchunk) wv[k] = __ldg(wr + c);
  }
  // The set of this layer was last written by the router kernel of an EARLIER call, which
  // completed before the previous expert kernel passed its own griddepcontrol.wait, i.e.
  // before this grid could launch: it can be read before this grid's wait, too.
  int32_t dtag = -2;
  unsigned long long dstamp = 0ull, dclock = 0ull;
  uint32_t dgen = 0u, dsgen = 0u;
  if (warp == 0) {
    if (a.covered) {
      if (lane < a.M) {
        dtag = a.tag[lane];
        dstamp = a.stamp[lane];
        dgen = a.gen[a.slot_base + lane];
      }
      dclock = *a.clock;
    }
    if (lane < a.K) dsgen = a.gen[a.staging_base + lane];  // staging slot of rank `lane`
  }
  griddep_launch_dependents();  // let the expert kernel's CTAs get resident early
  griddep_wait();               // x (written by the caller's previous kernel) is visible now
  if (a.sched_zero && threadIdx.x < 2 * kMaxK) a.sched_zero[threadIdx.x] = 0u;
  if (a.y_zero)                 // the fused expert kernel accumulates the K experts into y
    for (int i = threadIdx.x; i < (a.d >> 2); i += kThreads)
      reinterpret_cast<float4*>(a.y_zero)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  const int4* xv = reinterpret_cast<const int4*>(a.x);
  float acc = 0.f;
  if (active) {
#pragma unroll
    for (int k = 0; k < kPF; ++k) {
      const int c = c0 + k * stride;
      if (c < nchunk) acc += dot8_bf16(wv[k], __ldg(xv + c));
    }
    for (int c = c0 + kPF * stride; c < nchunk; c += stride) acc += dot8_bf16(__ldg(wr + c), __ldg(xv + c));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && active) part[e][g] = acc;
  __syncthreads();
  if (warp != 0) return;
  float zsum = 0.f;
  if (lane < n)
    for (int q = 0; q < G; ++q) zsum += part[lane][q];  // fixed order: deterministic

  const int K = a.K, M = a.M;
  // ---- top-K: K rounds of warp argmax, ties -> lower expert index
  const float z = lane < n ? zsum : -INFINITY;
  bool taken = lane >= n;
  for (int r = 0; r < K; ++r) {
    float v = taken ? -INFINITY : z;
    int idx = taken ? 0x7fffffff : lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
    if (lane == idx) taken = true;
    if (lane == 0) { sS[r] = idx; sZ[r] = v; }
  }
  __syncwarp();
  // ---- softmax over the K selected logits (rank order, fp32)
  if (lane == 0) {
    const float m = sZ[0];
    float sum = 0.f;
    for (int r = 0; r < K; ++r) { sW[r] = expf(sZ[r] - m); sum += sW[r]; }
    for (int r = 0; r < K; ++r) sW[r] = sW[r] / sum;
  }
  __syncwarp();

  // ---- cache probe + LRU update (lane = way)
  int myS = lane < K ? sS[lane] : -1;  // lane r < K carries rank r's decision
  int myHit = 0, myWay = -1, myEv = -1, mySlot = 0;
  uint32_t myGen = 0;
  unsigned long long clock = 0;
  int nhit = 0, nev = 0;
  if (a.covered) {
    int32_t tag = dtag;
    unsigned long long st = dstamp;
    uint32_t gen = dgen;
    clock = dclock;
    // step 1: partition against the pre-access state
    for (int r = 0; r < K; ++r) {
      const unsigned m = __ballot_sync(0xffffffffu, lane < M && tag == sS[r]);
      if (lane == r) { myHit = m != 0u; myWay = m ? __ffs(m) - 1 : -1; }
    }
    const bool is_static = a.policy == MOE_POLICY_STATIC_RANDOM;
    // step 2: touch hits in rank order (LRU; FIFO keeps insertion order; STATIC never changes)
    for (int r = 0; r < K; ++r) {
      const int h = __shfl_sync(0xffffffffu, myHit, r);
      const int w = __shfl_sync(0xffffffffu, myWay, r);
      if (h && a.policy == MOE_POLICY_LRU) {
        ++clock;
        if (lane == w) st = clock;
      }
    }
    // step 3: insert misses in rank order (STATIC: never; the miss is staged like an
    // uncovered layer's, "stored in the cache statically")
    for (int r = 0; r < K && !is_static; ++r) {
      if (__shfl_sync(0xffffffffu, myHit, r)) continue;
      const unsigned inval = __ballot_sync(0xffffffffu, lane < M && tag == -1);
      int v;
      if (inval) {
        v = __ffs(inval) - 1;
      } else {
        bool pinned = false;
        for (int q = 0; q < K; ++q) pinned |= (tag == sS[q]);
        const bool cand = lane < M && !pinned;
        unsigned long long key = cand ? st : ~0ull;
        int kl = cand ? lane : 64;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
          const int ol = __shfl_xor_sync(0xffffffffu, kl, o);
          if (ok < key || (ok == key && ol < kl)) { key = ok; kl = ol; }
        }
        v = kl;
      }
      const int ev = __shfl_sync(0xffffffffu, tag, v);
      ++clock;
      if (lane == v) { tag = sS[r]; st = clock; ++gen; }
      if (lane == r) { myWay = v; myEv = ev; }
    }
    // write the set back; per-rank slot / generation
    if (lane < M && !is_static) {
      a.tag[lane] = tag;
      a.stamp[lane] = st;
      a.gen[a.slot_base + lane] = gen;
    }
    const int wq = myWay < 0 ? 0 : myWay;
    const uint32_t g = __shfl_sync(0xffffffffu, gen, wq);
    if (lane < K) {
      if (is_static && !myHit) {
        mySlot = a.staging_base + lane;
        myGen = dsgen + 1u;
        a.gen[mySlot] = myGen;
      } else {
        mySlot = a.slot_base + myWay;
        myGen = g;
      }
    }
  } else {
    // beyond coverage: every expert is fetched into a staging slot, never inserted
    if (lane < K) {
      mySlot = a.staging_base + lane;
      myGen = dsgen + 1u;
      a.gen[mySlot] = myGen;
    }
  }
  // Miss handling (moe.h): FETCH — the slot (or staging slot) is filled, the expert kernel
  // waits for it; HOST_COMPUTE — the host computes the missed expert, covered
  // misses are post-fetched into their victim slot for future calls, and a hit on a slot
  // whose post-fetch has not landed waits for it (hit-under-fill).
  const bool hostmode = a.miss_mode == MOE_MISS_HOST_COMPUTE;
  const bool is_static_pol = a.policy == MOE_POLICY_STATIC_RANDOM;
  int myWait = 0, myHost = 0, myPost = 0;
  if (lane < K) {
    if (myHit) {
      if (hostmode) myWait = *((volatile const uint32_t*)(a.ready + mySlot)) < myGen;
    } else if (hostmode) {
      myHost = 1;
      myPost = a.covered && !is_static_pol;
    } else {
      myWait = 1;
      myPost = 1;
    }
  }
  nhit = __popc(__ballot_sync(0xffffffffu, lane < K && myHit));
  nev = __popc(__ballot_sync(0xffffffffu, lane < K && myEv >= 0));
  const int nhuf = __popc(__ballot_sync(0xffffffffu, lane < K && myHit && myWait));
  const int npost = __popc(__ballot_sync(0xffffffffu, lane < K && myPost));
  const unsigned missmask = __ballot_sync(0xffffffffu, lane < K && !myHit);
  if (hostmode && missmask)  // ship x to host memory for the host-side expert computation
    for (int i = lane; i < (a.d >> 3); i += 32)
      reinterpret_cast<int4*>(a.xmail)[i] = reinterpret_cast<const int4*>(a.x)[i];

  // ---- route record, trace, mailbox
  if (lane < K) {
    a.route->expert[lane] = myS;
    a.route->w[lane] = sW[lane];
    a.route->slot[lane] = mySlot;
    a.route->gen[lane] = myGen;
    a.route->wait[lane] = myWait;
    a.route->host[lane] = myHost;
    if (a.trace_idx + lane < a.trace_cap) {
      moe_access_record rec;
      rec.token = a.token;
      rec.layer = (uint16_t)a.layer;
      rec.rank = (uint8_t)lane;
      rec.hit = (uint8_t)myHit;
      rec.expert = (int16_t)myS;
      rec.evicted = (int16_t)myEv;
      rec.way = (int8_t)myWay;
      rec.coverage = (uint8_t)(!a.covered);
      rec.reserved = 0;
      rec.weight = sW[lane];
      a.trace[a.trace_idx + lane] = rec;
    }
    if (!myHit) {
      const int i = __popc(missmask & ((1u << lane) - 1u));
      a.mail->expert[i] = myS;
      a.mail->slot[i] = mySlot;
      a.mail->gen[i] = myGen;
      a.mail->rank[i] = lane;
      a.mail->postfetch[i] = myPost;
    }
  }
  const int nmiss = K - nhit;
  if (lane == 0) {
    a.route->K = K;
    if (a.covered) *a.clock = clock;
    // Counters: fire-and-forget reductions (RED), so the critical path never waits on
    // the read-modify-write round trips.
    DevStats* s = a.stats;
    atomicAdd(&s->accesses, 1ull);
    if (nhit > 0) atomicAdd(&s->at_least_one_hit, 1ull);
    if (nhit == K) atomicAdd(&s->all_k_hit, 1ull);
    if (nhit) atomicAdd(&s->expert_hits, (unsigned long long)nhit);
    if (nmiss) atomicAdd(&s->expert_misses, (unsigned long long)nmiss);
    if (npost) {
      atomicAdd(&s->fetches, (unsigned long long)npost);
      atomicAdd(&s->fetch_bytes, (unsigned long long)npost * (unsigned long long)a.slot_bytes);
    }
    if (hostmode && nmiss) atomicAdd(&s->host_computed, (unsigned long long)nmiss);
    if (!a.covered) atomicAdd(&s->coverage_misses, (unsigned long long)K);
    if (nev) atomicAdd(&s->evictions, (unsigned long long)nev);
    // hit_under_fill is 0 in FETCH mode by construction: a miss is filled before its own
    // call reads the slot, so no later access can find it still filling.
    if (nhuf) atomicAdd(&s->hit_under_fill, (unsigned long long)nhuf);
    if (nmiss) {
      a.mail->layer = a.layer;
      a.mail->nmiss = nmiss;
      a.mail->host = hostmode;
    }
  }
  __syncwarp();
  if (lane == 0 && a.route_flag) {
    // Hand the route to the expert kernel without waiting for this grid to complete: the
    // record, the zeroed y / work counters (written before the CTA barrier) and everything
    // this grid's griddepcontrol.wait made visible are released at gpu scope.
    __threadfence();
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a.route_flag), "l"(a.seq) : "memory");
  }
  if (lane == 0) {
    // Miss mailbox (host-mapped): an entry is written only when this call missed (payload,
    // system fence, seq). The progress word is published by the expert kernel at its end
    // (off this kernel's critical path): progress >= seq implies this kernel completed, so
    // an entry for seq is visible if it exists.
    if (nmiss) {
      __threadfence_system();
      a.mail->seq = a.seq;
    }
  }
}

__global__ void write_ready_kernel(uint32_t* ready, int slot, uint32_t gen) {
  *((volatile uint32_t*)(ready + slot)) = gen;
}

}  // namespace

cudaError_t preload_route_kernels() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, route_probe_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, write_ready_kernel);
  return e;
}

cudaError_t launch_route_probe(const RouteArgs& a, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, route_probe_kernel, a);
}

void launch_write_ready(uint32_t* ready, int slot, uint32_t gen, cudaStream_t s) {
  write_ready_kernel<<<1, 1, 0, s>>>(ready, slot, gen);
}

}  // namespace moe
