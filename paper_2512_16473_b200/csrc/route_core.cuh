// route_core.cuh — the routing decision of one decode call, as ONE warp's device code,
// shared by the standalone router kernel (route_probe.cu: split path) and the fused
// single-kernel decode (expert_fused.cu, where every CTA evaluates it redundantly from the
// same inputs and CTA 0 alone performs the side effects).
//
// Given the gate logits z (lane e < n holds z_e) and the layer's cache set as it was
// before this access, with one lane per expert and one lane per way:
//   top-K by (z desc, index asc) and softmax over the K           (R1, R2)
//   step 1 cache check of set `layer` against the pre-access state (R10)
//   LRU restamp of hits, then victim/insert of misses in rank order,
//   never evicting a way that holds an expert of this access       (R10)
//   layers >= N: coverage misses into staging slots, no insertion   (R13)
//   miss handling: FETCH (wait for the fill) or HOST_COMPUTE        (R19-R21)
// Every value of the decision is a deterministic function of (z, directory state), so all
// CTAs that evaluate it agree bit for bit. With `writer`, the warp also writes the set
// back, the generations, the access trace, the per-layer counters, the miss mailbox
// payload (not its seq) and, in HOST_COMPUTE mode, ships x to the host.
#pragma once
#include <math.h>

#include "moe_internal.cuh"

namespace moe {

// Directory state of the call's set, one lane per way (lane < M), read before the access.
struct DirState {
  int32_t tag = -2;
  unsigned long long stamp = 0ull, clock = 0ull;
  uint32_t gen = 0u;    // generation of the lane's way slot
  uint32_t sgen = 0u;   // generation of staging slot `lane` (lane < K)
};

__device__ __forceinline__ DirState dir_load(const RouteArgs& a, int lane) {
  DirState s;
  if (a.covered) {
    if (lane < a.M) {
      s.tag = a.tag[lane];
      s.stamp = a.stamp[lane];
      s.gen = a.gen[a.slot_base + lane];
    }
    s.clock = *a.clock;
  }
  if (lane < a.K) s.sgen = a.gen[a.staging_base + lane];
  return s;
}

// Decision of routing rank `lane` (valid for lane < K).
struct LaneRoute {
  int expert = -1;
  float w = 0.f;
  int slot = 0;
  uint32_t gen = 0u;
  int wait = 0;   // 1: wait until ready[slot] >= gen before reading the slot
  int host = 0;   // 1: computed by the host cores (HOST_COMPUTE miss)
};

struct NoEarlyRoute {
  __device__ void operator()(const LaneRoute&) const {}
};

// One full warp. sS/sW: per-warp shared scratch of >= K entries, sZ of >= n entries. Returns
// the number of misses (the writer publishes the mailbox seq itself, after its own ordering
// needs). When every routed expert hits, `early(lr)` is called (by the whole warp, lane r <
// K holding rank r's final slot, generation and wait flag — not yet its gate weight) as
// soon as the slots are known, before the softmax and the cache bookkeeping: the caller
// may start streaming then.
// `next` (optional): the set's state after this access (tag/stamp/gen per way lane, clock),
// for callers that replay several accesses in a row (moe_layer_prefill with M < n).
template <class Early = NoEarlyRoute>
__device__ __forceinline__ int route_decide(const RouteArgs& a, const float zsum, const DirState& ds,
                                            const bool writer, int* sS, float* sZ, float* sW, LaneRoute* out,
                                            unsigned long long* dts = nullptr, Early early = Early(),
                                            DirState* next = nullptr) {
  const int lane = threadIdx.x & 31;
  const int n = a.n, K = a.K, M = a.M;
  // ---- top-K by (z desc, index asc): lane e counts the experts that precede it (one
  // pass over the n logits in shared memory, all lanes in parallel); rank < K is selected
  if (lane < n) sZ[lane] = zsum;
  __syncwarp();
  int rank = 0;
#pragma unroll 8
  for (int j = 0; j < n; ++j) {  // branch-free compares (broadcast loads pipeline)
    const float zj = sZ[j];
    rank += (int)((zj > zsum) | ((zj == zsum) & (j < lane)));
  }
  if (lane < n && rank < K) { sS[rank] = lane; sW[rank] = zsum; }  // sW: selected logits for now
  __syncwarp();
  if (dts && lane == 0) dts[0] = clock64();

  // ---- cache probe (lane = way), step 1: partition against the pre-access state
  const int myS = lane < K ? sS[lane] : -1;  // lane r < K carries rank r's decision
  int myHit = 0, myWay = -1, myEv = -1, mySlot = 0;
  uint32_t myGen = 0;
  unsigned long long clock = 0;
  int32_t tag = ds.tag;
  unsigned long long st = ds.stamp;
  uint32_t gen = ds.gen;
  if (a.covered) {
    clock = ds.clock;
    for (int r = 0; r < K; ++r) {
      const unsigned m = __ballot_sync(0xffffffffu, lane < M && tag == sS[r]);
      if (lane == r) { myHit = m != 0u; myWay = m ? __ffs(m) - 1 : -1; }
    }
    // all K hit: slot and generation of every rank are final already (a hit never changes
    // its way's generation); the gate weights follow below (e.w is not set)
    const uint32_t gw = __shfl_sync(0xffffffffu, gen, myWay < 0 ? 0 : myWay);
    if (__ballot_sync(0xffffffffu, lane < K && myHit) == (K >= 32 ? 0xffffffffu : (1u << K) - 1u)) {
      LaneRoute e;
      if (lane < K) {
        e.expert = myS;
        e.slot = a.slot_base + myWay;
        e.gen = gw;
        e.wait = a.miss_mode == MOE_MISS_HOST_COMPUTE ? *((volatile const uint32_t*)(a.ready + e.slot)) < gw : 0;
        e.host = 0;
      }
      early(e);
    }
  }
  if (dts && lane == 0) dts[1] = clock64();

  // ---- softmax over the K selected logits (rank order, fp32): e_r = exp(z_r - z_0),
  // summed in rank order
  const float er = lane < K ? expf(sW[lane] - sW[0]) : 0.f;
  __syncwarp();
  if (lane < K) sW[lane] = er;
  __syncwarp();
  float wr = 0.f;
  if (lane < K) {
    float sum = 0.f;
    for (int r = 0; r < K; ++r) sum += sW[r];
    wr = er / sum;
  }
  __syncwarp();
  if (lane < K) sW[lane] = wr;
  __syncwarp();

  if (a.covered) {
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
    if (next) {
      next->tag = tag;
      next->stamp = st;
      next->gen = gen;
      next->clock = clock;
      next->sgen = ds.sgen;
    }
    // write the set back; per-rank slot / generation
    if (writer && lane < M && !is_static) {
      a.tag[lane] = tag;
      a.stamp[lane] = st;
      a.gen[a.slot_base + lane] = gen;
    }
    const int wq = myWay < 0 ? 0 : myWay;
    const uint32_t g = __shfl_sync(0xffffffffu, gen, wq);
    if (lane < K) {
      if (is_static && !myHit) {
        mySlot = a.staging_base + lane;
        myGen = ds.sgen + 1u;
        if (writer) a.gen[mySlot] = myGen;
      } else {
        mySlot = a.slot_base + myWay;
        myGen = g;
      }
    }
  } else {
    // beyond coverage: every expert is fetched into a staging slot, never inserted
    if (lane < K) {
      mySlot = a.staging_base + lane;
      myGen = ds.sgen + 1u;
      if (writer) a.gen[mySlot] = myGen;
    }
  }
  // Miss handling (moe.h): FETCH — the slot (or staging slot) is filled, the expert kernel
  // waits for it; HOST_COMPUTE — the host computes the missed expert, covered
  // misses are post-fetched into their victim slot for future calls, and a hit on a slot
  // whose post-fetch has not landed waits for it (hit-under-fill).
  if (dts && lane == 0) dts[2] = clock64();
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
  const int nhit = __popc(__ballot_sync(0xffffffffu, lane < K && myHit));
  const int nmiss = K - nhit;
  if (lane < K) {
    out->expert = myS;
    out->w = sW[lane];
    out->slot = mySlot;
    out->gen = myGen;
    out->wait = myWait;
    out->host = myHost;
  }
  if (!writer) return nmiss;

  const int nev = __popc(__ballot_sync(0xffffffffu, lane < K && myEv >= 0));
  const int nhuf = __popc(__ballot_sync(0xffffffffu, lane < K && myHit && myWait));
  const int npost = __popc(__ballot_sync(0xffffffffu, lane < K && myPost));
  const unsigned missmask = __ballot_sync(0xffffffffu, lane < K && !myHit);
  const bool mailbox = a.miss_mode != MOE_MISS_PULL;  // PULL: the kernel fills the slots itself
  if (hostmode && missmask)  // ship x to host memory for the host-side expert computation
    for (int i = lane; i < (a.d >> 3); i += 32)
      reinterpret_cast<int4*>(a.xmail)[i] = reinterpret_cast<const int4*>(a.x)[i];

  // ---- trace, mailbox payload
  if (lane < K) {
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
    if (!myHit && mailbox) {
      const int i = __popc(missmask & ((1u << lane) - 1u));
      a.mail->expert[i] = myS;
      a.mail->slot[i] = mySlot;
      a.mail->gen[i] = myGen;
      a.mail->rank[i] = lane;
      a.mail->postfetch[i] = myPost;
      a.mail->dest[i] = 0;
    }
  }
  if (lane == 0) {
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
    if (nmiss && mailbox) {
      a.mail->layer = a.layer;
      a.mail->nmiss = nmiss;
      a.mail->host = hostmode;
    }
  }
  return nmiss;
}

// The writer's lane 0, after route_decide: the miss mailbox entry's seq (FETCH /
// HOST_COMPUTE misses: payload, system fence, seq — the fetch thread's trigger), then
// the call's progress word. progress >= seq tells the fetch thread that the entry of seq,
// if any, is visible; without a miss nothing needs ordering, so the all-hit path issues no
// system-scope fence (a fence at the end of the kernel delayed its completion, and with it
// the next call's PDL wait, by ~2 us).
__device__ __forceinline__ void publish_progress(const RouteArgs& a, int nmiss) {
  if (nmiss && a.miss_mode != MOE_MISS_PULL) {
    __threadfence_system();
    a.mail->seq = a.seq;
    __threadfence_system();
  }
  *a.last_seq = a.seq;
}

}  // namespace moe
