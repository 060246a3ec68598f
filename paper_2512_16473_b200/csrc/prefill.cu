// prefill.cu — f4: router, cache pass and batching for a prompt of T tokens.
//
// Semantics: moe_layer_prefill(x[T]) == T successive moe_layer_forward calls on the rows
// of x for everything the cache sees (routing, hit/miss/evict sequence, counters, trace,
// token indices; S:120 decode order), while the expert FFN runs batched per distinct
// routed expert on the tensor cores (prefill_gemm.cu). Requires full associativity
// (M = n, so no expert is evicted inside the batch and every expert keeps one slot).
//
// With M = n nothing is evicted, so the sequential cache semantics decompose into
// parallel steps (same decisions as the sequential walk; GPU parity tests vs the oracle):
//  prefill_route_kernel   per token: logits, top-K, softmax, first access key per expert
//  prefill_plan_kernel    resident experts, ways of first-touch experts in access order,
//                         fills (mailbox), plan blocks (expert id order, 128-row padded)
//  prefill_access_kernel  per token: hit = resident before or touched by an earlier token;
//                         trace, counters, LRU clock of each access (hits then misses)
//  prefill_lists_kernel   per expert: its tokens in order (block scan), final stamps/clock
//  prefill_gather_kernel  X_g[row] = x[tok[row]] (zeros on padding rows)
#include <math.h>

#include "gate_gemv.cuh"
#include "moe_internal.cuh"
#include "ptx.cuh"
#include "route_core.cuh"

namespace moe {
namespace {


// Scratch of one prefill call (device), initialised with cudaMemset(0x7f / 0):
struct PfScratch {
  int first[MOE_MAX_EXPERTS];                 // first access key t*K + r of expert e (0x7f7f7f7f: none)
  int cnt[MOE_MAX_EXPERTS];                   // routed (t, r) entries of expert e
  unsigned long long lastc[MOE_MAX_EXPERTS];  // LRU: clock of the last access of expert e
  int way[MOE_MAX_EXPERTS];                   // way holding e after the call
  int isnew[MOE_MAX_EXPERTS];                 // 1: e was not resident before the call (first touch = miss)
  int newrank[MOE_MAX_EXPERTS];               // order of e among the new experts (by first key)
  int offs[MOE_MAX_EXPERTS];                  // row offset of e's block in X_g
  unsigned long long clock0;
  int nnew;
  // M < n (evictions inside the prompt): the set before and after the replayed accesses
  int tag0[MOE_MAX_EXPERTS], tag1[MOE_MAX_EXPERTS];
  uint32_t gen0[MOE_MAX_EXPERTS], gen1[MOE_MAX_EXPERTS];
  int mn;  // 1: this call takes the M < n path (lists kernel leaves stamps and clock alone)
};

// (1) one CTA per token: logits z = Wg x_t in the decode path's order (gate_gemv.cuh), then
//     warp 0 takes top-K by (z desc, index asc), softmax over the K in rank
//     order (exactly the decode router's arithmetic order for the softmax), first access key
//     and entry count per expert.
__global__ void __launch_bounds__(256) prefill_route_kernel(const PrefillArgs a, const uint16_t* __restrict__ Wg,
                                                            const uint16_t* __restrict__ x, int d) {
  __shared__ float zpart[kGateWarpsMax * MOE_MAX_EXPERTS];
  const int t = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (t >= a.T) return;
  PfScratch* sc = reinterpret_cast<PfScratch*>(a.scratch);
  const int n = a.n, K = a.K;
  // logits in the decode path's summation order (gate_gemv.cuh): the 8 warps evaluate the
  // a.gw virtual warps (w, w + 8, ...), warp 0 sums them in order — so near-tied logits
  // round exactly as in moe_layer_forward and the routing is the same (moe.h)
  gate_virtual_warps(Wg, x + (size_t)t * d, d, n, a.gw, warp, 8, zpart);
  __syncthreads();
  if (warp != 0) return;
  const float zl = lane < n ? gate_sum_warps(zpart + lane, n, a.gw) : 0.f;
  if (a.zbuf && lane < n) a.zbuf[(size_t)t * n + lane] = zl;  // M < n: replayed by prefill_seq_kernel
  const float z = lane < n ? zl : -INFINITY;
  bool taken = lane >= n;
  int myS = -1;
  float myZ = 0.f;
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
    if (lane == r) { myS = idx; myZ = v; }
  }
  const float m = __shfl_sync(0xffffffffu, myZ, 0);
  float sum = 0.f, mine = 0.f;
  for (int r = 0; r < K; ++r) {
    const float e = expf(__shfl_sync(0xffffffffu, myZ, r) - m);
    sum += e;
    if (lane == r) mine = e;
  }
  if (lane < K) {
    a.rt_e[(size_t)t * K + lane] = myS;
    a.rt_w[(size_t)t * K + lane] = mine / sum;
    atomicMin(&sc->first[myS], t * K + lane);
    atomicAdd(&sc->cnt[myS], 1);
  }
}

// (2) one CTA: which experts are resident, ways for the first-touch experts (lowest invalid
//     way, in access order — R10 with M = n), fills (mailbox), plan blocks, directory tags.
__global__ void __launch_bounds__(64) prefill_plan_kernel(const PrefillArgs a) {
  // the walk below is serial and short (n, M <= 32): its inputs are staged in shared memory
  // by parallel loads first, so it does not pay a dependent global-memory round trip per step
  __shared__ int cnt[MOE_MAX_EXPERTS], first[MOE_MAX_EXPERTS], way[MOE_MAX_EXPERTS], tag[MOE_MAX_EXPERTS];
  __shared__ uint32_t gen[MOE_MAX_EXPERTS];
  PfScratch* sc = reinterpret_cast<PfScratch*>(a.scratch);
  const int n = a.n, M = a.M, i = threadIdx.x;
  if (i < n) {
    cnt[i] = sc->cnt[i];
    first[i] = sc->first[i];
  }
  if (i < M) {
    tag[i] = a.tag[i];
    gen[i] = a.gen[a.slot_base + i];
  }
  __syncthreads();
  if (i != 0) return;
  sc->clock0 = *a.clock;
  int nnew = 0;
  int isnew[MOE_MAX_EXPERTS];
  for (int e = 0; e < n; ++e) {
    way[e] = -1;
    isnew[e] = 0;
  }
  for (int w = 0; w < M; ++w)
    if (tag[w] >= 0 && tag[w] < n) way[tag[w]] = w;
  // first-touch experts in access order (selection by first key; n <= 32)
  const bool mailbox = a.miss_mode != MOE_MISS_PULL;  // PULL: a pull kernel fills the slots
  uint32_t done = 0;
  while (true) {
    int best = -1;
    for (int e = 0; e < n; ++e)
      if (!((done >> e) & 1u) && cnt[e] > 0 && way[e] < 0 && (best < 0 || first[e] < first[best])) best = e;
    if (best < 0) break;
    done |= 1u << best;
    int v = -1;
    for (int w = 0; w < M && v < 0; ++w)
      if (tag[w] == -1) v = w;
    tag[v] = best;
    way[best] = v;
    isnew[best] = 1;
    sc->newrank[best] = nnew;
    const uint32_t g = gen[v] + 1u;
    gen[v] = g;
    a.gen[a.slot_base + v] = g;
    a.tag[v] = best;
    if (mailbox) {
      a.mail->expert[nnew] = best;
      a.mail->slot[nnew] = a.slot_base + v;
      a.mail->gen[nnew] = g;
      a.mail->rank[nnew] = 0;
      a.mail->postfetch[nnew] = 1;
      a.mail->dest[nnew] = 0;
    }
    ++nnew;
  }
  sc->nnew = nnew;
  // plan: blocks in expert id order, 128-row padded
  int nb = 0, off = 0, mt = 0;
  for (int e = 0; e < n; ++e) {
    sc->way[e] = way[e];
    sc->isnew[e] = isnew[e];
    if (!cnt[e]) continue;
    const int tiles = (cnt[e] + 127) / 128;
    a.plan->row_off[nb] = off;
    a.plan->mt_pref[nb] = mt;
    a.plan->slot[nb] = a.slot_base + way[e];
    a.plan->gen[nb] = gen[way[e]];
    a.plan->wait[nb] = isnew[e];
    a.plan->expert[nb] = e;
    a.plan->stage[nb] = 0;
    sc->offs[e] = off;
    off += tiles * 128;
    mt += tiles;
    ++nb;
  }
  a.plan->mt_pref[nb] = mt;
  a.plan->nblk = nb;
  a.plan->total_mtiles = mt;
  a.plan->rows = off;
  // fills of the first-touch experts (mailbox: payload, system fence, seq) and the call's
  // progress word, published here, as soon as the entry is final: every later step of the
  // call may fail or be cancelled without leaving the fetch thread waiting for this seq
  if (nnew && mailbox) {
    a.mail->layer = a.layer;
    a.mail->nmiss = nnew;
    a.mail->host = 0;
    __threadfence_system();
    a.mail->seq = a.seq;
    __threadfence_system();
  }
  *a.last_seq = a.seq;
}

// (3) one warp per token: hit/miss (pre-access partition: hit iff resident before the call
//     or first touched by an earlier token), ways, trace records, counters, LRU clocks
//     (every access increments the clock: hits of the token first, then its misses, each
//     in rank order — the decode router's order).
__global__ void __launch_bounds__(256) prefill_access_kernel(const PrefillArgs a) {
  // per-CTA aggregation in shared memory (8 tokens), then one global atomic per counter and
  // per touched expert: the global atomics no longer serialise on a handful of addresses
  __shared__ unsigned long long cs[6];  // accesses, >=1 hit, all-K hit, hits, misses
  __shared__ unsigned long long lastc_s[MOE_MAX_EXPERTS];
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const PfScratch* sc = reinterpret_cast<const PfScratch*>(a.scratch);
  PfScratch* scw = reinterpret_cast<PfScratch*>(a.scratch);
  const int K = a.K;
  if (threadIdx.x < 6) cs[threadIdx.x] = 0ull;
  if (threadIdx.x < MOE_MAX_EXPERTS) lastc_s[threadIdx.x] = 0ull;
  __syncthreads();
  int e = -1, hit = 0;
  if (t < a.T && lane < K) {
    e = a.rt_e[(size_t)t * K + lane];
    hit = !sc->isnew[e] || (sc->first[e] / K) < t;
  }
  const unsigned hm = __ballot_sync(0xffffffffu, lane < K && hit && t < a.T);
  const unsigned mm = __ballot_sync(0xffffffffu, lane < K && !hit && t < a.T);
  if (t < a.T && lane < K) {
    const int pos = hit ? __popc(hm & ((1u << lane) - 1u)) : __popc(hm) + __popc(mm & ((1u << lane) - 1u));
    if (a.policy == MOE_POLICY_LRU)
      atomicMax(&lastc_s[e], sc->clock0 + (unsigned long long)t * K + pos + 1);
    const long long ti = a.trace_idx + (long long)t * K + lane;
    if (ti < a.trace_cap) {
      moe_access_record rec;
      rec.token = a.token0 + (uint32_t)t;
      rec.layer = (uint16_t)a.layer;
      rec.rank = (uint8_t)lane;
      rec.hit = (uint8_t)hit;
      rec.expert = (int16_t)e;
      rec.evicted = -1;
      rec.way = (int8_t)sc->way[e];
      rec.coverage = 0;
      rec.reserved = 0;
      rec.weight = a.rt_w[(size_t)t * K + lane];
      a.trace[ti] = rec;
    }
  }
  if (lane == 0 && t < a.T) {
    const int nh = __popc(hm);
    atomicAdd(&cs[0], 1ull);
    if (nh > 0) atomicAdd(&cs[1], 1ull);
    if (nh == K) atomicAdd(&cs[2], 1ull);
    if (nh) atomicAdd(&cs[3], (unsigned long long)nh);
    if (K - nh) atomicAdd(&cs[4], (unsigned long long)(K - nh));
  }
  __syncthreads();
  if (threadIdx.x < MOE_MAX_EXPERTS && lastc_s[threadIdx.x])
    atomicMax(&scw->lastc[threadIdx.x], lastc_s[threadIdx.x]);
  if (threadIdx.x == 0) {
    DevStats* s = a.stats;
    if (cs[0]) atomicAdd(&s->accesses, cs[0]);
    if (cs[1]) atomicAdd(&s->at_least_one_hit, cs[1]);
    if (cs[2]) atomicAdd(&s->all_k_hit, cs[2]);
    if (cs[3]) atomicAdd(&s->expert_hits, cs[3]);
    if (cs[4]) {
      atomicAdd(&s->expert_misses, cs[4]);
      atomicAdd(&s->fetches, cs[4]);
      atomicAdd(&s->fetch_bytes, cs[4] * (unsigned long long)a.slot_bytes);
    }
  }
}

// (4) per expert e (one CTA each): its tokens in token order -> rows [offs[e], ...) of the
//     gathered batch (block-wide scan), padding rows; block 0 also commits recency stamps
//     and the clock (LRU: clock of each expert's last access; FIFO: insertion order).
__global__ void __launch_bounds__(1024) prefill_lists_kernel(const PrefillArgs a) {
  __shared__ int part[1024];
  const PfScratch* sc = reinterpret_cast<const PfScratch*>(a.scratch);
  const int e = blockIdx.x, K = a.K, T = a.T;
  if (e == 0 && threadIdx.x < a.n && !sc->mn) {
    const int ex = threadIdx.x;
    if (sc->cnt[ex] > 0) {
      if (a.policy == MOE_POLICY_LRU) a.stamp[sc->way[ex]] = sc->lastc[ex];
      else if (sc->isnew[ex]) a.stamp[sc->way[ex]] = sc->clock0 + sc->newrank[ex] + 1;
    }
    if (threadIdx.x == 0)
      *a.clock = sc->clock0 + (a.policy == MOE_POLICY_LRU ? (unsigned long long)T * K : (unsigned long long)sc->nnew);
  }
  if (e >= a.n || sc->cnt[e] == 0) return;
  const int per = (T + blockDim.x - 1) / blockDim.x;
  const int t0 = threadIdx.x * per, t1 = min(T, t0 + per);
  int c = 0;
  for (int t = t0; t < t1; ++t)
    for (int r = 0; r < K; ++r) c += a.rt_e[(size_t)t * K + r] == e;
  part[threadIdx.x] = c;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // inclusive scan (Hillis-Steele)
    const int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int pos = sc->offs[e] + part[threadIdx.x] - c;
  for (int t = t0; t < t1; ++t)
    for (int r = 0; r < K; ++r)
      if (a.rt_e[(size_t)t * K + r] == e) {
        a.plan->tok[pos] = t;
        a.plan->wrow[pos] = a.rt_w[(size_t)t * K + r];
        ++pos;
      }
  if (threadIdx.x == blockDim.x - 1) {
    const int end = sc->offs[e] + ((sc->cnt[e] + 127) / 128) * 128;
    for (int p = sc->offs[e] + sc->cnt[e]; p < end; ++p) {
      a.plan->tok[p] = -1;
      a.plan->wrow[p] = 0.f;
    }
  }
}

// ---- M < n: the prompt's accesses can evict, so the cache pass is the decode router's own
// decision (route_core.cuh) replayed token by token by one warp, with the set's state kept in
// registers between tokens: routing (from the batched router's logits, the shared summation
// order), hit/miss, LRU/FIFO update, victims, trace records and counters are those of T
// successive moe_layer_forward calls by construction. The expert FFN then runs batched per
// distinct routed expert: experts resident at the end of the prompt are read from their
// (re)filled slots, the others from the prefill staging area (prefill_plan_mn_kernel).
__global__ void __launch_bounds__(32) prefill_seq_kernel(const PrefillArgs a) {
  __shared__ int sS[kMaxK];
  __shared__ float sZ[MOE_MAX_EXPERTS], sW[kMaxK];
  PfScratch* sc = reinterpret_cast<PfScratch*>(a.scratch);
  const int lane = threadIdx.x;
  RouteArgs ra;
  memset(&ra, 0, sizeof(ra));
  ra.d = 0; ra.n = a.n; ra.K = a.K; ra.M = a.M; ra.layer = a.layer; ra.covered = 1; ra.policy = a.policy;
  ra.miss_mode = MOE_MISS_PULL;  // (no mailbox entries: the plan below decides the physical fills)
  ra.tag = a.tag; ra.stamp = a.stamp; ra.slot_base = a.slot_base; ra.staging_base = a.staging_base;
  ra.gen = a.gen; ra.ready = a.ready; ra.clock = a.clock; ra.stats = a.stats; ra.trace = a.trace;
  ra.trace_cap = a.trace_cap; ra.slot_bytes = a.slot_bytes;
  DirState ds = dir_load(ra, lane);
  if (lane < a.M) {
    sc->tag0[lane] = ds.tag;
    sc->gen0[lane] = ds.gen;
  }
  if (lane == 0) {
    sc->mn = 1;
    sc->clock0 = ds.clock;
  }
  float znext = lane < a.n ? a.zbuf[lane] : 0.f;
  for (int t = 0; t < a.T; ++t) {
    const float z = znext;
    if (t + 1 < a.T && lane < a.n) znext = a.zbuf[(size_t)(t + 1) * a.n + lane];  // next token's logits in flight
    ra.token = a.token0 + (uint32_t)t;
    ra.trace_idx = a.trace_idx + (long long)t * a.K;
    LaneRoute lr;
    DirState nx;
    route_decide(ra, z, ds, true, sS, sZ, sW, &lr, nullptr, NoEarlyRoute(), &nx);
    ds.tag = nx.tag;
    ds.stamp = nx.stamp;
    ds.gen = nx.gen;
    ds.clock = nx.clock;
  }
  if (lane < a.M) {
    sc->tag1[lane] = ds.tag;
    sc->gen1[lane] = ds.gen;
  }
}

// M < n: plan blocks (expert id order) and the physical fills. A routed expert resident at
// the end of the prompt in way v is read from slot v; it needs a fill unless it already sat in
// v before the prompt with no insertion into v since (same generation). Every other routed
// expert gets a prefill staging slot and a fill (staging generation = the call's seq).
__global__ void __launch_bounds__(32) prefill_plan_mn_kernel(const PrefillArgs a) {
  PfScratch* sc = reinterpret_cast<PfScratch*>(a.scratch);
  if (threadIdx.x != 0) return;
  const int n = a.n, M = a.M;
  const bool mailbox = a.miss_mode != MOE_MISS_PULL;
  int nb = 0, off = 0, mt = 0, nfill = 0, nst = 0;
  for (int e = 0; e < n; ++e) {
    const int cnt = sc->cnt[e];
    if (!cnt) continue;
    int v = -1;
    for (int w = 0; w < M; ++w)
      if (sc->tag1[w] == e) v = w;
    int slot, stage, fill;
    uint32_t g;
    if (v >= 0) {
      slot = a.slot_base + v;
      stage = 0;
      g = sc->gen1[v];
      fill = !(sc->tag0[v] == e && sc->gen0[v] == g);
    } else {
      slot = nst++;
      stage = 1;
      g = (uint32_t)a.seq;
      fill = 1;
    }
    const int tiles = (cnt + 127) / 128;
    a.plan->row_off[nb] = off;
    a.plan->mt_pref[nb] = mt;
    a.plan->slot[nb] = slot;
    a.plan->gen[nb] = g;
    a.plan->wait[nb] = fill;
    a.plan->expert[nb] = e;
    a.plan->stage[nb] = stage;
    sc->offs[e] = off;
    off += tiles * 128;
    mt += tiles;
    ++nb;
    if (fill && mailbox) {
      a.mail->expert[nfill] = e;
      a.mail->slot[nfill] = slot;
      a.mail->gen[nfill] = g;
      a.mail->rank[nfill] = 0;
      a.mail->postfetch[nfill] = 1;
      a.mail->dest[nfill] = stage;
    }
    nfill += fill;
  }
  a.plan->mt_pref[nb] = mt;
  a.plan->nblk = nb;
  a.plan->total_mtiles = mt;
  a.plan->rows = off;
  if (nfill && mailbox) {
    a.mail->layer = a.layer;
    a.mail->nmiss = nfill;
    a.mail->host = 0;
    __threadfence_system();
    a.mail->seq = a.seq;
    __threadfence_system();
  }
  *a.last_seq = a.seq;
}

__global__ void __launch_bounds__(256) prefill_gather_kernel(const uint16_t* __restrict__ x, int d,
                                                             const PrefillPlan* __restrict__ plan,
                                                             uint16_t* __restrict__ xg, int rows_cap) {
  const int row = blockIdx.x;
  if (row >= plan->rows || row >= rows_cap) return;
  const int t = plan->tok[row];
  int4* dst = reinterpret_cast<int4*>(xg + (size_t)row * d);
  const int4* src = reinterpret_cast<const int4*>(x + (size_t)(t < 0 ? 0 : t) * d);
  for (int c = threadIdx.x; c < (d >> 3); c += blockDim.x) dst[c] = t < 0 ? make_int4(0, 0, 0, 0) : __ldg(src + c);
}

__global__ void publish_seq_kernel(volatile unsigned long long* word, unsigned long long seq) { *word = seq; }

}  // namespace

cudaError_t launch_publish_seq(volatile unsigned long long* word, unsigned long long seq, cudaStream_t s) {
  publish_seq_kernel<<<1, 1, 0, s>>>(word, seq);
  return cudaGetLastError();
}

cudaError_t preload_prefill_kernels() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, prefill_route_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, prefill_plan_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, prefill_access_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, prefill_lists_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, prefill_gather_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, publish_seq_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, prefill_seq_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, prefill_plan_mn_kernel);
  return e;
}

size_t prefill_scratch_bytes() { return sizeof(PfScratch); }

cudaError_t launch_prefill_route(const PrefillArgs& a, const uint16_t* Wg, const uint16_t* x, int d,
                                 cudaStream_t s) {
  // first[] = 0x7f7f7f7f (no access yet), the rest zero
  cudaError_t e = cudaMemsetAsync(a.scratch, 0, sizeof(PfScratch), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.scratch, 0x7f, sizeof(int) * MOE_MAX_EXPERTS, s);
  if (e != cudaSuccess) return e;
  const int blocks = (a.T + 7) / 8;
  prefill_route_kernel<<<a.T, 256, 0, s>>>(a, Wg, x, d);
  if (a.M < a.n) {  // evictions inside the prompt: replay the accesses in order
    prefill_seq_kernel<<<1, 32, 0, s>>>(a);
    prefill_plan_mn_kernel<<<1, 32, 0, s>>>(a);
  } else {
    prefill_plan_kernel<<<1, 64, 0, s>>>(a);
    prefill_access_kernel<<<blocks, 256, 0, s>>>(a);
  }
  prefill_lists_kernel<<<a.n, 1024, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_prefill_gather(const uint16_t* x, int d, const PrefillPlan* plan, uint16_t* xg, int rows_cap,
                                  cudaStream_t s) {
  prefill_gather_kernel<<<rows_cap, 128, 0, s>>>(x, d, plan, xg, rows_cap);
  return cudaGetLastError();
}

}  // namespace moe
