// prefill.cu — f4: router, cache pass and batching for a prompt of T tokens.
//
// Semantics: moe_layer_prefill(x[T]) == T successive moe_layer_forward calls on the rows
// of x for everything the cache sees (routing, hit/miss/evict sequence, counters, trace,
// token indices; S:120 decode order), while the expert FFN runs batched per distinct
// routed expert on the tensor cores (prefill_gemm.cu). Requires full associativity
// (M = n, so no expert is evicted inside the batch and every expert keeps one slot).
//
//  prefill_logits_kernel  z[t][e] = Wg x_t                     one warp per (t, e)
//  prefill_cache_kernel   warp 0 walks the tokens in order:    top-K + softmax (R1, R2),
//                         probe + LRU/FIFO update (R10) exactly as the decode
//                         router; then the CTA builds the plan: per distinct expert its
//                         tokens (token order) in 128-row padded blocks, gate weights, slot
//  prefill_gather_kernel  X_g[row] = x[tok[row]] (zeros on padding rows)
#include <math.h>

#include "moe_internal.cuh"
#include "ptx.cuh"

namespace moe {
namespace {

__device__ __forceinline__ float bfl(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bfh(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

__global__ void __launch_bounds__(256) prefill_logits_kernel(const uint16_t* __restrict__ Wg,
                                                             const uint16_t* __restrict__ x, int T, int n, int d,
                                                             float* __restrict__ z) {
  const int gw = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (gw >= T * n) return;
  const int t = gw / n, e = gw - t * n;
  const int4* wr = reinterpret_cast<const int4*>(Wg + (size_t)e * d);
  const int4* xv = reinterpret_cast<const int4*>(x + (size_t)t * d);
  float acc = 0.f;
  for (int c = lane; c < (d >> 3); c += 32) {
    const int4 a = __ldg(wr + c), b = __ldg(xv + c);
    acc = fmaf(bfl(a.x), bfl(b.x), acc);
    acc = fmaf(bfh(a.x), bfh(b.x), acc);
    acc = fmaf(bfl(a.y), bfl(b.y), acc);
    acc = fmaf(bfh(a.y), bfh(b.y), acc);
    acc = fmaf(bfl(a.z), bfl(b.z), acc);
    acc = fmaf(bfh(a.z), bfh(b.z), acc);
    acc = fmaf(bfl(a.w), bfl(b.w), acc);
    acc = fmaf(bfh(a.w), bfh(b.w), acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) z[(size_t)t * n + e] = acc;
}

__global__ void __launch_bounds__(256) prefill_cache_kernel(const PrefillArgs a) {
  __shared__ int cnt[MOE_MAX_EXPERTS];
  __shared__ int offs[MOE_MAX_EXPERTS + 1];
  __shared__ int bslot[MOE_MAX_EXPERTS];
  __shared__ uint32_t bgen[MOE_MAX_EXPERTS];
  __shared__ int bwait[MOE_MAX_EXPERTS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = a.n, K = a.K, M = a.M, T = a.T;
  if (threadIdx.x < MOE_MAX_EXPERTS) { cnt[threadIdx.x] = 0; bwait[threadIdx.x] = 0; }
  __syncthreads();
  if (warp == 0) {
    // ---- sequential pass in token order: identical decisions to T decode calls
    int32_t tag = lane < M ? a.tag[lane] : -2;
    unsigned long long st = lane < M ? a.stamp[lane] : 0ull;
    uint32_t gen = lane < M ? a.gen[a.slot_base + lane] : 0u;
    unsigned long long clock = *a.clock;
    unsigned long long nacc = 0, n1 = 0, nall = 0, nhitt = 0, nmisst = 0, nev = 0;
    int nmail = 0;
    for (int t = 0; t < T; ++t) {
      const float z = lane < n ? a.z[(size_t)t * n + lane] : -INFINITY;
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
      // softmax over the K (rank order, fp32): lane 0 computes like the decode router
      float w = 0.f;
      {
        const float m = __shfl_sync(0xffffffffu, myZ, 0);
        float sum = 0.f, mine = 0.f;
        for (int r = 0; r < K; ++r) {
          const float e = expf(__shfl_sync(0xffffffffu, myZ, r) - m);
          sum += e;
          if (lane == r) mine = e;
        }
        w = mine / sum;
      }
      // probe against the pre-access state
      int myHit = 0, myWay = -1, myEv = -1;
      for (int r = 0; r < K; ++r) {
        const int sr = __shfl_sync(0xffffffffu, myS, r);
        const unsigned m = __ballot_sync(0xffffffffu, lane < M && tag == sr);
        if (lane == r) { myHit = m != 0u; myWay = m ? __ffs(m) - 1 : -1; }
      }
      for (int r = 0; r < K; ++r) {  // touch hits (LRU)
        const int h = __shfl_sync(0xffffffffu, myHit, r);
        const int wv = __shfl_sync(0xffffffffu, myWay, r);
        if (h && a.policy == MOE_POLICY_LRU) {
          ++clock;
          if (lane == wv) st = clock;
        }
      }
      for (int r = 0; r < K; ++r) {  // insert misses (M = n: an invalid way always exists)
        if (__shfl_sync(0xffffffffu, myHit, r)) continue;
        const int sr = __shfl_sync(0xffffffffu, myS, r);
        const unsigned inval = __ballot_sync(0xffffffffu, lane < M && tag == -1);
        int v;
        if (inval) {
          v = __ffs(inval) - 1;
        } else {  // unreachable with M = n; kept for the general rule (R10)
          bool pinned = false;
          for (int q = 0; q < K; ++q) pinned |= (tag == __shfl_sync(0xffffffffu, myS, q));
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
        if (lane == v) { tag = sr; st = clock; ++gen; }
        if (lane == r) { myWay = v; myEv = ev; }
      }
      const int wq = myWay < 0 ? 0 : myWay;
      const uint32_t g = __shfl_sync(0xffffffffu, gen, wq);
      const int nh = __popc(__ballot_sync(0xffffffffu, lane < K && myHit));
      const unsigned missm = __ballot_sync(0xffffffffu, lane < K && !myHit);
      const int ne = __popc(__ballot_sync(0xffffffffu, lane < K && myEv >= 0));
      if (lane < K) {
        a.rt_e[(size_t)t * K + lane] = myS;
        a.rt_w[(size_t)t * K + lane] = w;
        const long long ti = a.trace_idx + (long long)t * K + lane;
        if (ti < a.trace_cap) {
          moe_access_record rec;
          rec.token = a.token0 + (uint32_t)t;
          rec.layer = (uint16_t)a.layer;
          rec.rank = (uint8_t)lane;
          rec.hit = (uint8_t)myHit;
          rec.expert = (int16_t)myS;
          rec.evicted = (int16_t)myEv;
          rec.way = (int8_t)myWay;
          rec.coverage = 0;
          rec.reserved = 0;
          rec.weight = w;
          a.trace[ti] = rec;
        }
        if (!myHit) {  // first touch: fill the expert's slot (one mailbox entry per call)
          const int i = nmail + __popc(missm & ((1u << lane) - 1u));
          a.mail->expert[i] = myS;
          a.mail->slot[i] = a.slot_base + myWay;
          a.mail->gen[i] = g;
          a.mail->rank[i] = lane;
          a.mail->postfetch[i] = 1;
          bwait[myS] = 1;
        }
        bslot[myS] = a.slot_base + myWay;
        bgen[myS] = g;
        atomicAdd(&cnt[myS], 1);
      }
      nmail += __popc(missm);
      nacc += 1;
      n1 += nh > 0;
      nall += nh == K;
      nhitt += nh;
      nmisst += K - nh;
      nev += ne;
      __syncwarp();
    }
    if (lane < M) {
      a.tag[lane] = tag;
      a.stamp[lane] = st;
      a.gen[a.slot_base + lane] = gen;
    }
    if (lane == 0) {
      *a.clock = clock;
      DevStats* s = a.stats;
      atomicAdd(&s->accesses, nacc);
      atomicAdd(&s->at_least_one_hit, n1);
      atomicAdd(&s->all_k_hit, nall);
      atomicAdd(&s->expert_hits, nhitt);
      atomicAdd(&s->expert_misses, nmisst);
      atomicAdd(&s->fetches, nmisst);
      atomicAdd(&s->fetch_bytes, nmisst * (unsigned long long)a.slot_bytes);
      atomicAdd(&s->evictions, nev);
      if (nmail) {
        a.mail->layer = a.layer;
        a.mail->nmiss = nmail;
        a.mail->host = 0;
        __threadfence_system();
        a.mail->seq = a.seq;
      }
    }
  }
  __syncthreads();
  // ---- plan: distinct experts in id order, 128-row padded blocks
  if (threadIdx.x == 0) {
    int nb = 0, off = 0, mt = 0;
    for (int e = 0; e < n; ++e) {
      if (!cnt[e]) continue;
      const int tiles = (cnt[e] + 127) / 128;
      a.plan->row_off[nb] = off;
      a.plan->mt_pref[nb] = mt;
      a.plan->slot[nb] = bslot[e];
      a.plan->gen[nb] = bgen[e];
      a.plan->wait[nb] = bwait[e];
      offs[e] = off;
      off += tiles * 128;
      mt += tiles;
      ++nb;
    }
    a.plan->mt_pref[nb] = mt;
    a.plan->nblk = nb;
    a.plan->total_mtiles = mt;
    a.plan->rows = off;
  }
  __syncthreads();
  if (threadIdx.x < n && cnt[threadIdx.x]) {  // tokens of expert e, in token order
    const int e = threadIdx.x;
    int pos = offs[e];
    for (int t = 0; t < T; ++t)
      for (int r = 0; r < K; ++r)
        if (a.rt_e[(size_t)t * K + r] == e) {
          a.plan->tok[pos] = t;
          a.plan->wrow[pos] = a.rt_w[(size_t)t * K + r];
          ++pos;
        }
    const int end = offs[e] + ((cnt[e] + 127) / 128) * 128;
    for (; pos < end; ++pos) {
      a.plan->tok[pos] = -1;
      a.plan->wrow[pos] = 0.f;
    }
  }
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
  cudaError_t e = cudaFuncGetAttributes(&fa, prefill_logits_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, prefill_cache_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, prefill_gather_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, publish_seq_kernel);
  return e;
}

cudaError_t launch_prefill_route(const PrefillArgs& a, const uint16_t* Wg, const uint16_t* x, int d,
                                 cudaStream_t s) {
  const int warps = a.T * a.n;
  prefill_logits_kernel<<<(warps + 7) / 8, 256, 0, s>>>(Wg, x, a.T, a.n, d, a.z);
  prefill_cache_kernel<<<1, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_prefill_gather(const uint16_t* x, int d, const PrefillPlan* plan, uint16_t* xg, int rows_cap,
                                  cudaStream_t s) {
  prefill_gather_kernel<<<rows_cap, 128, 0, s>>>(x, d, plan, xg, rows_cap);
  return cudaGetLastError();
}

}  // namespace moe
