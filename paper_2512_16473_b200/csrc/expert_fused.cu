// expert_fused.cu — the whole decode step of one MoE layer in ONE kernel (sm_100a):
// routing (gate GEMV, top-K, softmax, cache probe + LRU/FIFO/static update, miss handling),
// then the SwiGLU expert GEMVs and the gate-weighted combine.
//
//   routing  z = Wg x; S = top-K(z); w = softmax(z_S); set l probed and updated
//   phase A  h_r[j] = silu(W1_r[j,:] x) * (W3_r[j,:] x)              (R4)
//   phase B  y[c]  += w_r * (W2_r[c,:] h_r)
//
// Decode batch 1 makes every expert matrix a GEMV (~1 FLOP/byte): an HBM stream, not a
// tensor-core contraction. Design for B200:
//  - one CTA per SM (grid = #SMs; co-residency checked at init), launched with programmatic
//    dependent launch so the CTAs become resident while the previous call drains. Every CTA
//    takes the routing decision itself from the same inputs (deterministic; CTA 0 alone
//    writes the directory, trace, counters and miss mailbox): gate rows staged before the
//    PDL wait, the GEMV spread over the consumer threads, a router warp publishing the slots
//    through an mbarrier (all-hit fast path straight from the logits);
//  - every CTA works on every routed expert, in the order A_o0, A_o1, B_o0, B_o1 (resident
//    experts before ones still being fetched), rows scheduled static-then-steal (per-SM HBM
//    bandwidth varies by ~10%; the stolen tail evens it out). h_r depends on every CTA's
//    phase-A rows of expert r; B_o0 only starts after A_o1 has streamed, so the grid-wide
//    dependency (per-stage release publications, acquire before the h copy) costs no HBM
//    time;
//  - warp 0 / lane 0 is a producer streaming weight rows with bulk async copies
//    (cp.async.bulk — the TMA engine's linear path, SASS UBLKCP) into an NS-stage shared
//    memory ring guarded by full/empty mbarriers (L2 evict-first): phase A one W1+W3 row pair
//    per stage, phase B RB whole W2 rows per pair of stages. W2 rows do not depend on h, so
//    the producer streams through every phase and expert switch;
//  - consumers: 2 warps per phase-A stage (x as bf16, mixed-precision FMAs), 4 per phase-B
//    pair (h_r as fp32 in a 2-plane layout), fixed-order combination of the partials;
//  - merged phase B (small ff_r: every expert's h fits beside x): the router warp copies each
//    h_r in as soon as it is published and B_o0 / B_o1 stream without a switch;
//  - combine: y (zeroed by every CTA for its slice) += w_r * o_r[c] with fire-and-forget
//    fp32 reductions — K <= 2: two addends onto 0 commute, so y is bit-reproducible; other K
//    take the split path. Tensor parallel (f3): every term goes to every rank as a tagged
//    8-byte word instead, summed in a fixed order in the epilogue.
#include <math.h>

#include "moe_internal.cuh"
#include "gate_gemv.cuh"
#include "ptx.cuh"
#include "pull.cuh"
#include "route_core.cuh"

// Compiled twice: here with the FHFMA form of the gate GEMV (expert_fused_kernel), and from
// expert_fused_mma.cu with MOE_FUSED_MMA_GATE = 1 and its tensor-core form
// (expert_fused_mma_kernel, gate_mma_form(n, d): 9-16 experts). Two translation units so
// that neither kernel carries the other's code: the kernel pays for every instruction in its
// cold paths, and a change of its code layout alone measured 0.1-0.25 us on some shapes.
#ifndef MOE_FUSED_MMA_GATE
#define MOE_FUSED_MMA_GATE 0
#endif
#if MOE_FUSED_MMA_GATE
#define MOE_FUSED_KERNEL expert_fused_mma_kernel
#else
#define MOE_FUSED_KERNEL expert_fused_kernel
#endif

namespace moe {
namespace {

using namespace ptx;

// Debug marks (per-CTA globaltimer / clock64 timestamps, stage events) exist only in the
// debug build (-DMOE_DEBUG_MARKS, lib/libmoe_debug.so, used by tools/timeline.py): the
// production kernel carries none of their code (a kernel this size is sensitive to its
// instruction footprint: +1.3K SASS instructions cost Mixtral ~1 us).
#ifdef MOE_DEBUG_MARKS
#define TS(f) ((f).ts)
#define STS(f) ((f).sts)
#else
#define TS(f) ((unsigned long long*)nullptr)
#define STS(f) ((unsigned long long*)nullptr)
#endif

constexpr int kMaxNS = 10;                 // ring stages (phase B pairs them: NS even)
constexpr int kWarpsPerStage = 2;          // consumer warps sharing one stage
constexpr int kRouterWarp = 1 + kWarpsPerStage * kMaxNS;  // warp 0 producer, 1..2NS consumers
constexpr int kRouteBar = 13;              // named barrier: partial logits -> router warp
constexpr int kThreadsF = 32 * (kRouterWarp + 1);
constexpr int kMaxFusedK = 2;             // deterministic combine: 0 + a + b commutes
static_assert(2 * 2 * kMaxFusedK * kCtrStride == kCtrWords, "work-claim counter layout");
constexpr int kTsPerCta = kTsStride;      // debug timestamps per CTA (MOE_DEBUG_TS)
constexpr int kMaxRB = 16;                // phase B: max W2 rows per super-stage
// back-off of the polls on flags other CTAs set (interleaved A/B: a pure spin was 0.1-0.25 us
// slower per step on small shapes)
#define MOE_POLL_BACKOFF(ns) __nanosleep(ns)
constexpr int kPullBar = 14;
// A ring stage is released by every consumer warp that read it, as soon as its reads are done
// (before the cross-warp reduction of its partials): phase A 2 warps x 2, phase B 4 warps x 1,
// a marker by one thread x 4. The producer can refill the stage ~0.1-0.2 us earlier.
constexpr uint32_t kEmptyArrivals = 4;              // named barrier: consumers' MOE_MISS_PULL copies done
constexpr int kPullCtr = 16 * 8;          // bar[] word counting CTAs done pulling (every call adds G)

// Packed fp32 FMA (sm_100: FFMA2): acc.{x,y} += a.{x,y} * b.{x,y}
__device__ __forceinline__ float2 ffma2(const float2 a, const float2 b, const float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
        "l"(*reinterpret_cast<const unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}

// acc.{x,y} += w.{lo,hi} * x.{lo,hi}: sm_100 mixed-precision FMA (SASS FHFMA.BF16, the
// halves selected in the instruction), bf16 products exact in fp32, one rounding per step
__device__ __forceinline__ float2 fma_bf16x2(const uint32_t w, const uint32_t x, float2 acc) {
  asm("{\n\t.reg .b16 wl, wh, xl, xh;\n\t"
      "mov.b32 {wl, wh}, %2;\n\t"
      "mov.b32 {xl, xh}, %3;\n\t"
      "fma.rn.f32.bf16 %0, wl, xl, %0;\n\t"
      "fma.rn.f32.bf16 %1, wh, xh, %1;\n\t}"
      : "+f"(acc.x), "+f"(acc.y)
      : "r"(w), "r"(x));
  return acc;
}

// acc += w(8 bf16) . x(8 bf16)
__device__ __forceinline__ float2 dot8_bf(const int4 w, const int4 x, float2 acc) {
  acc = fma_bf16x2((uint32_t)w.x, (uint32_t)x.x, acc);
  acc = fma_bf16x2((uint32_t)w.y, (uint32_t)x.y, acc);
  acc = fma_bf16x2((uint32_t)w.z, (uint32_t)x.z, acc);
  acc = fma_bf16x2((uint32_t)w.w, (uint32_t)x.w, acc);
  return acc;
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
__device__ __forceinline__ void red_relaxed_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Relaxed h publication. A gpu-scope release (MEMBAR.GPU) inside this streaming kernel waits
// for the SM's outstanding memory traffic — the ring's bulk loads: ~4 us per release measured
// under a 705 MB stream (tools/fence_cost.cu), and the grid-wide h was complete only at the
// slowest of G x NS such releases (+2-6 us after the stages' last rows). Instead: every h
// word of a call's buffer (double-buffered by call parity) is armed with kHUnset during the
// previous call, writers store h with plain stores and count their segments with relaxed
// REDs (a hint: "probably complete"), and a reader that copied h into shared memory re-reads
// from L2 every word still carrying kHUnset until it is written. kHUnset (0xffffffff, a
// negative NaN) is never produced by arithmetic (the canonical NaN is 0x7fffffff), and aligned
// 4-byte stores are single-copy atomic, so a word is either armed or final.
constexpr uint32_t kHUnset = 0xffffffffu;
constexpr int kYCtr = 16 * 9;             // bar[] word: CTAs whose y slice is zeroed (every call adds G)

__device__ __forceinline__ float ld_relaxed_f32(const float* p) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
// h words [0, n) of a shared-memory copy (thread t of nt): re-read every still-armed word from
// `src` (L2) until it is written. Loads are batched 8 float4 deep with one branch per batch
// (one load-compare-branch chain per float4 made the router warp's scan of Phi's h 5 us).
// debug build only (MOE_DEBUG_STALE_H=1, a fault injection for the tests): before settling,
// re-arm one word of every float4 this thread checks in the shared-memory copy, as if its
// store had not reached L2 when the copy read it; the settle must fetch every one again
__device__ __forceinline__ void inject_stale_h(const FusedArgs& f, float* dst, int n, int t, int nt) {
#ifdef MOE_DEBUG_MARKS
  if (!f.dbg_stale) return;
  for (int i = 4 * t, k = 0; i < n; i += 4 * nt, ++k) dst[i + (k & 3)] = __uint_as_float(kHUnset);
#endif
}

__device__ __noinline__ void settle_h(float* dst, const float* src, int n, int t, int nt) {
  constexpr int U = 8;
  for (int base = 4 * t; base < n; base += 4 * nt * U) {
    float4 v[U];
    bool bad = false;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int i = base + 4 * nt * k;
      v[k] = i < n ? *reinterpret_cast<const float4*>(dst + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      bad |= (__float_as_uint(v[k].x) == kHUnset) | (__float_as_uint(v[k].y) == kHUnset) |
             (__float_as_uint(v[k].z) == kHUnset) | (__float_as_uint(v[k].w) == kHUnset);
    }
    if (!bad) continue;
    const unsigned long long t0 = globaltimer();
    for (int k = 0; k < U; ++k) {
      const int i0 = base + 4 * nt * k;
      if (i0 >= n) break;
      for (int e = 0; e < 4; ++e) {
        float w = dst[i0 + e];
        while (__float_as_uint(w) == kHUnset) {
          w = ld_relaxed_f32(src + i0 + e);
          if (__float_as_uint(w) == kHUnset) {
            MOE_POLL_BACKOFF(32);
            if (globaltimer() - t0 > 60ull * 1000000000ull) __trap();
          }
        }
        dst[i0 + e] = w;
      }
    }
  }
}

// spin until *p >= target (acquire); 60 s -> trap
// One stage's publication of h_r (its rows written with plain stores; readers settle what has
// not landed): the CTA's NS stages count in shared memory and the last of them adds NS to the
// grid-wide counter in one relaxed RED — G instead of G x NS same-address atomics per expert,
// which the L2 serialises (a tiny step saw h complete ~2 us after the last publication)
__device__ __forceinline__ void publish_h(unsigned* spub, unsigned long long* bar, int NS) {
  if (atomicAdd(spub, 1u) == (unsigned)NS - 1u) red_relaxed_add_u64(bar, (unsigned long long)NS);
}

__device__ __forceinline__ void wait_counter(const unsigned long long* p, unsigned long long target) {
  if (ld_acquire_u64(p) >= target) return;
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_u64(p) < target) {
    MOE_POLL_BACKOFF(64);
    if (globaltimer() - t0 > 60ull * 1000000000ull) __trap();
  }
}

// f3: fused tensor-parallel reduction of y over the ranks' exchange buffers (moe.h,
// moe_tp_connect_*), the "LL" low-latency protocol: every term w_r * o_r^(p)[c] of this
// rank's partial y^(p) is stored, as soon as a phase-B row (or a host-computed expert's
// column) is done, into slot [par][c][p][r] of EVERY rank as an 8-byte {value, tag} word
// (tag = this call's number; plain P2P stores over NVLink, a local store for its own rank;
// single-copy atomic, so a receiver that sees the tag sees the value: no fence, no counter,
// no grid barrier). Here, CTA b polls its own slots of its column slice [c0, c1) until every
// (source rank, routing rank) word carries the tag and sums them per column in a fixed tree
// order (K = 2: (v[p][0] + v[p][1]) per source rank, then pairs of ranks): y is
// bit-identical on every rank.
// Slots are double-buffered by call parity: a rank one call ahead writes the other half.
// Exchange slot layout ("tp_slot"): [parity][column][source rank][routing rank] of 8-byte
// words at kTpSlotOff of each rank's buffer — the P*K words a receiver sums are contiguous;
// the tag is (call number + 1) << 32.
// term w_r * o_r[c] of this rank -> every rank's slot (tp_slot's layout). Out of line with
// scalar arguments — the peers' buffers from a shared-memory copy — so that a single-GPU
// step's phase-B loop carries none of its code.
__device__ __noinline__ void tp_push(uint8_t* const* peer, int P, int rank, unsigned long long tp_calls, int K, int d,
                                     int r, int c, float v) {
  const unsigned long long w = ((unsigned long long)(uint32_t)(tp_calls + 1) << 32) | __float_as_uint(v);
  const int par = (int)(tp_calls & 1);
  for (int p = 0; p < P; ++p)
    st_relaxed_sys_u64(reinterpret_cast<unsigned long long*>(peer[p] + kTpSlotOff) + (((long long)par * d + c) * P + rank) * K + r,
                       w);
}
// (out of line with scalar arguments: a single-GPU step never runs it; it reads only this
// rank's own exchange buffer `own`)
__device__ __noinline__ void tp_reduce_epilogue(uint8_t* own, int P, int K, int d, unsigned long long tp_calls,
                                                float* yout, unsigned long long* ts, int b, int G, int ctid,
                                                int nthr) {
  const int PK = P * K;  // PK in {1, 2, 4, 8, 16}: divides 32 and nthr
  const int c0 = (int)((long long)d * b / G), c1 = (int)((long long)d * (b + 1) / G);
  const int total = (c1 - c0) * PK;
  const unsigned long long tag = (unsigned long long)(uint32_t)(tp_calls + 1) << 32;  // (tp_tag)
  const int par = (int)(tp_calls & 1);
  // [parity][column][source rank][routing rank] (tp_slot): the P*K words of a column are contiguous
  const unsigned long long* slots = reinterpret_cast<const unsigned long long*>(own + kTpSlotOff) + (long long)par * d * PK;
  if (ts && ctid == 0) ts[18] = globaltimer();
  // thread i holds word j = i % PK (source rank j / K, routing rank j % K) of column
  // c0 + i / PK: poll it until it carries this call's tag, then an xor-shuffle tree over the
  // PK lanes of the column (a fixed order, the same on every rank)
  constexpr int U = 4;                         // words in flight per thread (poll latency overlap)
  for (int base = 0; base < total; base += U * nthr) {
    unsigned long long w[U];
    const unsigned long long* wp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * nthr + ctid;
      wp[u] = nullptr;
      w[u] = 0ull;
      if (i < total) {
        wp[u] = slots + (long long)c0 * PK + i;
        w[u] = ld_relaxed_sys_u64(wp[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (wp[u] && (w[u] & 0xffffffff00000000ull) != tag) {
        const unsigned long long t0 = globaltimer();
        while (((w[u] = ld_relaxed_sys_u64(wp[u])) & 0xffffffff00000000ull) != tag) {
          MOE_POLL_BACKOFF(32);
          if (globaltimer() - t0 > 60ull * 1000000000ull) __trap();
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * nthr + ctid;
      float v = wp[u] ? __uint_as_float((uint32_t)w[u]) : 0.f;
      for (int o = 1; o < PK; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (i < total && i % PK == 0) yout[c0 + i / PK] = v;
    }
  }
  if (ts && ctid == 0) ts[21] = globaltimer();
}

// This CTA's loads are done: warm L2 with the first rows the NEXT call's phase A will read
// on this CTA (its static block starts at the same row for any expert) for every way of the
// next call's set — the routing of the next call is not known yet, so all ways are touched;
// the bytes move while the other CTAs finish this call (HBM otherwise idles in the tail and
// in the next call's prologue). L2 prefetch only: no effect on results.
__device__ __forceinline__ void prefetch_next(const FusedArgs& f, int b, int G, int ffr, int d) {
  if (!f.next_pool || f.next_rows <= 0) return;
  const int sb = (int)((unsigned)(ffr * f.pctA) / 100u / (unsigned)G);
  const int r0 = b * sb, nr = min(f.next_rows, sb);
  if (nr <= 0) return;
  for (int w = 0; w < f.next_ways; ++w) {
    const uint8_t* slot = f.next_pool + (long long)w * f.e.slot_bytes;
    bulk_prefetch_l2(slot + (long long)r0 * d * 2, (uint32_t)(nr * d * 2));                      // W1 rows
    bulk_prefetch_l2(slot + (long long)(ffr + r0) * d * 2, (uint32_t)(nr * d * 2));              // W3 rows
  }
}

// debug (MOE_DEBUG_TS): a stage's data was seen by its first consumer warp (time, bytes, phase)
__device__ __forceinline__ void record_event(const FusedArgs& f, int* evn, int b, unsigned bytes, unsigned phase) {
#ifndef MOE_DEBUG_MARKS
  return;
#endif
  if (!f.ev) return;
  const int i = atomicAdd(evn, 1);
  if (i < kEvPerCta) {
    f.ev[((long long)b * kEvPerCta + i) * 2] = globaltimer();
    f.ev[((long long)b * kEvPerCta + i) * 2 + 1] = (unsigned long long)bytes | ((unsigned long long)phase << 32);
  }
}

// Paths a single-GPU all-hit decode step never takes live out of line: the kernel is sensitive
// to its instruction footprint (~1 K never-executed instructions in its body cost 0.2-0.5 us
// per step in an interleaved A/B). Scalar arguments only (a reference to the kernel's
// parameter block would be copied to the stack).

// moe_layer_forward_host: x is read straight from the caller's pinned host buffer (one PCIe
// pass, by CTA 0's consumer threads) into the device staging buffer xd, then published to
// every CTA (no copy-engine transfer queued in front of the kernel)
__device__ __noinline__ void xhost_copy(uint16_t* xd, const uint16_t* xhost, uint32_t* xflag, uint32_t xseq, int d,
                                        int i, int nthr) {
  for (int k = i; k < (d >> 3); k += nthr) reinterpret_cast<int4*>(xd)[k] = reinterpret_cast<const int4*>(xhost)[k];
  named_bar_sync(12, nthr);
  if (i == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(xflag), "r"(xseq) : "memory");
  }
}

// MOE_MISS_PULL: this CTA's share of every missed expert's blob, host store -> slot; returns
// whether it copied anything
__device__ __noinline__ bool pull_missed(int K, long long slot_bytes, const uint8_t* const* hblob,
                                         const uint8_t* const* sbase, const int* swait, const int* shost,
                                         const int* sexp, int ctid, int nthr) {
  bool any = false;
  for (int r = 0; r < K; ++r) {
    if (!swait[r] || shost[r]) continue;
    any = true;
    long long u0, u1;
    pull_share(slot_bytes, blockIdx.x, gridDim.x, &u0, &u1);
    pull_copy(const_cast<uint8_t*>(sbase[r]), hblob[sexp[r]], u0, u1, ctid, nthr);
  }
  return any;
}

constexpr int kChunkA = 2;     // phase A rows per tail claim
constexpr int kChunkB = 1;     // phase B rows per tail claim

// Ring-slot meta word: >= 0 a weight chunk (phase A: (si << 24) | j, the W1/W3 row pair j
// of segment si's expert; phase B: (r << 24) | c, W2 rows c .. c + metaN - 1 of expert r);
// kEnd closes a phase; kSegB switches phase B to the next expert (segmented phase B only).
// Phase A has no segment markers: a stage's h writer publishes its rows of a segment when
// it meets the next segment's first row, or at kEnd.
constexpr int kEnd = -1;
constexpr int kSegB = -2;

// Static-then-steal schedule over `total` rows for CTA b of G: the first pct% of
// the rows are split into equal contiguous blocks, the tail is claimed in chunks from a
// per-segment counter, so every CTA ends each segment within about one chunk of the
// others, whatever its share of HBM bandwidth.
struct RowSched {
  int s0, s1;    // this CTA's static block
  int tail0;     // first tail row
};
__device__ __forceinline__ RowSched make_sched(int total, int b, int G, int pct) {
  RowSched rs;
  const int sb = (int)((unsigned)(total * pct) / 100u / (unsigned)G);  // total * pct < 2^31
  rs.s0 = b * sb;
  rs.s1 = rs.s0 + sb;
  rs.tail0 = G * sb;
  return rs;
}

// Shared memory: ring[NS][SB] | xh | full[NS] empty[NS] hbar | meta[NS] | part[NS][4] |
//                parB[NS/2] | metaN[NS] | partB[NS/2][2][kMaxRB][4]
//  - phase A: stage s (16 KB) = one W1 row + one W3 row, consumed by warps 2s, 2s+1 (one
//    half of the row each); x lives in xh as fp32.
//  - phase B: stages (2u, 2u+1) form one super-stage holding a whole W2 row (<= 2*SB),
//    guarded by full[2u]/empty[2u] and consumed by the 4 warps of stages 2u, 2u+1 (a
//    quarter of the row each); h_r lives in xh as fp32 in the 2-plane layout.
//  - partial sums of a stage's warps are combined in a fixed order after a named barrier
//    (deterministic, no atomics). Every consumer warp waits on one mbarrier per phase, and
//    its next wait is always one phase ahead of the part it just released: parity waits
//    cannot alias.
//
// Work order (all CTAs, no group split): phase A of every device-computed expert in turn
// (A_o0, A_o1), then phase B (B_o0, B_o1). h_r is complete once every stage of every CTA
// has moved past segment A_r (the next segment's first row, its own last row, or kEnd); each
// stage's single h writer publishes its rows then (publish_h: the CTA's last stage adds NS to
// bar[r] in one relaxed RED; readers settle words whose plain stores have not landed yet).
// B_o0 starts only after A_o1 has streamed, so its wait on bar[o0] is normally already
// satisfied: the grid-wide dependency costs no HBM time.
__global__ void __launch_bounds__(kThreadsF, 1) MOE_FUSED_KERNEL(const FusedArgs f) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ const uint8_t* sbase[kMaxFusedK];
  __shared__ float swgt[kMaxFusedK];
  __shared__ int swait[kMaxFusedK], shost[kMaxFusedK], sslot[kMaxFusedK], sorder[kMaxFusedK], sexp[kMaxFusedK];
  __shared__ uint32_t sgen[kMaxFusedK];
  __shared__ int snseg, smerged;
  __shared__ int rS[kMaxFusedK];                          // routing scratch (route_decide)
  __shared__ float rZ[MOE_MAX_EXPERTS], rW[kMaxFusedK];
  __shared__ __align__(8) uint64_t gbar, xbar, rbar, wbar;  // gate rows / x landed; slots / weights published
  __shared__ __align__(8) uint64_t hbarK[kMaxFusedK];     // merged phase B: h_r landed and settled (router warp)
  __shared__ __align__(8) uint64_t hrawK[kMaxFusedK];     // merged phase B: h_r's bulk copy landed
  __shared__ __align__(8) uint64_t ybar;                  // segmented phase B: every CTA's y slice zeroed
  __shared__ uint8_t* speer[8];                           // TP: the ranks' exchange buffers (tp_push)
  __shared__ int evn;                                     // debug: stage events recorded this call
  __shared__ volatile int slastA;                         // phase-A items this CTA issued (once known)
  __shared__ unsigned spub[kMaxFusedK];                   // stages that published h_r (publish_h)
  __shared__ __align__(8) uint64_t pairbar[kMaxNS / 2];  // merged phase B: pair u's even stage left phase A
  __shared__ RouteArgs ra;                                // routing arguments (read once, off the critical path)
  const ExpertArgs& a = f.e;
  const int NS = f.NS, SB = f.SB, NSB = NS >> 1;
  uint8_t* ring = smem;
  uint8_t* xh = smem + (size_t)NS * SB;
  uint64_t* full = reinterpret_cast<uint64_t*>(xh + f.xh_bytes);
  uint64_t* empty = full + NS;
  uint64_t* hbar = empty + NS;
  volatile int* meta = reinterpret_cast<volatile int*>(hbar + 1);
  volatile float* part = reinterpret_cast<volatile float*>(meta + NS);   // [NS][2][4] (row parity)
  volatile uint32_t* parB = reinterpret_cast<volatile uint32_t*>(part + 8 * NS);  // full[2u] parity at phase B start
  volatile int* metaN = reinterpret_cast<volatile int*>(parB + (NS >> 1));        // phase B: rows in the super-stage
  volatile float* partB = reinterpret_cast<volatile float*>(metaN + NS);          // [NS/2][2][kMaxRB][4] row partials
  const int RB = f.RB;
  const int RBp = f.RBp;                   // partB row stride (the plan's RB; MOE_ROWS_B may lower RB)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.K, d = a.d, ffr = a.ffr, n = f.r.n;
  const int G = gridDim.x, b = blockIdx.x;
  const int rowA = 4 * d;                       // bytes of one W1 row + one W3 row
  const int rowB = ffr * 2;                     // bytes of one W2 row (<= 2*SB)
  const long long w2off = 2ll * ffr * d * 2;    // W2 offset in a slot
  // bar[r] counts per-stage publications of h_r: G CTAs x NS stages per call
  const unsigned long long bar_target = (f.calls + 1) * (unsigned long long)G * (unsigned long long)NS;
  float* const hcur = f.hf + (long long)(f.calls & 1) * K * ffr;   // this call's h (relaxed publication)
  // work-claim counters of this call ([A r][B r]); the other parity is zeroed for the next
  unsigned* ctr = f.ctr + (f.calls & 1) * (2 * kMaxFusedK) * kCtrStride;  // (one 128-B line per counter)
  // the ring is free until the route is known: it stages the gate rows and x first
  // gate rows at a padded stride (+16 B: the 8 rows of an MMA fragment hit distinct banks)
  const int gstride = 2 * d + 16;
  float* zpart = reinterpret_cast<float*>(ring + (size_t)n * gstride);  // [consumer warp][n] partial logits
  // x (bf16) lives in xh through phase A; phase B reuses xh for h_r (fp32)
  const int cw = warp - 1;                      // consumer warp 0 .. 2*NS-1 (warp 0: producer)
  const int nthr = kWarpsPerStage * NS * 32;
  const int ctid = threadIdx.x - 32;

  if (STS(f) && threadIdx.x == 0) STS(f)[kStsHead + b] = globaltimer();
  if (TS(f) && threadIdx.x == 0) {
    TS(f)[b * kTsPerCta + 0] = globaltimer();
    TS(f)[b * kTsPerCta + 33] = clock64();
    TS(f)[b * kTsPerCta + 6] = 0;
    TS(f)[b * kTsPerCta + 7] = 0;
    TS(f)[b * kTsPerCta + 15] = 0;
    TS(f)[b * kTsPerCta + 16] = 0;
    TS(f)[b * kTsPerCta + 19] = 0;
    TS(f)[b * kTsPerCta + 20] = 0;
    TS(f)[b * kTsPerCta + 22] = 0;
    TS(f)[b * kTsPerCta + 23] = 0;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kEmptyArrivals);
    }
    mbar_init(hbar, 1);
    mbar_init(&gbar, 1);
    mbar_init(&xbar, 1);
    mbar_init(&rbar, 32);  // every router lane arrives after its own shared-memory writes
    mbar_init(&wbar, 32);
    mbar_init(&ybar, 1);
    evn = 0;
    for (int r = 0; r < kMaxFusedK; ++r) spub[r] = 0u;
    slastA = 0x7fffffff;
    for (int r = 0; r < kMaxFusedK; ++r) {
      mbar_init(hbarK + r, 32);             // merged: every router lane after settling its words
      mbar_init(hrawK + r, 1);              // merged: the bulk copy of h_r landed
    }
    for (int u = 0; u < kMaxNS / 2; ++u) mbar_init(pairbar + u, 1);
    fence_mbar_init();
    // the gate rows are weights, constant across calls: stream them in before the PDL wait
    const uint64_t pl = policy_evict_last();
    mbar_arrive_expect_tx(&gbar, (uint32_t)n * 2u * d);
    for (int e = 0; e < n; ++e) bulk_g2s(ring + (size_t)e * gstride, f.r.Wg + (size_t)e * d, 2u * d, &gbar, pl);
    // L2 prefetches while the previous call drains (hints only: L2 is coherent, so a line the
    // previous kernel still writes is never served stale): x, and this CTA's first row pairs
    // of every way of the set (the route is not known yet)
    if (f.pfx && !f.xhost) bulk_prefetch_l2(f.e.x, 2u * d);
    if (f.cur_pool && f.start_rows > 0) {
      const int sb = (int)((unsigned)(f.e.ffr * f.pctA) / 100u / (unsigned)gridDim.x);
      const int r0 = blockIdx.x * sb, nr = min(f.start_rows, sb);
      if (nr > 0)
        for (int w = 0; w < f.cur_ways; ++w) {
          const uint8_t* slot = f.cur_pool + (long long)w * f.e.slot_bytes;
          bulk_prefetch_l2(slot + (long long)r0 * d * 2, (uint32_t)(nr * d * 2));
          bulk_prefetch_l2(slot + (long long)(f.e.ffr + r0) * d * 2, (uint32_t)(nr * d * 2));
        }
    }
  }
  if (threadIdx.x == 32) ra = f.r;  // kernel parameters -> shared memory before the PDL wait
  if (threadIdx.x < 8 && f.tpP > 0) speer[threadIdx.x] = f.peer[threadIdx.x];
  __syncthreads();          // mbarrier inits and routing arguments visible
  const int nwc = kWarpsPerStage * NS;
  // Programmatic dependent launch: the previous call's kernel (cache directory, counters,
  // h) and the caller's x are complete and visible after this wait.
  griddep_wait();
  if (TS(f) && threadIdx.x == 0) TS(f)[b * kTsPerCta + 8] = globaltimer();
  DirState ds;
  if (warp == kRouterWarp) ds = dir_load(ra, lane);  // the router's directory loads in flight
  if (f.xhost && b == 0 && threadIdx.x >= 32 && threadIdx.x < 32 + nthr)
    xhost_copy(const_cast<uint16_t*>(a.x), f.xhost, f.xflag, f.xseq, d, threadIdx.x - 32, nthr);
  if (threadIdx.x == 0) {                    // (host entry: wait for CTA 0's copy of x first)
    const unsigned long long t0 = globaltimer();
    while (f.xhost && (int)(ld_acquire_u32(f.xflag) - f.xseq) < 0) {
      MOE_POLL_BACKOFF(32);
      if (globaltimer() - t0 > 60ull * 1000000000ull) __trap();
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_arrive_expect_tx(&xbar, 2u * d);
    bulk_g2s(xh, a.x, 2u * d, &xbar, policy_evict_last());
  }
  if (b == 0 && threadIdx.x >= 32 && threadIdx.x < 32 + 2 * kMaxFusedK)
    f.ctr[(((f.calls + 1) & 1) * (2 * kMaxFusedK) + threadIdx.x - 32) * kCtrStride] = 0u;
  unsigned long long* pm = TS(f) ? TS(f) + b * kTsPerCta + 24 : nullptr;  // debug marks
  if (cw >= 0 && cw < nwc) {
    // x: one bulk copy into xh (measured faster than per-thread L2 loads of the GEMV's own
    // chunks, which also had to be stored into xh for phase A)
    mbar_wait(&xbar, 0);
    if (TS(f) && threadIdx.x == 32) TS(f)[b * kTsPerCta + 9] = globaltimer();
    if (pm && threadIdx.x == 32) pm[1] = clock64();
    // Gate GEMV z = Wg x: a few KFLOP, latency-bound — spread over every consumer
    // thread instead of a dependent chain of MMAs: thread i takes 16-B chunks i, i + nthr, ...
    // of x and of 8 gate rows at a time (sm_100 mixed-precision FMAs, bf16 products exact
    // in fp32), then a warp reduce-scatter over the 8 experts. Per-warp partials, reduced in a fixed
    // order by the router warp (deterministic).
    mbar_wait(&gbar, 0);
    if (pm && threadIdx.x == 32) pm[0] = clock64();
#if MOE_FUSED_MMA_GATE
    {
      // 9-16 gate rows: the tensor-core form of the shared order (gate_gemv.cuh), virtual
      // warp = consumer warp
      const int g = lane >> 2, c4 = lane & 3;
      const bool hi = g + 8 < n;
      const float2 z = gate_mma_warp(ring + (size_t)g * gstride + 4 * c4,
                                     ring + (size_t)(hi ? g + 8 : g) * gstride + 4 * c4, xh + 4 * c4, d >> 4, cw, nwc);
      if (c4 == 0) {
        zpart[cw * n + g] = z.x;
        if (hi) zpart[cw * n + g + 8] = z.y;
      }
    }
#else
    {
      const int nch = d >> 3;                       // 16-B chunks per row
      const int4* xq = reinterpret_cast<const int4*>(xh);
      for (int e0 = 0; e0 < n; e0 += 8) {
        float2 acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = make_float2(0.f, 0.f);
        for (int ch = ctid; ch < nch; ch += nthr) {
          const int4 xv = xq[ch];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (e0 + j < n)
              acc[j] = dot8_bf(reinterpret_cast<const int4*>(ring + (size_t)(e0 + j) * gstride)[ch], xv, acc[j]);
        }
        // reduce-scatter over the warp (9 shuffles instead of 8 x 5): after the xor-16/8/4
        // steps lane L holds expert 4*L[4] + 2*L[3] + L[2] summed over 8 lanes, then xor-2/1
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = acc[j].x + acc[j].y;
        const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
        float w4[4], w2[2];
#pragma unroll
        for (int i = 0; i < 4; ++i)  // keep half b4 of the 8, send the other half
          w4[i] = (b4 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, b4 ? v[i] : v[i + 4], 16);
#pragma unroll
        for (int i = 0; i < 2; ++i)
          w2[i] = (b3 ? w4[i + 2] : w4[i]) + __shfl_xor_sync(0xffffffffu, b3 ? w4[i] : w4[i + 2], 8);
        float z = (b2 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? w2[0] : w2[1], 4);
        z += __shfl_xor_sync(0xffffffffu, z, 2);
        z += __shfl_xor_sync(0xffffffffu, z, 1);
        const int e = e0 + (b4 ? 4 : 0) + (b3 ? 2 : 0) + (b2 ? 1 : 0);
        if ((lane & 3) == 0 && e < n) zpart[cw * n + e] = z;
      }
    }
#endif
    if (pm && threadIdx.x == 32) pm[2] = clock64();
    named_bar_arrive(kRouteBar, nthr + 32);  // partial logits ready; on to phase A
    if (f.r.miss_mode == MOE_MISS_PULL) {
      // MOE_MISS_PULL: this CTA's share of every missed expert's blob, host store -> slot,
      // before any phase-A row is consumed (the producer streams resident experts meanwhile
      // and waits for every CTA's share before its first row of a pulled expert)
      mbar_wait(&rbar, 0);
      const bool any = pull_missed(K, a.slot_bytes, ra.hblob, sbase, swait, shost, sexp, ctid, nthr);
      if (any) named_bar_sync(kPullBar, nthr);  // (uniform: every consumer read the same route)
      // one arrival per CTA and call (the counter's target is (calls + 1) * G); a release only
      // when this CTA copied bytes (a gpu-scope release costs microseconds here)
      if (ctid == 0) {
        if (any) red_release_add_u64(f.bar + kPullCtr, 1ull);
        else red_relaxed_add_u64(f.bar + kPullCtr, 1ull);
      }
    } else if (ctid == 0) {
      red_relaxed_add_u64(f.bar + kPullCtr, 1ull);
    }
  } else if (warp == kRouterWarp) {
    // ---------------------------------------------------------------- router warp
    // routing decision (route_core.cuh), identical in every CTA; CTA 0 writes its effects.
    // The producer starts as soon as the slots are known (all hit: before the bookkeeping).
    // While the consumers run the gate GEMV: where each expert sits in the set (lane e:
    // its way and that way's generation, from the pre-access directory), so an all-hit
    // route can be published straight from the logits.
    const bool fast = ra.covered && ra.miss_mode != MOE_MISS_HOST_COMPUTE;
    int way_of = -1;
    uint32_t gen_of = 0u;
    if (fast)
      for (int w = 0; w < ra.M; ++w) {
        const int t = __shfl_sync(0xffffffffu, ds.tag, w);
        const uint32_t g = __shfl_sync(0xffffffffu, ds.gen, w);
        if (t == lane) { way_of = w; gen_of = g; }
      }
    named_bar_sync(kRouteBar, nthr + 32);
    if (TS(f) && lane == 0) TS(f)[b * kTsPerCta + 10] = globaltimer();
    if (pm && lane == 0) pm[3] = clock64();
    // the shared logit order (gate_gemv.cuh): virtual warp = consumer warp, summed in order
    // (every lane sums a valid column, branch-free; lanes >= n then drop theirs)
    const float zl = gate_sum_warps(zpart + (lane < n ? lane : 0), n, nwc);
    const float z = lane < n ? zl : 0.f;
    if (pm && lane == 0) pm[11] = clock64();
    bool published = false;
    if (fast) {
      // all-hit fast path: rank of expert `lane` by (z desc, index asc) — the same order
      // route_decide derives from the same z — and, if all K selected experts are resident,
      // their slots in rank order (a hit never changes its way's generation; FETCH: no wait)
      // all shuffles first, then branch-free compares: the shuffles pipeline instead of
      // each waiting for the previous compare (measured ~1300 -> ~100 cycles)
      float zz[MOE_MAX_EXPERTS];
#pragma unroll
      for (int j = 0; j < MOE_MAX_EXPERTS; ++j) zz[j] = __shfl_sync(0xffffffffu, z, j);
      int rank = 0;
#pragma unroll
      for (int j = 0; j < MOE_MAX_EXPERTS; ++j)
        rank += (int)((j < n) & ((zz[j] > z) | ((zz[j] == z) & (j < lane))));
      if (pm && lane == 0) pm[12] = clock64();
      const bool sel = lane < n && rank < K;
      if (__popc(__ballot_sync(0xffffffffu, sel && way_of >= 0)) == K) {
        if (pm && lane == 0) pm[13] = clock64();
        if (sel) {
          const int slot = ra.slot_base + way_of;
          sslot[rank] = slot;
          sgen[rank] = gen_of;
          swait[rank] = 0;
          shost[rank] = 0;
          sbase[rank] = a.pool + (long long)slot * a.slot_bytes;
          sorder[rank] = rank;
          sexp[rank] = lane;
        }
        if (lane == 0) {
          snseg = K;
          smerged = f.merge && K == kMaxFusedK;  // every expert resident and ready
        }
        mbar_arrive(&rbar);                // release (each lane its own writes): route published
        if (pm && lane == 0) pm[8] = clock64();
        if (TS(f) && lane == 0) TS(f)[b * kTsPerCta + 1] = globaltimer();
        published = true;
      }
    }
    auto publish = [&](const LaneRoute& lr) {
      if (published) return;               // (already published by the fast path)
      if (lane < K) {
        sslot[lane] = lr.slot;
        sgen[lane] = lr.gen;
        swait[lane] = lr.wait;
        shost[lane] = lr.host;
        sbase[lane] = a.pool + (long long)lr.slot * a.slot_bytes;
        sexp[lane] = lr.expert;
      }
      // device-computed experts in processing order: resident ones first, then the ones
      // whose fill may still be in flight (rank order within each)
      const unsigned dev_ready = __ballot_sync(0xffffffffu, lane < K && !lr.host && !lr.wait);
      const unsigned dev_wait = __ballot_sync(0xffffffffu, lane < K && !lr.host && lr.wait);
      const unsigned below = (1u << lane) - 1u;
      if (lane < K && !lr.host)
        sorder[lr.wait ? __popc(dev_ready) + __popc(dev_wait & below) : __popc(dev_ready & below)] = lane;
      if (lane == 0) {
        snseg = __popc(dev_ready | dev_wait);
        smerged = f.merge && K == kMaxFusedK && __popc(dev_ready) == K;
      }
      mbar_arrive(&rbar);                  // release (each lane its own writes): route published
      if (TS(f) && lane == 0) TS(f)[b * kTsPerCta + 1] = globaltimer();
      published = true;
    };
    LaneRoute lr;
    const bool writer = b == 0;
    const int nmiss = route_decide(ra, z, ds, writer, rS, rZ, rW, &lr, pm ? pm + 4 : nullptr, publish);
    if (TS(f) && lane == 0) TS(f)[b * kTsPerCta + 11] = globaltimer();
    if (pm && lane == 0) pm[7] = clock64();
    if (!published) publish(lr);
    if (lane < K) swgt[lane] = lr.w;       // gate weights: needed from phase B on
    mbar_arrive(&wbar);
    // miss mailbox entry (host-mapped: seq after its payload, P:200's trigger) and progress word
    if (lane == 0 && writer) publish_progress(ra, nmiss);
    griddep_launch_dependents();
    {
      // this CTA's slice of y (K == 2: the experts' terms accumulate onto 0) and its share of
      // the other parity's h buffer (armed for the next call), then one release: the
      // consumers of every CTA acquire it before their first y reduction. Off the critical
      // path: phase B starts at least one phase A later.
      const int c0 = (int)((long long)d * b / G), c1 = (int)((long long)d * (b + 1) / G);
      if (K == 2)
        for (int c = c0 + lane; c < c1; c += 32) a.y[c] = 0.f;
      const int hn = K * ffr;
      uint32_t* hnext = reinterpret_cast<uint32_t*>(f.hf + (long long)((f.calls + 1) & 1) * hn);
      const int h0 = (int)((long long)hn * b / G), h1 = (int)((long long)hn * (b + 1) / G);
      for (int i = h0 + lane; i < h1; i += 32) hnext[i] = kHUnset;
      __syncwarp();
      if (lane == 0) {
        red_release_add_u64(f.bar + kYCtr, 1ull);
        if (!smerged) {                    // segmented phase B: acquire every CTA's zeroing here,
          wait_counter(f.bar + kYCtr, (f.calls + 1) * (unsigned long long)G);  // off the h load's path
          mbar_arrive(&ybar);
        }
      }
    }
    __syncwarp();                          // (sorder / smerged written by other router lanes)
    const int nh = smerged ? K : (f.xsep && snseg > 0 ? 1 : 0);  // h buffers this warp fills
    if (nh > 0) {
      // merged phase B: bring every expert's h into its own buffer as soon as it is published
      // grid-wide (the buffers lie past x: no phase-A reader is disturbed); the y zeroing of
      // every CTA is acquired first (the consumers' reductions follow the h arrivals)
      // (xsep: the first segment's h into the one h buffer; the later ones are loaded by the
      // consumers after a CTA barrier, as in the segmented mode)
      if (lane == 0 && smerged) wait_counter(f.bar + kYCtr, (f.calls + 1) * (unsigned long long)G);
      for (int si = 0; si < nh; ++si) {
        const int r = sorder[si];
        float* hs = reinterpret_cast<float*>(xh + f.hoff + (smerged ? (size_t)r * f.hstride : 0));
        const float* hg = hcur + (long long)r * ffr;
        if (lane == 0) {
          const unsigned long long* bar = f.bar + 16 * r;
          const unsigned long long t0 = globaltimer();
          while (ld_acquire_u64(bar) < bar_target) {
            MOE_POLL_BACKOFF(64);
            if (globaltimer() - t0 > 60ull * 1000000000ull) __trap();
          }
          if (TS(f)) TS(f)[b * kTsPerCta + 19 + si] = globaltimer();  // h of segment si published grid-wide
          asm volatile("fence.proxy.async.global;" ::: "memory");
          mbar_arrive_expect_tx(hrawK + r, (uint32_t)ffr * 4u);
          bulk_g2s(hs, hg, (uint32_t)ffr * 4u, hrawK + r, policy_evict_first());
        }
        mbar_wait(hrawK + r, 0);
        if (TS(f) && lane == 0 && si == 1) TS(f)[b * kTsPerCta + 46] = globaltimer();  // h1 bulk copy landed
        inject_stale_h(f, hs, ffr, lane, 32);
        settle_h(hs, hg, ffr, lane, 32);   // words whose store had not reached L2 yet
        if (TS(f) && lane == 0 && si == 1) TS(f)[b * kTsPerCta + 47] = globaltimer();  // h1 settled
        mbar_arrive(hbarK + r);            // (count 32: each lane after its own settled words)
      }
    }
    return;
  }

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const RowSched sa = make_sched(ffr, b, G, f.pctA);  // (route-independent: before the wait)
      const RowSched sbk = make_sched(d, b, G, f.pctB);
      mbar_wait(&rbar, 0);                            // route published by the router warp
      const int nseg = snseg;
      for (int r = 0; r < K; ++r)  // host-computed experts have no h: publish them at once
        if (shost[r]) red_relaxed_add_u64(f.bar + 16 * r, (unsigned long long)NS);
      uint32_t use = 0;                               // per-stage use-count parity bits
      auto acquire = [&](int s) {                     // wait until stage s is free
        mbar_wait(empty + s, ((use >> s) & 1) ^ 1);
        use ^= 1u << s;
      };
      int t = 0;
      // Work claims: segment q = A of sorder[q] for q < nseg, B of sorder[q - nseg] after. A
      // segment's first claim is issued before its static block; the next segment's first claim
      // is issued ahead, while this segment's tail is within two grid-rounds of its end (the
      // short static blocks of phase B could not hide the atomic's latency: a restart bubble)
      unsigned pre = 0u;
      int pre_q = -1;
      auto seg_ctr = [&](int q) -> unsigned* {
        return ctr + (q < nseg ? sorder[q] : kMaxFusedK + sorder[q - nseg]) * kCtrStride;
      };
      auto seg_chunk = [&](int q) -> unsigned { return q < nseg ? (unsigned)kChunkA : (unsigned)RB; };
      auto first_claim = [&](int q) -> unsigned {
        if (pre_q == q) return pre;
        return atomicAdd(seg_ctr(q), seg_chunk(q));
      };
      auto claim_ahead = [&](int q, int tail_done, int tail_size) {  // (called with the claim just taken)
        if (f.claim_ahead && q + 1 < 2 * nseg && pre_q != q + 1 && tail_done + 2 * G * (int)seg_chunk(q) >= tail_size) {
          pre = atomicAdd(seg_ctr(q + 1), seg_chunk(q + 1));
          pre_q = q + 1;
        }
      };
      // phase A: per segment, static block then tail claims (two claims in flight hide the
      // atomic latency)
      for (int si = 0; si < nseg; ++si) {
        const int r = sorder[si];
        const uint8_t* base = sbase[r];
        if (swait[r]) {  // fill of this slot still in flight (FETCH) / being pulled by every CTA (PULL)
          if (ra.miss_mode == MOE_MISS_PULL) wait_counter(f.bar + kPullCtr, (f.calls + 1) * (unsigned long long)G);
          else wait_ready(a.ready, sslot[r], sgen[r]);
          asm volatile("fence.proxy.async.global;" ::: "memory");  // generic/DMA writes -> bulk reads
        }
        unsigned* cA = ctr + r * kCtrStride;
        auto issue_a = [&](int j) {
          const int s = t % NS;
          acquire(s);
          const uint8_t* w1 = base + (long long)j * d * 2;
          const uint8_t* w3 = w1 + (long long)ffr * d * 2;
          meta[s] = (si << 24) | j;
          mbar_arrive_expect_tx(full + s, (uint32_t)rowA);
          bulk_g2s(ring + (size_t)s * SB, w1, 2u * d, full + s, pol);
          bulk_g2s(ring + (size_t)s * SB + 2 * d, w3, 2u * d, full + s, pol);
          if (TS(f) && t == 0) TS(f)[b * kTsPerCta + 38] = globaltimer();  // first weight row issued
          ++t;
        };
        unsigned c1 = first_claim(si);
        for (int j = sa.s0; j < sa.s1; ++j) {
          if (f.pfA > 0 && j + f.pfA < sa.s1) {  // L2 prefetch pfA rows ahead (static block)
            const uint8_t* p1 = base + (long long)(j + f.pfA) * d * 2;
            bulk_prefetch_l2(p1, 2u * d);
            bulk_prefetch_l2(p1 + (long long)ffr * d * 2, 2u * d);
          }
          issue_a(j);
        }
        unsigned c2 = atomicAdd(cA, (unsigned)kChunkA);
        while (sa.tail0 + (int)c1 < ffr) {
          const int j0 = sa.tail0 + (int)c1, j1 = min(j0 + kChunkA, ffr);
          claim_ahead(si, (int)c1, ffr - sa.tail0);
          c1 = c2;
          if (sa.tail0 + (int)c1 < ffr) c2 = atomicAdd(cA, (unsigned)kChunkA);
          for (int j = j0; j < j1; ++j) issue_a(j);
        }
        if (pre_q != si + 1) claim_ahead(si, ffr, ffr);  // (a segment without a tail)
        // no marker between segments: a stage's consumers see the segment index change in
        // the row meta (its h writer then publishes the rows it wrote of the earlier
        // segment), so the ring does not drain at the expert switch
      }
      slastA = t;                                     // (consumers: a stage's last A row is known)
      if (TS(f)) TS(f)[b * kTsPerCta + 12] = globaltimer();  // last phase-A row issued
      if (f.prefetchB && nseg > 0 && !swait[sorder[0]]) {
        // the ring drains before phase B starts: have this CTA's first W2 rows on their way
        // to L2 meanwhile (same bytes, read from HBM once)
        const int nr = min(NSB * RB, sbk.s1 - sbk.s0);
        if (nr > 0) bulk_prefetch_l2(sbase[sorder[0]] + w2off + (long long)sbk.s0 * rowB, (uint32_t)(nr * rowB));
      }
      // phase B: whole W2 rows into super-stages (2u, 2u+1); W2 does not depend on h, so
      // these loads stream while the consumers finish phase A and load h. The end-of-A markers
      // go into a super-stage's two stages right before its first W2 rows, starting with the
      // super-stage whose stages drain first (the ring's next stages in issue order): W2 rows
      // enter as soon as one super-stage is free instead of after the whole ring drained.
      const int t_a = t;                              // phase-A items issued by this CTA
      // (only with a full ring of phase-A items: a CTA with a few rows — the tiny shapes —
      // publishes its h rows sooner with every end marker placed at once, +1.5 us otherwise)
      const bool lazy = f.lazy_marks && t_a >= NS;
      int tb = lazy ? ((t % NS) + 1) / 2 : 0;
      uint32_t marked = 0u;
      auto mark_end_a = [&](int u) {
        if ((marked >> u) & 1u) return;
        marked |= 1u << u;
        for (int k = 0; k < 2; ++k) {
          const int s = 2 * u + k;
          acquire(s);
          meta[s] = kEnd;
          mbar_arrive(full + s);
        }
      };
      auto marker_b = [&](int m) {
        for (int k = 0; k < NSB; ++k, ++tb) {
          const int s = 2 * (tb % NSB);
          mark_end_a(tb % NSB);
          acquire(s);
          meta[s] = m;
          mbar_arrive(full + s);
        }
      };
      if (lazy)                                       // super-stages that got no phase-A item: at once
        for (int u = 0; u < NSB; ++u)
          if (2 * u >= t_a) mark_end_a(u);
      if (!lazy) {                                    // every end-of-A marker first, in drain order
        for (int k = 0; k < NS; ++k, ++t) {
          const int s = t % NS;
          acquire(s);
          meta[s] = kEnd;
          mbar_arrive(full + s);
        }
        marked = (1u << NSB) - 1u;
      }
      if (smerged) {
        // Merged phase B (every expert resident and ready, every h resident in shared
        // memory, loaded by the router warp as soon as it is published): the experts' W2 rows
        // in turn with the same static-then-steal schedule, but no marker between experts
        // (no ring drain) and no CTA-wide h reload: every chunk's meta carries its expert and
        // a warp waits for that expert's h the first time it meets it.
        auto issue_b = [&](int r, int c, int nr) {
          const int s = 2 * (tb % NSB);
          mark_end_a(tb % NSB);
          acquire(s);
          meta[s] = (r << 24) | c;
          metaN[s] = nr;
          mbar_arrive_expect_tx(full + s, (uint32_t)(nr * rowB));
          bulk_g2s(ring + (size_t)s * SB, sbase[r] + w2off + (long long)c * rowB, (uint32_t)(nr * rowB), full + s, pol);
          ++tb;
        };
        for (int si = 0; si < nseg; ++si) {     // experts in turn, without markers between them
          const int r = sorder[si];
          unsigned* cB = ctr + (kMaxFusedK + r) * kCtrStride;
          unsigned e1 = first_claim(nseg + si);
          for (int c = sbk.s0; c < sbk.s1; c += RB) issue_b(r, c, min(RB, sbk.s1 - c));
          unsigned e2 = atomicAdd(cB, (unsigned)RB);
          while (sbk.tail0 + (int)e1 < d) {
            const int r0 = sbk.tail0 + (int)e1, r1 = min(r0 + RB, d);
            claim_ahead(nseg + si, (int)e1, d - sbk.tail0);
            e1 = e2;
            if (sbk.tail0 + (int)e1 < d) e2 = atomicAdd(cB, (unsigned)RB);
            issue_b(r, r0, r1 - r0);
            if (f.pfB && sbk.tail0 + (int)e1 < d) {  // the next claim's rows towards L2
              const int q0 = sbk.tail0 + (int)e1, q1 = min(q0 + RB, d);
              bulk_prefetch_l2(sbase[r] + w2off + (long long)q0 * rowB, (uint32_t)((q1 - q0) * rowB));
            }
          }
        }
        if (TS(f)) TS(f)[b * kTsPerCta + 14] = globaltimer();  // last phase-B row issued
        marker_b(kEnd);
        prefetch_next(f, b, G, ffr, d);
        return;
      }
      if (!f.xsep)                                    // segmented: every consumer loads h first
        for (int u = 0; u < NSB; ++u) mark_end_a((tb + u) % NSB);
      for (int si = 0; si < nseg; ++si) {
        const int r = sorder[si];
        const uint8_t* w2 = sbase[r] + w2off;
        unsigned* cB = ctr + (kMaxFusedK + r) * kCtrStride;
        // RB consecutive W2 rows (contiguous in the slot) per super-stage: short rows
        // (small ff_r) would otherwise leave too few bytes in flight per SM
        auto issue_b = [&](int c, int nr) {
          const int s = 2 * (tb % NSB);
          mark_end_a(tb % NSB);
          acquire(s);
          meta[s] = (r << 24) | c;
          metaN[s] = nr;
          mbar_arrive_expect_tx(full + s, (uint32_t)(nr * rowB));
          bulk_g2s(ring + (size_t)s * SB, w2 + (long long)c * rowB, (uint32_t)(nr * rowB), full + s, pol);
          ++tb;
        };
        if (si > 0) {
          if (TS(f)) TS(f)[b * kTsPerCta + 13] = globaltimer();  // last B_o0 row issued
          marker_b(kSegB);
        }
        unsigned c1 = first_claim(nseg + si);
        for (int c = sbk.s0; c < sbk.s1; c += RB) issue_b(c, min(RB, sbk.s1 - c));
        unsigned c2 = atomicAdd(cB, (unsigned)RB);
        while (sbk.tail0 + (int)c1 < d) {
          const int r0 = sbk.tail0 + (int)c1, r1 = min(r0 + RB, d);
          claim_ahead(nseg + si, (int)c1, d - sbk.tail0);
          c1 = c2;
          if (sbk.tail0 + (int)c1 < d) c2 = atomicAdd(cB, (unsigned)RB);
          issue_b(r0, r1 - r0);
          if (f.pfB && sbk.tail0 + (int)c1 < d) {  // the next claim's rows towards L2
            const int q0 = sbk.tail0 + (int)c1, q1 = min(q0 + RB, d);
            bulk_prefetch_l2(w2 + (long long)q0 * rowB, (uint32_t)((q1 - q0) * rowB));
          }
        }
      }
      if (TS(f)) TS(f)[b * kTsPerCta + 14] = globaltimer();  // last phase-B row issued
      marker_b(kEnd);
      prefetch_next(f, b, G, ffr, d);
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  if (cw >= nwc) return;
  const int sA = cw >> 1, half = cw & 1;   // phase A: stage and half of the row
  uint32_t ph = 0;                         // parity of the barrier this warp waits on
  {
    const int nchA = d >> 3;               // 16-B chunks per W1 (or W3) row
    const int c0 = half * (nchA >> 1), c1 = half ? nchA : (nchA >> 1);
    const int4* xq = reinterpret_cast<const int4*>(xh);  // x, bf16
    const int4* w1 = reinterpret_cast<const int4*>(ring + (size_t)sA * SB);
    const int4* w3 = reinterpret_cast<const int4*>(ring + (size_t)sA * SB + 2 * d);
    bool first = true;
    int pubseg = 0;                        // (h writer) first segment not yet published
    int rc = 0;                            // rows of this stage so far (partials double-buffered)
    int ti = sA - NS;                      // ring item index of this stage's current item
    while (true) {
      ti += NS;
      mbar_wait(full + sA, ph);
      ph ^= 1;
      const int m = meta[sA];
      if (m < 0) break;                    // kEnd
      const int si = m >> 24, j = m & 0xFFFFFF;
      const int r = sorder[si];
      if (half == 0 && lane == 0) record_event(f, &evn, b, (unsigned)rowA, (unsigned)si);
      // a row of a later segment: this stage's h writer (half 0, lane 0) has written every
      // row of the earlier segments it produced; publish them (release at gpu scope covers
      // its own stores)
      if (half == 0 && lane == 0)
        for (; pubseg < si; ++pubseg) {
          if (TS(f) && sA == 0 && pubseg == 0) TS(f)[b * kTsPerCta + 39] = globaltimer();
          publish_h(spub + sorder[pubseg], f.bar + 16 * sorder[pubseg], NS);
          if (TS(f) && sA == 0 && pubseg == 0) TS(f)[b * kTsPerCta + 40] = globaltimer();
        }
      if (TS(f) && first && cw == 0 && lane == 0) TS(f)[b * kTsPerCta + 2] = globaltimer();
      first = false;
      float2 g = make_float2(0.f, 0.f), u = make_float2(0.f, 0.f);
#pragma unroll 4
      for (int c = c0 + lane; c < c1; c += 32) {
        const int4 xc = xq[c];
        g = dot8_bf(w1[c], xc, g);
        u = dot8_bf(w3[c], xc, u);
      }
      // partials by row parity: the stage is released before they are combined, so the next
      // row's partials (written after the refill) go to the other buffer; the one after that
      // needs this warp's next release, which follows its own read of these
      volatile float* pp = part + 8 * sA + 4 * (rc++ & 1);
      const float gs = warp_sum(g.x + g.y);
      const float us = warp_sum(u.x + u.y);
      if (lane == 0) {
        pp[2 * half] = gs;
        pp[2 * half + 1] = us;
        mbar_arrive_cnt(empty + sA, 2);    // this half's reads of the stage are done
      }
      named_bar_sync(2 + sA, 64);          // both halves' partials written
      if (half == 0 && lane == 0) {
        const float gg = pp[0] + pp[2];    // fixed order: half 0 + half 1
        const float uu = pp[1] + pp[3];
        hcur[(long long)r * ffr + h_plane_index(j, ffr)] = gg / (1.0f + expf(-gg)) * uu;
        // this stage's last phase-A row (known once the producer issued its last one): publish
        // every segment now instead of at the next item (end marker or W2 rows)
        if (ti + NS >= slastA)
          for (const int nseg = snseg; pubseg < nseg; ++pubseg) publish_h(spub + sorder[pubseg], f.bar + 16 * sorder[pubseg], NS);
      }
    }
    if (half == 0 && lane == 0)            // the rest of this stage's segments
      for (const int nseg = snseg; pubseg < nseg; ++pubseg) {
        if (TS(f) && sA == 0) TS(f)[b * kTsPerCta + 41 + 2 * pubseg] = globaltimer();
        publish_h(spub + sorder[pubseg], f.bar + 16 * sorder[pubseg], NS);
        if (TS(f) && sA == 0) TS(f)[b * kTsPerCta + 42 + 2 * pubseg] = globaltimer();
      }
    named_bar_sync(2 + sA, 64);
    if (lane == 0) mbar_arrive_cnt(empty + sA, 2);  // release the end marker's stage (both halves)
    if (half == 0 && lane == 0 && (sA & 1) == 0) {
      parB[sA >> 1] = ph;                  // full[sA] parity for phase B
      mbar_arrive(pairbar + (sA >> 1));    // (release; merged phase B starts without a CTA barrier)
    }
  }
  if (TS(f) && cw == 0 && lane == 0) TS(f)[b * kTsPerCta + 3] = globaltimer();
  // h_r -> shared memory (xh) before phase-B segment r: every consumer is done with xh,
  // every stage of every CTA has published its rows of h_r (acquire), then ONE bulk copy
  // (the async proxy reads global memory written through the generic proxy by other CTAs:
  // fence the proxies first).
  uint32_t hph = 0;
  const int hbo = f.xsep ? f.hoff : 0;     // segmented: h over x; xsep: h beside x
  auto load_h = [&](int r, bool first_h) {
    named_bar_sync(1, nthr);
    if (cw == 0 && lane == 0) {
      const unsigned long long* bar = f.bar + 16 * r;
      const bool dbg = TS(f) && TS(f)[b * kTsPerCta + 16] == 0;
      if (dbg) TS(f)[b * kTsPerCta + 16] = globaltimer();  // first h load: CTA out of phase A
      if (ld_acquire_u64(bar) < bar_target) {
        const unsigned long long t0 = globaltimer();
        while (ld_acquire_u64(bar) < bar_target) {
          MOE_POLL_BACKOFF(32);
          if (globaltimer() - t0 > 60ull * 1000000000ull) __trap();
        }
      }
      if (dbg) TS(f)[b * kTsPerCta + 17] = globaltimer();  // first h published grid-wide
      if (first_h) mbar_wait(&ybar, 0);    // y zeroed by every CTA (acquired by the router warp)
      asm volatile("fence.proxy.async.global;" ::: "memory");
      mbar_arrive_expect_tx(hbar, (uint32_t)ffr * 4u);
      bulk_g2s(xh + hbo, hcur + (long long)r * ffr, (uint32_t)ffr * 4u, hbar, policy_evict_first());
    }
    mbar_wait(hbar, hph);
    hph ^= 1;
    inject_stale_h(f, reinterpret_cast<float*>(xh + hbo), ffr, ctid, nthr);
    settle_h(reinterpret_cast<float*>(xh + hbo), hcur + (long long)r * ffr, ffr, ctid, nthr);
    named_bar_sync(1, nthr);               // every settled word visible to every consumer
  };
  const int nseg = snseg;                  // (visible: published before the producer's first marker)
  const bool mm = smerged;                 // merged phase B: one pass over every expert
  mbar_wait(&wbar, 0);                     // gate weights (long published by now)
  {
    const int u = cw >> 2, q = cw & 3;     // super-stage and quarter of the W2 row
    const bool active = u < NSB;           // (NS odd: the last stage's warps sit out phase B)
    const int s = 2 * u;
    const int nck = rowB >> 4;
    const int k0 = (nck * q) >> 2, k1 = (nck * (q + 1)) >> 2;
    const int4* wv = reinterpret_cast<const int4*>(ring + (size_t)s * SB);
    // pair u's named barrier: its even stage's phase-A id (that stage has left phase A by the
    // time any of the pair's warps uses it: no mixed 64/128-thread use of one id)
    const int bid = 2 + 2 * u;
    uint32_t seen = 0u;                    // merged: experts whose h this warp has waited for
    uint32_t nchunk = 0u;                  // chunks this pair has processed
    for (int si = 0; si < (mm ? 1 : nseg); ++si) {
      if (mm || (f.xsep && si == 0)) {     // no CTA barrier: start once the pair's even stage is out
        if (active) {
          mbar_wait(pairbar + u, 0);
          ph = parB[u];
        }
      } else {
        // (xsep: a super-stage that got no chunk of the first expert never waited for its h —
        // and with it for the y counter — so the reload acquires the y zeroing here too)
        load_h(sorder[si], si == 0 || f.xsep);
        if (si == 0 && active) ph = parB[u];  // written before load_h's barrier
      }
      if (TS(f) && cw == 0 && lane == 0) TS(f)[b * kTsPerCta + (si == 0 ? 4 : 6)] = globaltimer();
      if (!active) continue;
      while (true) {
        mbar_wait(full + s, ph);
        ph ^= 1;
        const int m = meta[s];
        if (TS(f) && cw == 0 && lane == 0 && !TS(f)[b * kTsPerCta + 15]) TS(f)[b * kTsPerCta + 15] = globaltimer();
        if (m < 0) {                       // kSegB (next expert) or kEnd
          named_bar_sync(bid, 128);
          if (q == 0 && lane == 0) mbar_arrive_cnt(empty + s, kEmptyArrivals);
          break;
        }
        const int r = m >> 24, c = m & 0xFFFFFF;  // expert (routing rank), first row
        const float w = swgt[r];
        if ((mm || (f.xsep && si == 0)) && !((seen >> r) & 1u)) {  // h_r copied in by the router warp
          mbar_wait(hbarK + r, 0);
          seen |= 1u << r;
          if (TS(f) && cw == 0 && lane == 0 && r == sorder[1 % nseg]) TS(f)[b * kTsPerCta + 22] = globaltimer();
        }
        // h_r[8k .. 8k+3] / h_r[8k+4 .. 8k+7] (2-plane layout)
        const float4* hp0 = reinterpret_cast<const float4*>(xh + (mm ? f.hoff + (size_t)r * f.hstride : hbo));
        const float4* hp1 = hp0 + (ffr >> 3);
        const int nr = metaN[s];           // rows c .. c+nr-1, contiguous in the stage
        if (q == 0 && lane == 0) record_event(f, &evn, b, (unsigned)(nr * rowB), 2u + (unsigned)r);
        // partials double-buffered by chunk parity: the next chunk's writes go to the other
        // buffer, so every write-after-read is ordered by a named barrier
        volatile float* pb = partB + (u * 2 + (nchunk++ & 1)) * RBp * 4;
        for (int i = 0; i < nr; ++i) {
          const int4* wr = wv + i * nck;
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll 4
          for (int cc = k0 + lane; cc < k1; cc += 32) acc = dot8(wr[cc], hp0[cc], hp1[cc], acc);
          const float sum = warp_sum(acc.x + acc.y);
          if (lane == 0) pb[4 * i + q] = sum;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_cnt(empty + s, 1);  // this quarter's reads of the stage are done
        named_bar_sync(bid, 128);          // the 4 quarters of these rows are done
        if (TS(f) && cw == 0 && lane == 0) TS(f)[b * kTsPerCta + 23] = globaltimer();  // (last: final B chunk)
        if (q == 0) {                      // lane i combines row i in a fixed order
          float o = 0.f;
          if (lane < nr) o = ((pb[4 * lane] + pb[4 * lane + 1]) + pb[4 * lane + 2]) + pb[4 * lane + 3];
          if (lane < nr) {
            if (f.tpP > 0) tp_push(speer, f.tpP, f.tp_rank, f.tp_calls, K, d, r, c + lane, w * o);  // f3 / LL
            else if (K == 1) a.y[c + lane] = w * o;
            else red_add_f32(a.y + c + lane, w * o);  // K == 2: 0 + a + b is order-independent
          }
        }
      }
    }
  }
  // host-computed experts (MOE_MISS_HOST_COMPUTE): wait for the host's result on the
  // activation stream and add w_r * o_r over this CTA's share of y
  for (int r = 0; r < K; ++r) {
    if (!shost[r]) continue;
    if (cw == 0 && lane == 0) {
      // every CTA zeroed its slice of y before its release on the y counter
      wait_counter(f.bar + kYCtr, (f.calls + 1) * (unsigned long long)G);
      const uint32_t want = (uint32_t)a.seq;
      const unsigned long long t0 = globaltimer();
      unsigned ns = 256;
      while (ld_acquire_u32(a.host_flag + r) != want) {
        __nanosleep(ns);
        if (ns < 8192) ns <<= 1;
        if (globaltimer() - t0 > 60ull * 1000000000ull) __trap();
      }
    }
    named_bar_sync(1, nthr);
    const int c0 = (int)((long long)d * b / G), c1 = (int)((long long)d * (b + 1) / G);
    const float w = swgt[r];
    const float* o = a.host_out + (size_t)r * d;
    for (int c = c0 + ctid; c < c1; c += nthr) {
      const float v = w * __ldcg(o + c);
      if (f.tpP > 0) tp_push(speer, f.tpP, f.tp_rank, f.tp_calls, K, d, r, c, v);
      else if (K == 1) a.y[c] = v;
      else red_add_f32(a.y + c, v);  // K == 2: 0 + a + b is order-independent
    }
  }
  if (f.tpP > 0)
    tp_reduce_epilogue(f.peer[f.tp_rank], f.tpP, K, d, f.tp_calls, f.yout, TS(f) ? TS(f) + b * kTsPerCta : nullptr, b, G,
                       ctid, nthr);
  if (f.donef) {  // host-buffer entry point: this CTA's slice of y is in host memory
    named_bar_sync(kPullBar, nthr);
    if (ctid == 0) {
      __threadfence_system();
      f.donef[b] = f.donetag;
    }
  }
  if (TS(f) && cw == 0 && lane == 0) {
    TS(f)[b * kTsPerCta + 45] = (unsigned long long)evn;  // (this warp's count; the tool trims by time)
    TS(f)[b * kTsPerCta + 5] = globaltimer();
    TS(f)[b * kTsPerCta + 34] = clock64();
  }
  if (STS(f) && cw == 0 && lane == 0) STS(f)[kStsHead + G + b] = globaltimer();
}

}  // namespace

#if MOE_FUSED_MMA_GATE
cudaError_t fused_mma_kernel_attrs(int threads, size_t smem, int* blocks_per_sm) {
  if (blocks_per_sm) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, expert_fused_mma_kernel, threads, smem);
  cudaFuncAttributes fa;
  const cudaError_t e = cudaFuncGetAttributes(&fa, expert_fused_mma_kernel);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(expert_fused_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedMaxDynSmem);
}
cudaError_t launch_expert_fused_mma(const cudaLaunchConfig_t& cfg, const FusedArgs& f) {
  return cudaLaunchKernelEx(&cfg, expert_fused_mma_kernel, f);
}
#else

// CTAs of the fused kernel wait on each other (h publication), so the whole grid (one CTA
// per SM) must be resident at once: check that one CTA of this plan fits on an SM.
int fused_blocks_per_sm(const FusedPlan& p) {
  int nb = 0, nbm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, expert_fused_kernel, p.threads, p.smem) != cudaSuccess ||
      fused_mma_kernel_attrs(p.threads, p.smem, &nbm) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return min(nb, nbm);
}

cudaError_t preload_fused_kernels() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, expert_fused_kernel);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(expert_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedMaxDynSmem);
  if (e != cudaSuccess) return e;
  return fused_mma_kernel_attrs(0, 0, nullptr);
}

bool plan_fused(int d, int ffr, int n, int K, int grid, FusedPlan* p) {
  if (K > 2 || grid < K) return false;          // deterministic combine needs K <= 2
  const int SB = max(16384, 4 * d);              // one W1+W3 row pair per stage
  if (2 * ffr > 2 * SB) return false;            // a W2 row fits one super-stage (2 stages)
  const int RB = min(kMaxRB, (2 * SB) / (2 * ffr));  // W2 rows per phase-B super-stage
  // partB: [NS/2][2][RB][4]; sized for kMaxRB rows except with single-row chunks (xsep below:
  // Mixtral's x beside h fits only with the trimmed tail) — the stage counts of the other
  // shapes stay the measured ones (8x22B P = 2 with 8 instead of 6 stages: +1-2 us)
  auto tail_of = [&](int rb) {
    return 2 * kMaxNS * 8 + 8 + kMaxNS * 4 + kMaxNS * 32 + kMaxNS * 4 + kMaxNS * 4 + (kMaxNS / 2) * 2 * rb * 16 + 64;
  };
  const int tail = tail_of(RB == 1 ? 1 : kMaxRB);
  const int xh1 = ((max(2 * d, ffr * 4) + 127) / 128) * 128;  // x (bf16) | one expert's h (fp32)
  const int hoff = ((2 * d + 127) / 128) * 128, hstride = ((ffr * 4 + 127) / 128) * 128;
  const int xh2 = hoff + K * hstride;            // x | every expert's own h buffer (merged phase B)
  auto stages = [&](int xh) {
    int ns = (kFusedMaxDynSmem - xh - tail) / SB;
    if (ns > kMaxNS) ns = kMaxNS;
    return ns & ~1;                              // stages pair into super-stages in phase B
  };
  // merged phase B when holding every expert's h costs no ring stage (small ff_r) ...
  // ... and also where it costs ring stages, as long as the smaller ring still holds 144 KB
  // in flight per SM (interleaved A/B: 8x22B P = 4 slice, 8 -> 6 stages of 24 KB: -2.7 us;
  // Mixtral, 10 -> 6 stages of 16 KB: +2.6 us)
  const bool merge = K == kMaxFusedK &&
                     (stages(xh2) == stages(xh1) || (stages(xh2) >= 4 && (long long)stages(xh2) * SB >= 144 * 1024));
  // otherwise x and ONE h buffer side by side when that costs no ring stage either: phase B of
  // the first expert then starts per super-stage as in the merged mode (xsep)
  const int xh3 = hoff + hstride;
  // (interleaved A/B: Mixtral -1.0-1.2 us, 8x22B unsplit -0.7; with multi-row W2 chunks — the
  // P = 2 / 4 slices — +0.6-1.0 us, so only for single-row chunks)
  const bool xsep = !merge && K == kMaxFusedK && stages(xh3) == stages(xh1) && RB == 1;
  const int xh = merge ? xh2 : xsep ? xh3 : xh1;
  const int NS = stages(xh);
  if (NS < 4) return false;
  // the gate rows and x are staged in the (still empty) ring before the route is known
  const long long gate = (2ll * d + 16) * n;                            // staged in the ring
  const long long zp = 4ll * kWarpsPerStage * kMaxNS * MOE_MAX_EXPERTS;  // partial logits
  if (n > MOE_MAX_EXPERTS || d % 8 || gate + zp > (long long)NS * SB || 2ll * n * d >= (1ll << 20)) return false;
  p->SB = SB;
  p->NS = NS;
  p->xh_bytes = xh;
  p->RB = RB;
  p->xsep = xsep ? 1 : 0;
  // static shares (rest stolen in chunks): measured on B200 across the BASELINE shapes
  // (bench_shapes.py sweeps): 95% of phase A; 10% of phase B with 1-2-row chunks, 20% with
  // bigger ones (8x22B slices) — phase B's expert switch and the end of the step leave the
  // CTAs unevenly advanced, and a long stolen tail re-balances them
  // Round 2, interleaved A/B per shape class: fewer than 32 phase-A rows per CTA and expert
  // (8x22B P = 4 / 8, Mixtral P = 8 slices): a 10% stolen phase-A tail (-0.1-0.3 us); 24 KB
  // stages (d = 6144: 8x22B unsplit / P = 2): 2% (-0.85 / -0.9 us); sets of 16 or more
  // experts with short W2 rows (Phi): 2% of phase A and 15% of phase B stolen (-0.35 us);
  // Mixtral keeps 95 / 10 (98 / 15: +0.6-1.5 us).
  const int rows_per_cta = ffr / grid;
  p->pctA = rows_per_cta < 32 ? 90 : (SB > 16384 || n >= 16) ? 98 : 95;
  p->pctB = p->RB <= 2 ? (n >= 16 ? 15 : 10) : 20;
  p->merge = merge ? 1 : 0;
  p->prefetchB = 1;
  p->next_rows = -1;  // (runtime default by the number of ways)
  // L2 prefetch ahead of the ring (interleaved A/B): phase-A static rows 10 / 20 ahead cost
  // +1.5-10 us (off); the next phase-B claim's rows: Phi -0.56 us, 8x22B P = 4 -0.13, but
  // Mixtral's single 28 KB rows +0.45 -> on only with multi-row chunks
  p->pfA = 0;
  p->pfB = p->RB >= 2 ? 1 : 0;
  p->start_rows = -1;  // (runtime default by the number of ways)
  // interleaved A/B: issuing the next segment's first claim early was neutral to slightly
  // slower (off); end-of-A markers placed per super-stage before its first W2 rows: Phi -0.5
  // us, 8x22B P = 8 -0.3, Mixtral -0.3 (on)
  p->claim_ahead = 0;
  p->lazy_marks = 1;
  p->pfx = 1;
  p->hoff = hoff;
  p->hstride = hstride;
  p->smem = (size_t)NS * SB + xh + tail;
  p->threads = kThreadsF;
  return p->smem <= (size_t)kFusedMaxDynSmem;
}

cudaError_t launch_expert_fused(const FusedArgs& f, const FusedPlan& p, int grid, cudaStream_t s, bool pdl, bool coop) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(p.threads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  if (gate_mma_form(f.r.n, f.e.d)) return launch_expert_fused_mma(cfg, f);
  return cudaLaunchKernelEx(&cfg, expert_fused_kernel, f);
}

#endif  // MOE_FUSED_MMA_GATE
}  // namespace moe
