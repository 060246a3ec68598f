// moe_internal.cuh — device-side records, kernel argument blocks and launchers
// shared by the runtime (runtime.cu) and the sm_100a kernels (route_probe.cu,
// expert_gemv.cu). Not part of the ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cuda_bf16.h>

#include "moe.h"

namespace moe {

constexpr int kMaxK = MOE_MAX_EXPERTS;  // K <= n <= 32
// fused kernel work-claim counters: 2 call parities x (phase A, phase B) x 2 experts, each on
// its own 128-B line (same-line atomics serialise in one L2 slice)
constexpr int kCtrStride = 32;
constexpr int kCtrWords = 2 * 2 * 2 * kCtrStride;
constexpr int kMailRing = 1024;         // miss-notification mailbox entries (host-mapped)
constexpr int kStsRing = 64;            // debug step-timestamp records (MOE_DEBUG_TS)
constexpr int kStsHead = 8;             // router marks per record

// Per-layer device counters, same order as moe_layer_stats.
struct DevStats {
  unsigned long long accesses, at_least_one_hit, all_k_hit, expert_hits, expert_misses,
      coverage_misses, evictions, fetches, fetch_bytes, hit_under_fill, host_computed;
};
static_assert(sizeof(DevStats) == sizeof(moe_layer_stats), "stats layout");

// Routing decision of the current call, written by the router kernel and read by the
// expert kernels on the same stream (stream order = no race).
struct RouteRec {
  int32_t K;
  int32_t expert[kMaxK];
  float w[kMaxK];
  int32_t slot[kMaxK];   // slot index in the pool (cache way or staging slot)
  uint32_t gen[kMaxK];   // fill generation the slot must reach before it is read
  int32_t wait[kMaxK];   // 1: wait until ready[slot] >= gen before reading the slot
  int32_t host[kMaxK];   // 1: computed by the host cores (MOE_MISS_HOST_COMPUTE miss)
};

// Miss mailbox entry, in HOST-MAPPED pinned memory, written by the router kernel only for
// calls that missed: payload, system fence, then `seq`. Every call also publishes its seq
// in a host-mapped progress word; the runtime's fetch thread scans seqs up to it and
// issues the copies of the missed experts on the fetch stream.
struct Mail {
  volatile unsigned long long seq;
  int32_t layer, nmiss;
  int32_t expert[kMaxK];
  int32_t slot[kMaxK];
  uint32_t gen[kMaxK];
  int32_t rank[kMaxK];       // routing rank of the miss
  int32_t postfetch[kMaxK];  // 1: copy the weights into `slot` (covered miss)
  int32_t dest[kMaxK];       // 0: `slot` of the pool; 1: `slot` of the prefill staging area (M < n)
  int32_t host;              // 1: the host computes these experts (x is in the call's x slot)
};

struct RouteArgs {
  const uint16_t* Wg;  // [n][d] gate of this layer (device)
  const uint16_t* x;   // [d] (device)
  int d, n, K, M, layer, covered, policy, miss_mode;
  int gw;              // virtual warps of the gate-logit summation order (gate_gemv.cuh)
  int32_t* tag;        // [M] set of this layer (covered only)
  unsigned long long* stamp;  // [M]
  int slot_base;       // first slot of this layer's set (= layer * M)
  int staging_base;    // first staging slot (= covered_layers * M)
  uint32_t* gen;       // [slots + K] fill generation per slot
  const uint32_t* ready;  // [slots + K] landed generation per slot (written by the fetch stream)
  unsigned long long* clock;
  DevStats* stats;     // &stats[layer]
  RouteRec* route;
  moe_access_record* trace;
  long long trace_idx, trace_cap;
  uint32_t token;
  Mail* mail;          // device alias of the host-mapped ring entry for this call
  uint16_t* xmail;     // device alias of the host-mapped x slot of this call (host compute)
  unsigned long long seq;
  long long slot_bytes;
  unsigned long long* sts;  // debug (MOE_DEBUG_TS): this call's step-timestamp record, or nullptr
  const uint8_t* const* hblob;  // [n] device-accessible pinned host blobs of this layer (MOE_MISS_PULL)
  volatile unsigned long long* last_seq;  // host-mapped progress word (CTA 0's router publishes seq)
};

struct ExpertArgs {
  const RouteRec* route;
  const uint8_t* pool;
  long long slot_bytes;
  const uint16_t* x;  // [d]
  int d, ffr, K;
  float* h;           // [K][ffr] SwiGLU activations (scratch)
  float* y;           // [d]
  const uint32_t* ready;
  volatile unsigned long long* last_seq;  // host-mapped progress word, written at the end
  unsigned long long seq;                 // this call's sequence number
  const float* host_out;                  // [kMaxK][d] host-computed expert outputs (device copy)
  const uint32_t* host_flag;              // [kMaxK] == (uint32_t)seq once host_out[r] landed
};

// Fused persistent expert kernel (expert_fused.cu).
constexpr int kEvPerCta = 512;  // debug stage events per CTA and call
constexpr int kTsStride = 48;   // debug timestamps per CTA (expert_fused.cu's kTsPerCta)
constexpr int kFusedMaxDynSmem = 232448 - 1024;  // 227 KB opt-in minus static shared memory
struct FusedArgs {
  RouteArgs r;                    // routing inputs (every CTA takes the decision; CTA 0 writes it)
  ExpertArgs e;
  unsigned long long* bar;        // per-expert h publication counters [K] (monotonic across calls)
  float* hf;                      // h [2 (call parity)][K][ffr], words armed with kHUnset
  unsigned long long calls;       // number of earlier fused launches on this context
  unsigned* ctr;                  // work-claim counters [2][kMaxK] (phase A rows, phase B rows), zeroed per call
  int NS, SB;                     // ring stages / stage bytes
  int xh_bytes;
  int pctA, pctB;                 // share of phase A / B rows assigned statically (rest: stolen)
  int RB;                         // W2 rows per phase-B super-stage
  int RBp;                        // row stride of the phase-B partials (the plan's RB)
  int xsep;                       // 1: x and one h buffer side by side (first expert's phase B
                                  //    starts per super-stage, h copied in by the router warp)
  int merge;                      // 1: merged phase B when every routed expert is resident and ready
  int prefetchB;                  // 1: L2 prefetch of the first W2 rows at the end of phase A
  int pfA, pfB;                   // L2 prefetch: phase-A static rows pfA ahead; phase-B next claim
  const uint8_t* next_pool;       // != nullptr: at its end, each CTA prefetches into L2 the first
  int next_ways, next_rows;       //   next_rows W1/W3 row pairs of its static block of every way
                                  //   of the NEXT call's set (slots from next_pool, stride slot_bytes)
  const uint8_t* cur_pool;        // != nullptr: before its PDL wait, each CTA prefetches into L2 the
  int cur_ways, start_rows;       //   first start_rows W1/W3 row pairs of its static block of every
                                  //   way of THIS call's set (slots from cur_pool)
  int pfx;                        // 1: x prefetched into L2 before the PDL wait
  int claim_ahead;                // 1: a segment's first work claim issued near the end of the previous one
  int lazy_marks;                 // 1: end-of-A markers placed per super-stage right before its first W2 rows
  int hoff, hstride;              // merged: h_r at xh + hoff + r * hstride
  unsigned* dbg;                  // host-mapped progress counters (MOE_DEBUG_KERNEL=1) or nullptr
  int dbg_stale;                  // debug build: MOE_DEBUG_STALE_H=1 re-arms h words before the settle
  unsigned long long* ts;         // per-CTA phase timestamps [grid][8] (MOE_DEBUG_TS=1) or nullptr
  unsigned long long* ev;         // per-CTA stage events [grid][kEvPerCta][2] {time, bytes} (MOE_DEBUG_TS=1)
  unsigned long long* sts;        // this call's step record [kStsHead + 2*grid] (MOE_DEBUG_TS=1) or nullptr
  // fused TP reduction (f3, moe_tp_connect_*): every term of this rank's partial y goes to
  // the ranks' exchange buffers (layout below); the epilogue sums them into yout
  int tpP, tp_rank;               // tpP == 0: no fused reduction
  unsigned long long tp_calls;    // earlier fused-TP calls on this context (same on every rank)
  uint8_t* peer[8];               // exchange buffer base of every rank (peer[tp_rank] = own)
  float* yout;                    // [d] all-reduced y (caller's buffer)
  // moe_layer_forward_host: x is read from this (device-accessible) pinned host pointer by
  // CTA 0 into e.x, which then releases xseq on *xflag; every CTA acquires it before loading
  // x. nullptr: x is ready in e.x.
  const uint16_t* xhost;
  uint32_t* xflag;
  uint32_t xseq;
  // moe_layer_forward_host: after writing its slice of y to host memory, every CTA stores
  // donetag into donef[blockIdx.x] (host-mapped, after a system fence); the host spins on
  // these words instead of a CUDA event. nullptr: no flags.
  volatile uint32_t* donef;
  uint32_t donetag;
};
// Exchange buffer of one TP rank: slots[2][d][P][K] u64 at kTpSlotOff (call parity, column,
// source rank, routing rank), each word {fp32 term w_r * o_r[c] | call tag << 32}, written
// by the source rank with 8-byte stores.
constexpr int kTpSlotOff = 256;
inline long long tp_xchg_bytes(int P, int K, int d) { return kTpSlotOff + 2ll * P * K * d * 8; }
struct FusedPlan {
  int SB, NS, xh_bytes, threads, pctA, pctB, RB, merge, prefetchB, next_rows, pfA, pfB, hoff, hstride;
  int start_rows, pfx, xsep, claim_ahead, lazy_marks;
  size_t smem;
};
bool plan_fused(int d, int ffr, int n, int K, int grid, FusedPlan* p);

cudaError_t launch_expert_fused(const FusedArgs& f, const FusedPlan& p, int grid, cudaStream_t s, bool pdl, bool coop);
cudaError_t preload_fused_kernels();
int fused_blocks_per_sm(const FusedPlan& p);
// the fused kernel with the gate GEMV's tensor-core form (expert_fused_mma.cu): occupancy
// (blocks_per_sm != null) or attribute preload; launch
cudaError_t fused_mma_kernel_attrs(int threads, size_t smem, int* blocks_per_sm);
cudaError_t launch_expert_fused_mma(const cudaLaunchConfig_t& cfg, const FusedArgs& f);

cudaError_t launch_route_probe(const RouteArgs& a, cudaStream_t s, bool pdl);

// ---------------------------------------------------------------- prefill (f4, tensor cores)
constexpr int kPrefillMaxBlk = MOE_MAX_EXPERTS;
// Device-side plan of one prefill call: the distinct routed experts ("blocks"), each with
// its tokens gathered into rows [row_off, row_off + 128*mtiles) of X_g / H_g.
struct PrefillPlan {
  int nblk, total_mtiles, rows;
  int row_off[kPrefillMaxBlk];
  int mt_pref[kPrefillMaxBlk + 1];
  int slot[kPrefillMaxBlk];
  uint32_t gen[kPrefillMaxBlk];
  int wait[kPrefillMaxBlk];   // 1: the slot is filled by this call -> wait for gen
  int expert[kPrefillMaxBlk]; // expert of each block
  int stage[kPrefillMaxBlk];  // 1: `slot` indexes the prefill staging area (M < n: routed in the
                              //    prompt but not resident at its end), 0: the slot pool
  int* tok;      // [rows_cap] token of each gathered row (-1 = padding)
  float* wrow;   // [rows_cap] gate weight of that token for the block's expert
};
struct PrefillArgs {
  int T, n, K, M, layer, policy, miss_mode;
  int gw;                      // virtual warps of the gate-logit summation order (gate_gemv.cuh)
  int32_t* tag;                // set of the layer
  unsigned long long* stamp;
  int slot_base;
  uint32_t* gen;
  unsigned long long* clock;
  DevStats* stats;
  int* rt_e;                   // [T][K] routed experts (rank order)
  float* rt_w;                 // [T][K] gate weights
  moe_access_record* trace;
  long long trace_idx, trace_cap;
  uint32_t token0;
  Mail* mail;
  unsigned long long seq;
  volatile unsigned long long* last_seq;  // host-mapped progress word (the plan kernel publishes seq)
  long long slot_bytes;
  PrefillPlan* plan;
  void* scratch;               // prefill_scratch_bytes() of device scratch
  // M < n (evictions inside the prompt): the cache pass replays the T accesses in order
  float* zbuf;                 // [T][n] router logits
  const uint32_t* ready;       // landed generation per pool slot
  int staging_base;            // (RouteArgs field; unused: prefill layers are covered)
  int stage_slots;             // prefill staging slots (n - M)
};
// MOE_MISS_PULL outside the fused kernel (split decode path, prefill): copy the listed
// blobs (flag[i] != 0, i < *count) from the pinned host store into their slots, then
// publish ready[slot[i]] = gen[i] (pull.cu).
struct PullJob {
  const int32_t* count;
  const int32_t* expert;
  const int32_t* slot;
  const uint32_t* gen;
  const int32_t* flag;
  const uint8_t* const* hblob;  // [n] blobs of the layer
  const int32_t* only;          // optional: copy entry i only if only[i] == only_val
  int only_val;
  uint8_t* pool;
  long long slot_bytes;
  uint32_t* ready;
  unsigned* done;               // completion counter (zero between launches)
};
cudaError_t preload_pull_kernels();
cudaError_t launch_pull(const PullJob& j, int grid, cudaStream_t s);

size_t prefill_scratch_bytes();
cudaError_t preload_prefill_kernels();
cudaError_t launch_prefill_route(const PrefillArgs& a, const uint16_t* Wg, const uint16_t* x, int d, cudaStream_t s);
cudaError_t launch_prefill_gather(const uint16_t* x, int d, const PrefillPlan* plan, uint16_t* xg, int rows_cap,
                                  cudaStream_t s);
cudaError_t launch_publish_seq(volatile unsigned long long* word, unsigned long long seq, cudaStream_t s);
enum { TC_MODE_PLAIN = 0, TC_MODE_SWIGLU = 1, TC_MODE_DOWN = 2 };
struct TcArgs {
  CUtensorMap mapA;   // A operand (K-major rows)
  CUtensorMap mapB;   // B operand(s) (K-major rows)
  int mode, M, N, K;  // output rows (PLAIN), output cols, reduction length (multiple of 64)
  int d, ffr, ldh;
  float* C;                    // PLAIN: [M][N]
  __nv_bfloat16* H;            // SWIGLU: H_g rows (ldh = ffr)
  float* y;                    // DOWN: y [T][d]
  const PrefillPlan* plan;     // SWIGLU / DOWN
  const uint32_t* ready;       // landed fill generation per slot
  CUtensorMap mapB2;           // B operand view of the prefill staging area (plan->stage blocks)
  const uint32_t* ready2;      // landed fill generation per staging slot
  int has_stage;               // mapB2 / ready2 valid
  CUtensorMap mapBp, mapB2p;   // DOWN on CTA pairs: mapB / mapB2 with 128-row boxes
  int has_pair_maps;
  int num_sms;                 // persistent grid size (0: the current device's SM count)
  int pick_grid;               // grid of the one-CTA variants (the variant pick must agree across kernels)
  int mt_c2;                   // >0: both m-tiles-per-tile variants are launched and each exits
                               // unless the exact tile counts pick it (cost of a 2-m-tile tile
                               // = mt_c2/100 of a 1-m-tile one); 0: this variant runs
};
cudaError_t preload_tc_kernels();
cudaError_t launch_tc_plain(const TcArgs& p, cudaStream_t s);
cudaError_t launch_tc_swiglu(const TcArgs& p, int max_mtiles, int mt, cudaStream_t s);
cudaError_t launch_tc_down(const TcArgs& p, int max_mtiles, int mt, cudaStream_t s);
void launch_expert_gateup(const ExpertArgs& a, cudaStream_t s, int num_sms);
void launch_expert_down(const ExpertArgs& a, cudaStream_t s, int num_sms);
void launch_write_ready(uint32_t* ready, int slot, uint32_t gen, cudaStream_t s);

// Force-load every kernel of this library now (CUDA lazy loading would otherwise load a
// kernel at its first launch; loading while another kernel spins on a flag can deadlock).
cudaError_t preload_route_kernels();
cudaError_t preload_expert_kernels();

}  // namespace moe
