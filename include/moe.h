/*
 * moe.h — C-ABI of the B200-native expert-cached MoE decode block
 *         (arXiv 2512.16473, "Efficient CPU-GPU Collaborative Inference for
 *          MoE-based LLMs on Memory-Limited Systems").
 *
 * One call of moe_layer_forward() is one pass of the paper's per-layer MoE block
 * at single-request decode (Fig.4a):
 *   router gating — gate GEMV, top-K, softmax over the K      (DESIGN R1/R2)
 *   (1) cache check of the layer's set in the N x M cache
 *   (3) LRU update; a missed expert is fetched from pinned host
 *       memory into its victim slot on a side stream
 *   (2a) SwiGLU expert FFN GEMVs over the (now) resident slots,
 *        combined by the gate weights
 *   tensor-parallel only: per-layer NCCL all-reduce of y        (north_star (4))
 * Layers >= N (beyond coverage) take the miss path through a staging slot
 * and are never inserted.
 *
 * Conventions (all entry points):
 *  - Every call returns moe_status; 0 == MOE_OK. No C++ exception crosses the ABI.
 *    On a non-OK status moe_last_error() returns a thread-local message and the
 *    context is left unchanged (arguments are validated before anything is enqueued).
 *  - No torch types: plain host/device pointers, sizes, and a cudaStream_t passed
 *    as void*. The library sets the context's CUDA device on entry.
 *  - Single-threaded per context: calls on one ctx must not race, and all
 *    moe_layer_forward calls of one ctx must be ordered on one stream.
 *  - Decode batch = 1. bf16 values are passed as their uint16_t bit patterns.
 *  - The decode kernel is a persistent grid of one CTA per SM whose CTAs wait on each other
 *    (grid-wide h / pull counters; across ranks in the fused TP reduction). It is launched
 *    non-cooperatively after an occupancy check, so while a call runs its context expects
 *    the GPU's SMs to itself: kernels of other streams or processes that hold SMs for long
 *    can delay its CTAs (they wait with a 60 s watchdog that traps, poisoning the context).
 *    Set MOE_COOP=1 to have the driver check co-residency at every launch (cooperative
 *    launch, ~2.5 us per call).
 */
#ifndef MOE_H_
#define MOE_H_

#include <stdint.h>

#if defined(__GNUC__)
#define MOE_API __attribute__((visibility("default")))
#else
#define MOE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t moe_status;
#define MOE_OK 0
#define MOE_ERR_INVALID_ARG 1   /* bad pointer / size / index / geometry */
#define MOE_ERR_OUT_OF_MEMORY 2 /* device or pinned-host allocation failed */
#define MOE_ERR_CUDA 3          /* a CUDA runtime/driver call failed */
#define MOE_ERR_NCCL 4          /* NCCL missing or an NCCL call failed */
#define MOE_ERR_STATE 5         /* call out of order (e.g. forward before cache_configure) */
#define MOE_ERR_UNSUPPORTED 6   /* valid but not implemented (e.g. a NEXT policy) */

#define MOE_ABI_VERSION 1
#define MOE_MAX_EXPERTS 32 /* n <= 32: one warp lane per expert / per way in the router kernel */

typedef struct moe_ctx moe_ctx; /* opaque; created by moe_init, freed by moe_destroy */

/* Model shape (Table II) and placement.
 *  num_layers L >= 1; d_model d % 8 == 0; d_ff ff; num_experts n in [1, 32];
 *  top_k K in [1, n]; device = CUDA ordinal.
 *  tp_size P in {1, 2, 4, 8}: each expert's intermediate dimension is split across P
 *  ranks (north_star (4)); ff % (8 * P) == 0; rank tp_rank holds rows
 *  [tp_rank*ff/P, (tp_rank+1)*ff/P) of W1/W3 and the matching columns of W2.
 *  nccl_unique_id: 128 bytes from moe_nccl_unique_id() on rank 0, broadcast by the
 *  caller (e.g. torch.distributed); must be NULL if tp_size == 1. NULL with tp_size > 1
 *  means no NCCL communicator: the y reduction must then be the fused peer-memory one
 *  (moe_tp_connect_ipc / moe_tp_connect_local) before the first forward. */
typedef struct {
  int32_t num_layers, d_model, d_ff, num_experts, top_k;
  int32_t device;
  int32_t tp_size, tp_rank;
  const uint8_t* nccl_unique_id;
} moe_model_desc;

/* Host backing store of ALL weights ("store model weights in CPU memory").
 *  gate[l]          -> Wg of layer l, [n][d] bf16 row-major. Copied to the device at
 *                      moe_init (router networks stay resident on the GPU).
 *  expert_blob[l*n+e] -> this rank's slice of expert e of layer l, one contiguous blob
 *                      of slot_bytes = 3*d*(ff/P)*2 bytes laid out as
 *                      { W1[ff/P][d], W3[ff/P][d], W2[d][ff/P] } (nn.Linear layout).
 *  All pointers are HOST pointers, CALLER-OWNED, and must outlive the ctx.
 *  already_pinned: nonzero if the blobs are page-locked (cudaHostAlloc / torch
 *  pin_memory); 0 -> the library cudaHostRegister()s them and unregisters in
 *  moe_destroy. Copies from unpinned memory would not be asynchronous. */
typedef struct {
  const uint16_t* const* gate;
  const uint16_t* const* expert_blob;
  int32_t already_pinned;
} moe_weights;

/* Validates desc/weights, uploads the gate weights, pins the host blobs, creates the
 * fetch stream (the weight channel of P:226's two streams), the miss-notification
 * mailbox and, if tp_size > 1, the NCCL communicator (collective over the TP group:
 * all ranks must call moe_init concurrently). *out receives the new context. */
MOE_API moe_status moe_init(const moe_model_desc* desc, const moe_weights* weights, moe_ctx** out);

/* Waits for all outstanding work, frees device memory, unpins, destroys the comm. NULL ok. */
MOE_API moe_status moe_destroy(moe_ctx* ctx);

typedef enum {
  MOE_POLICY_LRU = 0,          /* P:217 (default; the paper's policy) */
  MOE_POLICY_FIFO = 1,         /* P:218 compared policy: no recency update on a hit */
  MOE_POLICY_STATIC_RANDOM = 2 /* P:360 analytic baseline: per covered layer M experts drawn at
                                  configure time (seeded partial Fisher-Yates over splitmix64(seed ^
                                  layer<<32 ^ i)), preloaded, never replaced; misses are staged like
                                  uncovered layers' (no insertion, no eviction). warm_start ignored. */
} moe_policy;

/* Cache geometry and policy.
 *  cache_bytes >= 0: S = floor(cache_bytes / slot_bytes), N_raw = floor(S / M)
 *                    (P:214), covered layers = min(N_raw, L) (set l <-> layer l, R7).
 *  cache_bytes == -1: N = indexes directly (0 <= indexes <= L), S = N * M.
 *  ways M: K <= M <= n (M < K is rejected, reading R12).
 *  warm_start: 0 = cold (all ways invalid); 1 = experts 0..M-1 of every covered layer
 *              preloaded into ways 0..M-1 with recency 1..M (blocking H2D; not counted
 *              as fetches; reading R9).
 *  pool/pool_bytes: optional caller-provided DEVICE memory for the slot pool (e.g. a
 *              torch tensor), >= (covered*M + K) * slot_bytes; NULL -> cudaMalloc.
 *              The K extra slots stage uncovered-layer experts.
 *  Resets directory, recency clock, stats, trace and token counters. S == 0 is legal:
 *  every layer is uncovered. Synchronizes the device. */
/* Miss handling.
 *  MOE_MISS_FETCH (default, the B200 design): a missed expert is copied from pinned host
 *    memory into its victim slot on the fetch stream and then computed on the GPU (one
 *    PCIe pass; the same call waits for its fill).
 *  MOE_MISS_HOST_COMPUTE (the paper's ②(b)/③): the router kernel
 *    ships x to host memory; the host cores compute the missed expert from the pinned
 *    backing store while its weights are post-fetched into the victim slot on the fetch
 *    stream "for future access"; the result comes back on a second (activation) stream and
 *    the expert kernel adds it. Layers beyond coverage are computed on the host only
 *    (P:201). A later hit on a slot whose post-fetch has not landed waits for it
 *    (counted in hit_under_fill). Requires K <= 2 (fused expert kernel).
 *  MOE_MISS_PULL (B200 design, no host thread on the path): the call's own kernel copies a
 *    missed expert from the pinned backing store into its victim slot (or staging slot)
 *    with SM loads over PCIe — every CTA pulls a 1/grid share of the blob, a grid-wide
 *    counter orders the copy before the expert GEMVs read the slot — and then computes it
 *    on the GPU. Same cache semantics, counters and trace as MOE_MISS_FETCH (a miss is
 *    filled before its own call computes it: hit_under_fill = 0). Nothing waits on a host
 *    thread or a copy engine, so a call behaves like any stream-ordered kernel under
 *    serialising tools (ncu replay, compute-sanitizer) and inside CUDA graph capture.
 *    Requires every expert blob to be device-accessible pinned memory (cudaHostAlloc,
 *    cudaHostRegister; checked in cache_configure: MOE_ERR_UNSUPPORTED otherwise). */
#define MOE_MISS_FETCH 0
#define MOE_MISS_HOST_COMPUTE 1
#define MOE_MISS_PULL 2

typedef struct {
  int64_t cache_bytes;
  int32_t ways;
  int32_t indexes;
  int32_t policy;
  int32_t warm_start;
  uint64_t seed; /* STATIC_RANDOM only: seed of the resident draw */
  void* pool;
  int64_t pool_bytes;
  int32_t miss_mode;    /* MOE_MISS_FETCH | MOE_MISS_HOST_COMPUTE | MOE_MISS_PULL */
  int32_t host_threads; /* host-compute threads (<= 0: all hardware threads) */
} moe_cache_config;

typedef struct {
  int64_t slots_S, slot_bytes, pool_bytes;
  int32_t ways_M, indexes_N_raw, covered_layers, reserved;
} moe_cache_geometry;

MOE_API moe_status cache_configure(moe_ctx* ctx, const moe_cache_config* cfg, moe_cache_geometry* out);

/* One decode step of the MoE block of `layer` for one token.
 *  x: DEVICE bf16 [d], caller-owned, ready on `stream` at call time.
 *  y: DEVICE fp32 [d], caller-owned, fully overwritten (no residual added); valid once
 *     `stream` reaches this point. TP: every rank passes the same x and gets the
 *     all-reduced y.
 *  stream: cudaStream_t (void*; NULL = legacy default stream).
 * Enqueue-only: never synchronizes the host on the hit path. Calls MUST come in decode
 * order (token-major, layer-ascending): call order defines LRU recency and the
 * token index of each layer (its number of previous calls). Invalid layer ->
 * MOE_ERR_INVALID_ARG and no cache mutation. Misses are filled on the fetch stream by a
 * runtime thread; the expert kernels wait on the slot's ready generation. */
MOE_API moe_status moe_layer_forward(moe_ctx* ctx, int32_t layer, const void* x, float* y, void* stream);

/* Prefill (f4): the MoE block for T prompt tokens at once.
 *  x: DEVICE bf16 [T][d]; y: DEVICE fp32 [T][d] (fully overwritten); both 16-B aligned.
 * For the cache it is exactly T successive moe_layer_forward calls on the rows of x (same
 * routing, hit/miss sequence, counters, trace, token indices); the expert FFN runs batched
 * per distinct routed expert as two tcgen05 tensor-core GEMMs (SwiGLU fused into the first,
 * the gate-weighted combine into the second; h rounded to bf16 between them, so outputs
 * differ from the decode path by up to ~1e-3 relative). Requirements (else
 * MOE_ERR_UNSUPPORTED): full associativity (ways == n), layer covered, MOE_MISS_FETCH or MOE_MISS_PULL,
 * K <= 2, d % 64 == 0, (ff/P) % 128 == 0. First-touch misses are fetched into their slots. */
MOE_API moe_status moe_layer_prefill(moe_ctx* ctx, int32_t layer, const void* x, float* y, int32_t T, void* stream);

/* End-to-end variant of moe_layer_forward with HOST buffers x (bf16 [d]) and y (fp32 [d]):
 * runs the layer on the context's own stream and synchronizes (polling). With pinned,
 * device-mapped buffers (cudaHostAlloc / moe_host_alloc / torch pin_memory, 16-B aligned) on
 * the fused path the kernel reads x from and writes y to host memory itself (zero-copy);
 * otherwise x and y are copied with cudaMemcpyAsync around the kernel. */
MOE_API moe_status moe_layer_forward_host(moe_ctx* ctx, int32_t layer, const uint16_t* x_host, float* y_host);

/* Per-layer counters (Fig.6 hit-rate definitions; SPEC CacheStats S:203-207).
 *  at_least_one_hit = the paper's "expert(s) hit"; all_k_hit = "2 experts hit" (K=2).
 *  expert_misses includes coverage_misses (layers >= N). fetches / fetch_bytes count
 *  host->device expert copies (one per miss, including staging fills).
 *  hit_under_fill: hits on a slot whose fill had not landed yet at probe time (timing
 *  dependent — not part of the bit-exact contract; always 0 with MOE_MISS_FETCH / PULL, where a
 *  miss is filled before its own call computes it).
 *  host_computed: experts computed by the host cores (MOE_MISS_HOST_COMPUTE). In that mode
 *  fetches count post-fetches (covered misses only). */
typedef struct {
  uint64_t accesses, at_least_one_hit, all_k_hit, expert_hits, expert_misses, coverage_misses,
      evictions, fetches, fetch_bytes, hit_under_fill, host_computed;
} moe_layer_stats;

/* layer in [0, L) or -1 for the sum over layers. Synchronizes the context's streams. */
MOE_API moe_status cache_stats(moe_ctx* ctx, int32_t layer, moe_layer_stats* out);

/* One record per (token, layer, rank) in call order (SPEC trace vocabulary S:354).
 *  way = -1 and coverage = 1 for layers beyond coverage; evicted = -1 if no eviction. */
typedef struct {
  uint32_t token;
  uint16_t layer;
  uint8_t rank, hit;
  int16_t expert, evicted;
  int8_t way;
  uint8_t coverage;
  uint16_t reserved;
  float weight; /* gate weight w_r (fp32) */
} moe_access_record;

/* Copies up to cap records (oldest first) into host_out; *n_out = number recorded since
 * cache_configure (may exceed the device ring capacity set by MOE_TRACE_CAP, default
 * 2^20 records; records beyond it are dropped). Synchronizes. */
MOE_API moe_status cache_trace(moe_ctx* ctx, moe_access_record* host_out, int64_t cap, int64_t* n_out);

/* Kernel timing (diagnostics for the roofline report). When enabled, CUDA events are
 * recorded around every kernel on the launch stream. moe_profile_read synchronizes and
 * returns the accumulated device time (ms) and launch count per kernel class:
 *  0 route_probe (router + cache kernel), 1 expert_ffn (the fused persistent expert
 *  kernel; on the split fallback path: the gate/up kernel; prefill: the SwiGLU tensor-core
 *  GEMM), 2 expert_down (split fallback path; prefill: the down tensor-core GEMM),
 *  3 allreduce (TP). Reading resets. */
#define MOE_PROF_KINDS 4
typedef struct {
  double ms[MOE_PROF_KINDS];
  uint64_t launches[MOE_PROF_KINDS];
} moe_profile_t;
MOE_API moe_status moe_profile_enable(moe_ctx* ctx, int32_t enable);
MOE_API moe_status moe_profile_read(moe_ctx* ctx, moe_profile_t* out);

/* Which kernels this context launches (diagnostics): expert_path 1 = fused persistent
 * expert kernel (bulk-copy ring, grid barrier), 0 = split gate/up + down kernels (used
 * when the fused plan does not fit shared memory); pdl = programmatic dependent launch
 * in use; ring_stages / stage_bytes / grid of the fused kernel; tp_reduce = how a
 * tensor-parallel y is summed: 0 none (tp_size 1, or P > 1 with neither NCCL nor a
 * connected exchange yet), 1 ncclAllReduce after the kernel,
 * 2 fused peer-memory reduction in the kernel's epilogue (moe_tp_connect_*). */
typedef struct {
  int32_t expert_path, pdl, ring_stages, stage_bytes, grid, tp_reduce, reserved[2];
} moe_runtime_info;
MOE_API moe_status moe_get_runtime_info(moe_ctx* ctx, moe_runtime_info* out);

/* The host-CPU expert FFN used by MOE_MISS_HOST_COMPUTE, exposed for testing/benchmarking:
 * out[d] = W2 (silu(W1 x) * (W3 x)) for one blob in the slot layout (fp32 accumulation,
 * AVX-512 BF16 when available). threads <= 0: all hardware threads. No GPU needed. */
MOE_API moe_status moe_host_expert_ffn(const uint16_t* blob, const uint16_t* x, int32_t d, int32_t ffr, float* out,
                                       int32_t threads);

/* Page-locked host memory for the backing store (cudaHostAlloc, portable): exact size,
 * no power-of-two rounding. Pass already_pinned = 1 in moe_weights for blobs inside it. */
MOE_API moe_status moe_host_alloc(int64_t bytes, void** out);
MOE_API moe_status moe_host_free(void* p);

/* 128-byte NCCL unique id for a TP group (dlopens libnccl.so.2). */
MOE_API moe_status moe_nccl_unique_id(uint8_t* out128);

/* Fused tensor-parallel reduction over peer memory (north_star (4)).
 * The per-layer sum y = sum_p y^(p) of the ff-split (every rank holds the ff/P slice of
 * every expert) moves INTO the decode kernel's epilogue instead of a separate
 * ncclAllReduce launch. Every term w_r * o_r^(p)[c] of rank p's partial y^(p) (r = routing
 * rank, c = column) is stored, as soon as the kernel has it, into slot [c][p][r] of EVERY
 * rank's exchange buffer as an 8-byte {value, call tag} word (plain stores over NVLink P2P /
 * NVSwitch; a local store for p itself; single-copy atomic, so no fence, counter or grid
 * barrier is needed — the "LL" protocol). Each CTA then polls its own slots of its column
 * slice until every word carries this call's tag and sums the P*K terms of each column in a
 * fixed tree order (K = 2: w_0 o_0^(p) + w_1 o_1^(p) per source rank, then pairs of ranks),
 * so all ranks get bit-identical y (their next layer's routing stays identical).
 * The exchange buffer is double-buffered by call parity, so a rank running one call ahead
 * never overwrites slots a peer is still reading; tags and counters are monotonic.
 * Scope: the fused decode path (K <= 2; moe_get_runtime_info expert_path == 1), both miss
 * modes. The split fallback and moe_layer_prefill keep the NCCL all-reduce (they need a
 * communicator: pass nccl_unique_id).
 *
 * Setup, after moe_init on every rank and before the first forward:
 *   multi-process (one GPU per process): moe_tp_exchange_buffer on every rank -> all-gather
 *     the 64-byte CUDA IPC handles (e.g. torch.distributed) -> moe_tp_connect_ipc on every
 *     rank -> a barrier across ranks (each rank zeroes its own counters in connect).
 *   one process (several contexts; e.g. P ranks emulated on ONE GPU, or P GPUs driven by one
 *     process): moe_tp_connect_local with all P contexts. Contexts on the same device then
 *     split the SMs (grid = #SMs / P each, so the P grids are co-resident) and launch without
 *     PDL; their calls for one layer must be enqueued for all ranks before any rank's next
 *     call is waited on.
 * With a connected exchange, tp_size > 1 contexts may be created with nccl_unique_id NULL
 * (then only the fused decode path is available). Deadlock note: every rank must make the
 * same sequence of forward calls; a rank whose peer never arrives traps after 60 s. */
typedef struct {
  void* dev_ptr;          /* this rank's exchange buffer (device memory, library-owned) */
  int64_t bytes;          /* 256 + 2 * P * K * d * 8 */
  uint8_t ipc_handle[64]; /* cudaIpcMemHandle_t of dev_ptr */
} moe_tp_exchange;
MOE_API moe_status moe_tp_exchange_buffer(moe_ctx* ctx, moe_tp_exchange* out);
/* handles: [P][64] IPC handles of ranks 0..P-1 (this rank's own entry is ignored). Opens the
 * peers' buffers (cudaIpcOpenMemHandle, closed in moe_destroy) and zeroes this rank's
 * counters. MOE_ERR_STATE if tp_size == 1; MOE_ERR_UNSUPPORTED if the fused path is off. */
MOE_API moe_status moe_tp_connect_ipc(moe_ctx* ctx, const uint8_t* handles);
/* ctxs: the P contexts of one TP group (any order; tp_rank must be a permutation of 0..P-1,
 * all with the same shape and tp_size == P). Enables peer access between distinct devices. */
MOE_API moe_status moe_tp_connect_local(moe_ctx* const* ctxs, int32_t P);
/* Back to the NCCL all-reduce (or to no reduction without a communicator): closes the
 * peers' IPC mappings. Use it on every rank when one rank's connect failed. Synchronizes. */
MOE_API moe_status moe_tp_disconnect(moe_ctx* ctx);

MOE_API const char* moe_last_error(void);
MOE_API int32_t moe_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MOE_H_ */
