// runtime.cu — host runtime behind the C-ABI (include/moe.h).
//
// Owns: device copy of the router gates, the expert slot pool and its directory
// (tag / recency stamp per way, fill generation and landed generation per slot), the
// per-layer counters and access trace, the fetch stream (P:226's weight channel), a
// host-mapped miss mailbox and the fetch thread that turns mailbox entries into
// H2D copies + ready-generation writes, optional NCCL communicator for the
// ff-split (north_star (4)), and per-kernel profiling events.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "gate_gemv.cuh"
#include "host_expert.h"
#include "moe_internal.cuh"
#include "nccl.h"
#include <nvtx3/nvToolsExt.h>  // (CUDA toolkit) header-only NVTX: ranges for nsys / ncu when a tool is attached

using namespace moe;

// ----------------------------------------------------------------------------- errors
static thread_local std::string g_err;

static moe_status fail(moe_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? MOE_ERR_OUT_OF_MEMORY : MOE_ERR_CUDA, \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

// ----------------------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
static NcclApi g_nccl;
static std::mutex g_nccl_mu;

static bool nccl_load(std::string* why) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.h) return true;
  const char* env = getenv("MOE_NCCL_LIB");
  void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    *why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
    return false;
  }
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.AllReduce || !g_nccl.CommDestroy) {
    *why = "libnccl.so.2 lacks required symbols";
    dlclose(h);
    return false;
  }
  g_nccl.h = h;
  return true;
}

// ----------------------------------------------------------------------------- context
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2-D bf16 tensor map for tcgen05 operands: rows of `inner` elements (row stride
// row_bytes), box = 64 elements (128 B, one swizzle row) x box_rows, 128-B swizzle.
static bool encode_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t row_bytes,
                          uint32_t box_rows) {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return false;
    }
    fn = (PFN_encodeTiled)f;
  }
  const cuuint64_t dims[2] = {inner, rows};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct ProfEv {
  int kind;
  cudaEvent_t a, b;
};

// Stream timeline (MOE_STREAM_TIMELINE=1, diagnostics): device-timed intervals of every
// kernel launch on the caller's stream, every weight copy on the fetch stream (P:226's weight
// channel) and every host-result copy on the activation stream, so the overlap of PCIe
// transfers with compute can be read without a system profiler (tools/stream_timeline.py).
enum { TL_KERNEL = 0, TL_FETCH = 1, TL_ACT = 2 };
struct TlRec {
  int kind;
  unsigned long long seq;
  long long bytes;
  cudaEvent_t a, b;
};

struct moe_ctx {
  // shape
  int L = 0, d = 0, ff = 0, n = 0, K = 0, P = 1, rank = 0, ffr = 0, device = 0;
  long long slot_bytes = 0;
  int num_sms = 0;
  // weights
  std::vector<const uint16_t*> blobs;
  std::vector<void*> registered;
  const uint8_t** d_hblob = nullptr;  // [L*n] device-accessible aliases of the blobs (MOE_MISS_PULL)
  bool hblob_ok = false;              // every blob is device-accessible pinned memory
  unsigned* d_pull_done = nullptr;    // pull kernel completion counter (split path / prefill)
  uint16_t* d_gate = nullptr;
  // streams
  cudaStream_t fetch_stream = nullptr, own_stream = nullptr;
  PFN_writeValue32 write_value32 = nullptr;
  // cache
  bool configured = false;
  int M = 0, Ncov = 0, Nraw = 0, policy = 0;
  long long S = 0, nslots = 0;
  uint8_t* pool = nullptr;
  bool pool_owned = false;
  long long pool_bytes = 0;
  int32_t* d_tag = nullptr;
  unsigned long long* d_stamp = nullptr;
  uint32_t* d_gen = nullptr;
  uint32_t* d_ready = nullptr;
  unsigned long long* d_clock = nullptr;
  DevStats* d_stats = nullptr;
  RouteRec* d_route = nullptr;
  float* d_h = nullptr;
  float* d_hf = nullptr;
  int plan_RBp = 0;                    // phase-B partials row stride (plan's RB before MOE_ROWS_B)
  int dbg_stale = 0;                   // MOE_DEBUG_STALE_H=1 (debug build): settle fault injection
  static constexpr size_t kDevPtrCache = 1024;  // forward_host: pinned host -> device pointers
  const void* dp_host[kDevPtrCache] = {};       // (identity-mapped pointers seen)               // fused kernel: h [2 (call parity)][K][ffr], see expert_fused.cu
  moe_access_record* d_trace = nullptr;
  long long trace_cap = 0, trace_count = 0;
  std::vector<uint32_t> tokens;  // per-layer call count = token index
  // mailbox + fetch thread
  Mail* h_mail = nullptr;
  Mail* d_mail = nullptr;
  volatile unsigned long long* h_last = nullptr;  // host-mapped progress word
  unsigned long long* d_last = nullptr;
  std::atomic<unsigned long long> issued{0}, consumed{0};
  std::atomic<bool> stop{false};
  std::atomic<int> fetch_error{0};
  std::string fetch_error_msg;
  std::thread fetcher;
  // end-to-end buffers
  uint16_t* d_x_e2e = nullptr;
  float* d_y_e2e = nullptr;
  uint32_t* d_xflag = nullptr;       // x staged by CTA 0 from host memory (zero-copy forward_host)
  uint32_t xseq = 0;
  uint8_t* d_ll1 = nullptr;          // single-rank LL slots: y written straight to host memory
  volatile uint32_t* h_done = nullptr;  // per-CTA completion words of forward_host (host-mapped)
  uint32_t* d_done = nullptr;
  uint32_t done_tag = 0;
  unsigned long long ll_calls = 0;
  // profiling
  bool prof = false;
  std::vector<ProfEv> prof_events;
  std::vector<cudaEvent_t> ev_free;
  double prof_ms[MOE_PROF_KINDS] = {0, 0, 0, 0};
  uint64_t prof_launches[MOE_PROF_KINDS] = {0, 0, 0, 0};
  cudaEvent_t done_ev = nullptr;
  cudaEvent_t host_ev = nullptr;  // completion of moe_layer_forward_host
  bool tl = false;                // MOE_STREAM_TIMELINE
  std::mutex tl_mu;
  std::vector<TlRec> tl_recs;
  cudaEvent_t tl_base = nullptr;
  bool any_call = false;
  // TP
  ncclComm_t comm = nullptr;
  // fused peer-memory TP reduction (f3, moe_tp_connect_*)
  uint8_t* d_xchg = nullptr;          // this rank's exchange buffer (tp_xchg_bytes)
  float* d_ypart = nullptr;           // this rank's partial y^(p) [d]
  uint8_t* tp_peer[8] = {};           // exchange buffers of ranks 0..P-1 (own included)
  std::vector<void*> ipc_opened;      // peers' buffers opened with cudaIpcOpenMemHandle
  bool tp_fused = false;
  unsigned long long tp_calls = 0;
  // fused persistent expert kernel
  bool fused = false, pdl = true;
  FusedPlan plan{};
  int fused_grid = 0;
  unsigned long long* d_bar = nullptr;
  unsigned* d_ctr = nullptr;  // fused kernel work-claim counters
  // MOE_MISS_HOST_COMPUTE: x ring (host-mapped), host outputs, activation stream
  int miss_mode = MOE_MISS_FETCH;
  HostExpert* host = nullptr;
  uint16_t* h_xring = nullptr;
  uint16_t* d_xring = nullptr;
  float* h_hout = nullptr;       // pinned [kMaxK][d]
  float* d_hout = nullptr;       // device [kMaxK][d]
  uint32_t* d_hflag = nullptr;   // device [kMaxK]
  cudaStream_t act_stream = nullptr;
  // prefill (f4) buffers, grown on demand
  int pf_T = 0, pf_rows = 0;
  void* d_pfscratch = nullptr;
  int* d_rt_e = nullptr;
  float* d_rt_w = nullptr;
  PrefillPlan* d_plan = nullptr;
  int* d_tok = nullptr;
  float* d_wrow = nullptr;
  uint16_t* d_xg = nullptr;
  uint16_t* d_hg = nullptr;
  CUtensorMap map_xg{}, map_hg{}, map_pool_d{}, map_pool_f{}, map_pool_f128{};
  bool pool_maps = false;
  // prefill with M < n: logits of the prompt, staging area for routed experts that are not
  // resident at the end of the prompt (n - M slots), its landed generations and tensor maps
  float* d_zbuf = nullptr;
  int zbuf_T = 0;
  uint8_t* d_pfstage = nullptr;
  int pfstage_slots = 0;
  uint32_t* d_pfready = nullptr;
  CUtensorMap map_stage_d{}, map_stage_f{}, map_stage_f128{};
  unsigned long long fused_calls = 0;
  unsigned* h_dbg = nullptr;  // host-mapped kernel progress words (MOE_DEBUG_KERNEL=1)
  unsigned* d_dbg = nullptr;
  unsigned long long* d_ts = nullptr;  // per-CTA phase timestamps (MOE_DEBUG_TS=1)
  unsigned long long* d_ev = nullptr;  // per-CTA stage events (MOE_DEBUG_TS=1)
  bool coop = false;                   // cooperative launch of the fused kernel (MOE_COOP=1)
  unsigned long long* d_sts = nullptr; // per-call step timestamps, ring of kStsRing (MOE_DEBUG_TS=1)
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

cudaEvent_t tl_event() {
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// open / close one timeline interval on stream st (no-ops unless MOE_STREAM_TIMELINE)
void tl_begin(moe_ctx* c, int kind, unsigned long long seq, long long bytes, cudaStream_t st, TlRec* r) {
  if (!c->tl) return;
  r->kind = kind;
  r->seq = seq;
  r->bytes = bytes;
  r->a = tl_event();
  r->b = tl_event();
  cudaEventRecord(r->a, st);
}

void tl_end(moe_ctx* c, cudaStream_t st, TlRec* r) {
  if (!c->tl) return;
  cudaEventRecord(r->b, st);
  std::lock_guard<std::mutex> lk(c->tl_mu);
  if (c->tl_recs.size() < (1u << 20)) c->tl_recs.push_back(*r);
}

void fetch_thread_main(moe_ctx* c) {
  cudaSetDevice(c->device);
  const char* dly = getenv("MOE_DEBUG_FETCH_DELAY_US");  // fault injection (tests only)
  const long delay_us = dly ? atol(dly) : 0;
  const bool log = getenv("MOE_DEBUG_FETCH_LOG") != nullptr;
  unsigned long long next = c->consumed.load() + 1;
  std::chrono::steady_clock::time_point stop_seen{};
  bool stopping = false;
  while (true) {
    Mail* m = &c->h_mail[next % kMailRing];
    if (m->seq != next) {
      // No entry (yet). Once the device progress word reaches `next`, the call's router
      // kernel has completed, so a missing entry means the call had no miss.
      if (*c->h_last >= next) {
        std::atomic_thread_fence(std::memory_order_acquire);
        if (m->seq == next) continue;  // the entry landed between the two reads: process it
        c->consumed.store(next, std::memory_order_release);
        ++next;
        continue;
      }
      if (c->stop.load()) {
        if (next > c->issued.load()) break;
        if (!stopping) { stopping = true; stop_seen = std::chrono::steady_clock::now(); }
        // the device never published (e.g. a trapped kernel): give up after 5 s
        if (std::chrono::steady_clock::now() - stop_seen > std::chrono::seconds(5)) break;
      }
      std::this_thread::sleep_for(std::chrono::microseconds(next <= c->issued.load() ? 2 : 20));
      continue;
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    const int layer = m->layer, nmiss = m->nmiss;
    auto note = [&](cudaError_t err, CUresult cr) {
      if ((err != cudaSuccess || cr != CUDA_SUCCESS) && !c->fetch_error.load()) {
        c->fetch_error_msg = std::string("fetch: ") + cudaGetErrorString(err);
        c->fetch_error.store(1);
      }
    };
    auto publish = [&](cudaStream_t st, uint32_t* word, uint32_t val) -> CUresult {
      if (c->write_value32) return c->write_value32((CUstream)st, (CUdeviceptr)word, val, 0);
      launch_write_ready(word, 0, val, st);
      return CUDA_SUCCESS;
    };
    // weight channel: fills (FETCH) or post-fetches for future calls (HOST_COMPUTE)
    for (int i = 0; i < nmiss; ++i) {
      if (!m->postfetch[i]) continue;
      const int slot = m->slot[i];
      const int e = m->expert[i];
      const uint32_t gen = m->gen[i];
      if (delay_us > 0) std::this_thread::sleep_for(std::chrono::microseconds(delay_us));
      if (log) fprintf(stderr, "[moe fetch] seq=%llu layer=%d expert=%d slot=%d gen=%u\n", next, layer, e, slot, gen);
      nvtxRangePushA("moe fetch (weight copy, fetch stream)");
      TlRec tr;
      tl_begin(c, TL_FETCH, next, c->slot_bytes, c->fetch_stream, &tr);
      const bool stg = m->dest[i] != 0;  // prefill (M < n) staging slot instead of a pool slot
      cudaError_t err = cudaMemcpyAsync((stg ? c->d_pfstage : c->pool) + (long long)slot * c->slot_bytes,
                                        c->blobs[(size_t)layer * c->n + e], (size_t)c->slot_bytes,
                                        cudaMemcpyHostToDevice, c->fetch_stream);
      tl_end(c, c->fetch_stream, &tr);
      nvtxRangePop();
      CUresult cr = CUDA_SUCCESS;
      if (err == cudaSuccess) cr = publish(c->fetch_stream, (stg ? c->d_pfready : c->d_ready) + slot, gen);
      note(err, cr);
    }
    // activation channel: the host cores compute the missed experts
    if (m->host && c->host) {
      const uint16_t* x = c->h_xring + (size_t)(next % kMailRing) * c->d;
      for (int i = 0; i < nmiss; ++i) {
        const int rk = m->rank[i];
        float* o = c->h_hout + (size_t)rk * c->d;
        nvtxRangePushA("moe host expert (host cores)");
        c->host->ffn(c->blobs[(size_t)layer * c->n + m->expert[i]], x, c->d, c->ffr, o);
        nvtxRangePop();
        TlRec tr;
        tl_begin(c, TL_ACT, next, (long long)sizeof(float) * c->d, c->act_stream, &tr);
        cudaError_t err = cudaMemcpyAsync(c->d_hout + (size_t)rk * c->d, o, sizeof(float) * c->d,
                                          cudaMemcpyHostToDevice, c->act_stream);
        tl_end(c, c->act_stream, &tr);
        CUresult cr = CUDA_SUCCESS;
        if (err == cudaSuccess) cr = publish(c->act_stream, c->d_hflag + rk, (uint32_t)next);
        note(err, cr);
      }
    }
    c->consumed.store(next, std::memory_order_release);
    ++next;
  }
}

cudaEvent_t prof_event(moe_ctx* c) {
  if (!c->ev_free.empty()) {
    cudaEvent_t e = c->ev_free.back();
    c->ev_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void prof_begin(moe_ctx* c, int kind, cudaStream_t s, ProfEv* pe) {
  if (!c->prof) return;
  pe->kind = kind;
  pe->a = prof_event(c);
  pe->b = prof_event(c);
  cudaEventRecord(pe->a, s);
}

void prof_end(moe_ctx* c, cudaStream_t s, ProfEv* pe) {
  if (!c->prof) return;
  cudaEventRecord(pe->b, s);
  c->prof_events.push_back(*pe);
  if (c->prof_events.size() > 65536) {  // fold to bound memory
    for (auto& p : c->prof_events) {
      float ms = 0;
      cudaEventSynchronize(p.b);
      cudaEventElapsedTime(&ms, p.a, p.b);
      c->prof_ms[p.kind] += ms;
      c->prof_launches[p.kind] += 1;
      c->ev_free.push_back(p.a);
      c->ev_free.push_back(p.b);
    }
    c->prof_events.clear();
  }
}

void free_cache(moe_ctx* c) {
  if (c->pool_owned && c->pool) cudaFree(c->pool);
  c->pool = nullptr;
  c->pool_owned = false;
  cudaFree(c->d_tag);
  cudaFree(c->d_stamp);
  cudaFree(c->d_gen);
  cudaFree(c->d_ready);
  cudaFree(c->d_clock);
  cudaFree(c->d_stats);
  cudaFree(c->d_trace);
  c->d_tag = nullptr;
  c->d_stamp = nullptr;
  c->d_gen = nullptr;
  c->d_ready = nullptr;
  c->d_clock = nullptr;
  c->d_stats = nullptr;
  c->d_trace = nullptr;
  c->configured = false;
}

// Wait until every issued call's mailbox was consumed and the fetch stream drained.
moe_status drain(moe_ctx* c) {
  if (c->any_call) CUDA_TRY(cudaEventSynchronize(c->done_ev));
  // every issued call has completed on the device, so its progress word is published: the
  // fetch thread catches up within its polling period unless something is broken
  const auto t0 = std::chrono::steady_clock::now();
  while (c->consumed.load(std::memory_order_acquire) < c->issued.load()) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
      return fail(MOE_ERR_STATE, "fetch thread did not reach the last issued call within 60 s");
    std::this_thread::yield();
  }
  CUDA_TRY(cudaStreamSynchronize(c->fetch_stream));
  if (c->act_stream) CUDA_TRY(cudaStreamSynchronize(c->act_stream));
  if (c->fetch_error.load()) return fail(MOE_ERR_CUDA, c->fetch_error_msg);
  return MOE_OK;
}

}  // namespace

// ============================================================================= ABI
extern "C" {

MOE_API const char* moe_last_error(void) { return g_err.c_str(); }
MOE_API int32_t moe_abi_version(void) { return MOE_ABI_VERSION; }

// Debug / test only (not in moe.h): C[M][N] = A[M][K] B[N][K]^T on the tcgen05 path (device
// pointers, bf16 in, fp32 out, K % 64 == 0). Validates descriptors / TMA / TMEM plumbing.
MOE_API int moe_debug_tc_gemm(const void* A, const void* B, float* C, int M, int N, int K, void* stream) {
  static bool loaded = false;
  if (!loaded) {
    if (preload_tc_kernels() != cudaSuccess) return 3;
    loaded = true;
  }
  if (K % 64 || M < 1 || N < 1) return 1;
  TcArgs p;
  memset(&p, 0, sizeof(p));
  if (!encode_map_2d(&p.mapA, A, (uint64_t)K, (uint64_t)M, (uint64_t)K * 2, 128)) return 2;
  if (!encode_map_2d(&p.mapB, B, (uint64_t)K, (uint64_t)N, (uint64_t)K * 2, 128)) return 2;
  p.mode = TC_MODE_PLAIN;
  p.M = M; p.N = N; p.K = K;
  p.C = C;
  cudaError_t e = launch_tc_plain(p, (cudaStream_t)stream);
  return e == cudaSuccess ? 0 : 3;
}

// Debug only (not in moe.h): per-CTA timestamps of the last fused launch -> host.
MOE_API int moe_debug_timestamps(moe_ctx* c, unsigned long long* out, long long cap) {
  // copies at most cap words ([grid][stride]); returns the per-CTA stride (0: no marks)
  if (!c || !c->d_ts) return 0;
  cudaDeviceSynchronize();
  const long long n = (long long)kTsStride * c->fused_grid;
  cudaMemcpy(out, c->d_ts, sizeof(unsigned long long) * (size_t)(cap < n ? cap : n), cudaMemcpyDeviceToHost);
  return kTsStride;
}

// Debug only (not in moe.h): per-CTA stage events of the last fused launch -> host
// ([grid][kEvPerCta][2] {globaltimer ns, bytes | phase << 32}; phase 0/1 = A of segment 0/1,
// 2 + r = B of routing rank r). Entries of earlier calls may remain: filter by time.
MOE_API int moe_debug_events(moe_ctx* c, unsigned long long* out) {
  if (!c || !c->d_ev) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(out, c->d_ev, sizeof(unsigned long long) * 2 * kEvPerCta * c->fused_grid, cudaMemcpyDeviceToHost);
  return kEvPerCta;
}

// Debug only (not in moe.h): the per-call step timestamps (globaltimer ns) of the last
// kStsRing calls, [kStsRing][kStsHead + 2*grid] = router marks (after its PDL wait, publish,
// gate GEMV done, softmax done, before the release fence), expert CTA starts, expert CTA ends; slot = seq % kStsRing. Returns the record stride or 0.
MOE_API int moe_debug_step_ts(moe_ctx* c, unsigned long long* out) {
  if (!c || !c->d_sts) return 0;
  cudaDeviceSynchronize();
  const int stride = kStsHead + 2 * c->fused_grid;
  cudaMemcpy(out, c->d_sts, sizeof(unsigned long long) * kStsRing * stride, cudaMemcpyDeviceToHost);
  return stride;
}

// Debug only (not in moe.h): host pointer to the mapped kernel progress words, or NULL.
MOE_API const unsigned* moe_debug_words(moe_ctx* c) { return c ? c->h_dbg : nullptr; }

MOE_API moe_status moe_host_expert_ffn(const uint16_t* blob, const uint16_t* x, int32_t d, int32_t ffr, float* out,
                                       int32_t threads) {
  if (!blob || !x || !out || d < 1 || ffr < 1) return fail(MOE_ERR_INVALID_ARG, "bad argument");
  HostExpert he(threads);
  he.ffn(blob, x, d, ffr, out);
  return MOE_OK;
}

MOE_API moe_status moe_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes <= 0) return fail(MOE_ERR_INVALID_ARG, "bad argument");
  *out = nullptr;
  cudaError_t e = cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    return fail(MOE_ERR_OUT_OF_MEMORY, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
  }
  return MOE_OK;
}

MOE_API moe_status moe_host_free(void* p) {
  if (!p) return MOE_OK;
  CUDA_TRY(cudaFreeHost(p));
  return MOE_OK;
}

MOE_API moe_status moe_nccl_unique_id(uint8_t* out128) {
  if (!out128) return fail(MOE_ERR_INVALID_ARG, "out128 is NULL");
  std::string why;
  if (!nccl_load(&why)) return fail(MOE_ERR_NCCL, why);
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(MOE_ERR_NCCL, "ncclGetUniqueId failed");
  static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
  memcpy(out128, &id, 128);
  return MOE_OK;
}

MOE_API moe_status moe_init(const moe_model_desc* desc, const moe_weights* w, moe_ctx** out) {
  if (!desc || !w || !out) return fail(MOE_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  const int L = desc->num_layers, d = desc->d_model, ff = desc->d_ff, n = desc->num_experts,
            K = desc->top_k, P = desc->tp_size, rank = desc->tp_rank;
  if (L < 1 || d < 8 || d % 8 || ff < 8 || n < 1 || n > MOE_MAX_EXPERTS || K < 1 || K > n)
    return fail(MOE_ERR_INVALID_ARG, "bad shape (need L>=1, d%8==0, 1<=K<=n<=32)");
  if (!(P == 1 || P == 2 || P == 4 || P == 8) || rank < 0 || rank >= P || ff % (8 * P))
    return fail(MOE_ERR_INVALID_ARG, "bad tensor-parallel split (P in {1,2,4,8}, ff % (8P) == 0)");
  if (P == 1 && desc->nccl_unique_id != nullptr)
    return fail(MOE_ERR_INVALID_ARG, "nccl_unique_id must be NULL if tp_size == 1");
  if (!w->gate || !w->expert_blob) return fail(MOE_ERR_INVALID_ARG, "NULL weight table");
  for (int l = 0; l < L; ++l)
    if (!w->gate[l]) return fail(MOE_ERR_INVALID_ARG, "NULL gate pointer");
  for (int i = 0; i < L * n; ++i)
    if (!w->expert_blob[i]) return fail(MOE_ERR_INVALID_ARG, "NULL expert blob pointer");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (desc->device < 0 || desc->device >= ndev) return fail(MOE_ERR_INVALID_ARG, "bad device ordinal");
  DeviceGuard g(desc->device);

  moe_ctx* c = new moe_ctx();
  c->L = L; c->d = d; c->ff = ff; c->n = n; c->K = K; c->P = P; c->rank = rank;
  c->ffr = ff / P; c->device = desc->device;
  c->slot_bytes = 3ll * d * c->ffr * 2;
  c->tokens.assign(L, 0);
  auto bail = [&](moe_status st) {
    moe_destroy(c);
    return st;
  };
  cudaError_t e;
#define INIT_TRY(expr)                                                                  \
  do {                                                                                  \
    e = (expr);                                                                         \
    if (e != cudaSuccess)                                                               \
      return bail(fail(e == cudaErrorMemoryAllocation ? MOE_ERR_OUT_OF_MEMORY : MOE_ERR_CUDA, \
                       std::string(#expr) + ": " + cudaGetErrorString(e)));             \
  } while (0)
  INIT_TRY(preload_route_kernels());
  INIT_TRY(preload_expert_kernels());
  INIT_TRY(preload_fused_kernels());
  INIT_TRY(preload_tc_kernels());
  INIT_TRY(preload_prefill_kernels());
  INIT_TRY(preload_pull_kernels());
  INIT_TRY(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  c->blobs.assign(w->expert_blob, w->expert_blob + (size_t)L * n);
  if (!w->already_pinned) {
    for (auto* b : c->blobs) {
      e = cudaHostRegister((void*)b, (size_t)c->slot_bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
      if (e == cudaSuccess) c->registered.push_back((void*)b);
      else if (e == cudaErrorHostMemoryAlreadyRegistered) cudaGetLastError();
      else return bail(fail(MOE_ERR_CUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e)));
    }
  }
  {
    // device aliases of the pinned blobs, read by the kernels in MOE_MISS_PULL mode
    std::vector<const uint8_t*> hb((size_t)L * n);
    c->hblob_ok = true;
    for (size_t i = 0; i < hb.size() && c->hblob_ok; ++i) {
      void* dp = nullptr;
      if (cudaHostGetDevicePointer(&dp, (void*)c->blobs[i], 0) != cudaSuccess || !dp || ((uintptr_t)dp & 15)) {
        cudaGetLastError();
        c->hblob_ok = false;
      }
      hb[i] = (const uint8_t*)dp;
    }
    INIT_TRY(cudaMalloc(&c->d_hblob, sizeof(const uint8_t*) * hb.size()));
    if (c->hblob_ok)
      INIT_TRY(cudaMemcpy(c->d_hblob, hb.data(), sizeof(const uint8_t*) * hb.size(), cudaMemcpyHostToDevice));
    INIT_TRY(cudaMalloc(&c->d_pull_done, sizeof(unsigned)));
    INIT_TRY(cudaMemset(c->d_pull_done, 0, sizeof(unsigned)));
  }
  const size_t gate_elems = (size_t)n * d;
  INIT_TRY(cudaMalloc(&c->d_gate, gate_elems * 2 * L));
  for (int l = 0; l < L; ++l)
    INIT_TRY(cudaMemcpy(c->d_gate + gate_elems * l, w->gate[l], gate_elems * 2, cudaMemcpyHostToDevice));
  INIT_TRY(cudaStreamCreateWithFlags(&c->fetch_stream, cudaStreamNonBlocking));
  INIT_TRY(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
  INIT_TRY(cudaEventCreateWithFlags(&c->done_ev, cudaEventDisableTiming));
  INIT_TRY(cudaEventCreateWithFlags(&c->host_ev, cudaEventDisableTiming));
  INIT_TRY(cudaHostAlloc((void**)&c->h_mail, sizeof(Mail) * kMailRing, cudaHostAllocMapped));
  memset((void*)c->h_mail, 0, sizeof(Mail) * kMailRing);
  INIT_TRY(cudaHostGetDevicePointer((void**)&c->d_mail, c->h_mail, 0));
  {
    unsigned long long* hl = nullptr;
    INIT_TRY(cudaHostAlloc((void**)&hl, 64, cudaHostAllocMapped));
    memset(hl, 0, 64);
    c->h_last = hl;
    INIT_TRY(cudaHostGetDevicePointer((void**)&c->d_last, hl, 0));
  }
  INIT_TRY(cudaMalloc(&c->d_route, sizeof(RouteRec)));
  INIT_TRY(cudaMalloc(&c->d_h, sizeof(float) * (size_t)K * c->ffr));
  // the fused kernel's h: two buffers by call parity, every word armed with the "not yet
  // written" pattern (expert_fused.cu: relaxed h publication)
  INIT_TRY(cudaMalloc(&c->d_hf, sizeof(float) * 2 * (size_t)K * c->ffr));
  INIT_TRY(cudaMemset(c->d_hf, 0xff, sizeof(float) * 2 * (size_t)K * c->ffr));
  INIT_TRY(cudaMalloc(&c->d_x_e2e, sizeof(uint16_t) * d));
  INIT_TRY(cudaMalloc(&c->d_y_e2e, sizeof(float) * d));
  INIT_TRY(cudaMalloc(&c->d_xflag, sizeof(uint32_t)));
  INIT_TRY(cudaMemset(c->d_xflag, 0, sizeof(uint32_t)));
  INIT_TRY(cudaMalloc(&c->d_bar, sizeof(unsigned long long) * 16 * kMaxK));
  INIT_TRY(cudaMemset(c->d_bar, 0, sizeof(unsigned long long) * 16 * kMaxK));
  INIT_TRY(cudaMalloc(&c->d_ctr, sizeof(unsigned) * kCtrWords));
  INIT_TRY(cudaHostAlloc((void**)&c->h_xring, sizeof(uint16_t) * (size_t)d * kMailRing, cudaHostAllocMapped));
  INIT_TRY(cudaHostGetDevicePointer((void**)&c->d_xring, c->h_xring, 0));
  INIT_TRY(cudaHostAlloc((void**)&c->h_hout, sizeof(float) * (size_t)d * kMaxK, cudaHostAllocDefault));
  INIT_TRY(cudaMalloc(&c->d_hout, sizeof(float) * (size_t)d * kMaxK));
  INIT_TRY(cudaMalloc(&c->d_hflag, sizeof(uint32_t) * kMaxK));
  INIT_TRY(cudaMemset(c->d_hflag, 0, sizeof(uint32_t) * kMaxK));
  INIT_TRY(cudaStreamCreateWithFlags(&c->act_stream, cudaStreamNonBlocking));
  INIT_TRY(cudaMemset(c->d_ctr, 0, sizeof(unsigned) * kCtrWords));
  {
    const char* path = getenv("MOE_EXPERT_PATH");
    const char* pdl = getenv("MOE_PDL");
    c->pdl = !(pdl && pdl[0] == '0');
    // The fused grid is one CTA per SM and its CTAs wait on each other, so it must be fully
    // resident: guaranteed by the occupancy check below while nothing else holds SMs for
    // long (MOE_COOP=1 makes the launch cooperative — the driver then checks co-residency —
    // at the cost of the early PDL start, ~2.5 us per call).
    const char* coop = getenv("MOE_COOP");
    c->coop = coop && coop[0] == '1';
    c->fused_grid = c->num_sms;
    c->fused = !(path && strcmp(path, "split") == 0) && plan_fused(d, c->ffr, n, K, c->fused_grid, &c->plan) &&
               fused_blocks_per_sm(c->plan) >= 1;
    if (c->fused) {  // schedule knobs (experiments): static share of phase A / B rows, percent
      const char* pa = getenv("MOE_STATIC_A");
      const char* pb = getenv("MOE_STATIC_B");
      if (pa && atoi(pa) >= 0 && atoi(pa) <= 100) c->plan.pctA = atoi(pa);
      if (pb && atoi(pb) >= 0 && atoi(pb) <= 100) c->plan.pctB = atoi(pb);
      const char* pfb = getenv("MOE_PREFETCH_B");  // L2 prefetch of the first W2 rows (default on)
      if (pfb && pfb[0] == '0') c->plan.prefetchB = 0;
      const char* pa2 = getenv("MOE_PF_AHEAD_A");     // phase-A static rows prefetched ahead into L2
      if (pa2 && atoi(pa2) >= 0) c->plan.pfA = atoi(pa2);
      const char* pb2 = getenv("MOE_PF_AHEAD_B");     // phase-B: the next claim's rows into L2
      if (pb2) c->plan.pfB = pb2[0] == '1';
      const char* pfn = getenv("MOE_PREFETCH_NEXT");  // rows of the next call's set warmed in L2
      if (pfn && atoi(pfn) >= 0) c->plan.next_rows = atoi(pfn);
      const char* pfs = getenv("MOE_PREFETCH_START");  // rows of this call's set warmed before the PDL wait
      if (pfs && atoi(pfs) >= 0) c->plan.start_rows = atoi(pfs);
      const char* pfx = getenv("MOE_PREFETCH_X");      // x into L2 before the PDL wait
      if (pfx) c->plan.pfx = pfx[0] == '1';
      c->plan_RBp = c->plan.RB;                   // (before MOE_ROWS_B)
      const char* ca = getenv("MOE_CLAIM_AHEAD");  // next segment's first claim issued early
      if (ca) c->plan.claim_ahead = ca[0] == '1';
      const char* lm = getenv("MOE_LAZY_MARKS");   // end-of-A markers per super-stage, lazily
      if (lm) c->plan.lazy_marks = lm[0] == '1';
      const char* xs = getenv("MOE_XSEP");        // x beside one h buffer (default: when the plan allows)
      if (xs && xs[0] == '0') c->plan.xsep = 0;
      const char* mg = getenv("MOE_MERGE");   // merged phases (default: when the plan allows)
      if (mg && mg[0] == '0') c->plan.merge = 0;
      const char* rb = getenv("MOE_ROWS_B");  // W2 rows per phase-B super-stage (<= plan's)
      if (rb && atoi(rb) >= 1 && atoi(rb) < c->plan.RB) c->plan.RB = atoi(rb);
    }
    c->dbg_stale = getenv("MOE_DEBUG_STALE_H") != nullptr;
    if (getenv("MOE_STREAM_TIMELINE")) {
      c->tl = true;
      INIT_TRY(cudaEventCreate(&c->tl_base));
      INIT_TRY(cudaEventRecord(c->tl_base, c->own_stream));
    }
    if (getenv("MOE_DEBUG_KERNEL")) {  // progress words in host-mapped memory (slow: PCIe atomics)
      INIT_TRY(cudaHostAlloc((void**)&c->h_dbg, 64, cudaHostAllocMapped));
      memset(c->h_dbg, 0, 64);
      INIT_TRY(cudaHostGetDevicePointer((void**)&c->d_dbg, c->h_dbg, 0));
    }
    if (getenv("MOE_DEBUG_TS")) {      // per-CTA phase timestamps in device memory (cheap)
      INIT_TRY(cudaMalloc(&c->d_ts, sizeof(unsigned long long) * kTsStride * c->fused_grid));
      INIT_TRY(cudaMemset(c->d_ts, 0, sizeof(unsigned long long) * kTsStride * c->fused_grid));
      INIT_TRY(cudaMalloc(&c->d_ev, sizeof(unsigned long long) * 2 * kEvPerCta * c->fused_grid));
      INIT_TRY(cudaMemset(c->d_ev, 0, sizeof(unsigned long long) * 2 * kEvPerCta * c->fused_grid));
      INIT_TRY(cudaMalloc(&c->d_sts, sizeof(unsigned long long) * kStsRing * (kStsHead + 2 * c->fused_grid)));
      INIT_TRY(cudaMemset(c->d_sts, 0, sizeof(unsigned long long) * kStsRing * (kStsHead + 2 * c->fused_grid)));
    }
    if (getenv("MOE_DEBUG_KERNEL") || getenv("MOE_DEBUG_TS")) {
      fprintf(stderr, "[moe init] fused=%d NS=%d SB=%d RB=%d merge=%d xsep=%d xh=%d smem=%zu grid=%d\n", (int)c->fused,
              c->plan.NS, c->plan.SB, c->plan.RB, c->plan.merge, c->plan.xsep, c->plan.xh_bytes, c->plan.smem,
              c->fused_grid);
  }
  }
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &fn, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      c->write_value32 = (PFN_writeValue32)fn;
    cudaGetLastError();
    if (getenv("MOE_DEBUG_FETCH_LOG"))
      fprintf(stderr, "[moe init] cuStreamWriteValue32 %s\n", c->write_value32 ? "available" : "MISSING");
  }
  if (P > 1 && desc->nccl_unique_id) {
    std::string why;
    if (!nccl_load(&why)) return bail(fail(MOE_ERR_NCCL, why));
    ncclUniqueId id;
    memcpy(&id, desc->nccl_unique_id, sizeof(id));
    ncclResult_t r = g_nccl.CommInitRank(&c->comm, P, id, rank);
    if (r != ncclSuccess) {
      c->comm = nullptr;
      return bail(fail(MOE_ERR_NCCL, std::string("ncclCommInitRank: ") +
                                         (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?")));
    }
  }
#undef INIT_TRY
  c->fetcher = std::thread(fetch_thread_main, c);
  *out = c;
  return MOE_OK;
}

MOE_API moe_status moe_destroy(moe_ctx* c) {
  if (!c) return MOE_OK;
  DeviceGuard g(c->device);
  if (c->any_call) cudaEventSynchronize(c->done_ev);
  c->stop.store(true);
  if (c->fetcher.joinable()) c->fetcher.join();
  if (c->fetch_stream) cudaStreamSynchronize(c->fetch_stream);
  if (c->act_stream) cudaStreamSynchronize(c->act_stream);
  for (auto& p : c->prof_events) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->ev_free) cudaEventDestroy(e);
  for (auto& r : c->tl_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  if (c->tl_base) cudaEventDestroy(c->tl_base);
  free_cache(c);
  cudaFree(c->d_gate);
  cudaFree(c->d_hblob);
  cudaFree(c->d_pull_done);
  cudaFree(c->d_route);
  cudaFree(c->d_h);
  cudaFree(c->d_hf);
  cudaFree(c->d_x_e2e);
  cudaFree(c->d_y_e2e);
  cudaFree(c->d_xflag);
  cudaFree(c->d_ll1);
  if (c->h_done) cudaFreeHost((void*)c->h_done);
  cudaFree(c->d_bar);
  cudaFree(c->d_ctr);
  cudaFree(c->d_hout);
  cudaFree(c->d_hflag);
  cudaFree(c->d_pfscratch);
  cudaFree(c->d_rt_e);
  cudaFree(c->d_rt_w);
  cudaFree(c->d_plan);
  cudaFree(c->d_tok);
  cudaFree(c->d_wrow);
  cudaFree(c->d_xg);
  cudaFree(c->d_hg);
  cudaFree(c->d_zbuf);
  cudaFree(c->d_pfstage);
  cudaFree(c->d_pfready);
  if (c->h_xring) cudaFreeHost(c->h_xring);
  if (c->h_hout) cudaFreeHost(c->h_hout);
  if (c->act_stream) cudaStreamDestroy(c->act_stream);
  delete c->host;
  c->host = nullptr;
  cudaFree(c->d_ts);
  cudaFree(c->d_ev);
  cudaFree(c->d_sts);
  if (c->h_mail) cudaFreeHost(c->h_mail);
  if (c->h_last) cudaFreeHost((void*)c->h_last);
  for (void* p : c->registered) cudaHostUnregister(p);
  if (c->done_ev) cudaEventDestroy(c->done_ev);
  if (c->host_ev) cudaEventDestroy(c->host_ev);
  if (c->fetch_stream) cudaStreamDestroy(c->fetch_stream);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  cudaFree(c->d_xchg);
  cudaFree(c->d_ypart);
  cudaGetLastError();
  delete c;
  return MOE_OK;
}

MOE_API moe_status cache_configure(moe_ctx* c, const moe_cache_config* cfg, moe_cache_geometry* out) {
  if (!c || !cfg) return fail(MOE_ERR_INVALID_ARG, "NULL argument");
  DeviceGuard g(c->device);
  const int M = cfg->ways;
  if (M < c->K || M > c->n) return fail(MOE_ERR_INVALID_ARG, "ways must satisfy K <= M <= n");
  if (cfg->miss_mode != MOE_MISS_FETCH && cfg->miss_mode != MOE_MISS_HOST_COMPUTE && cfg->miss_mode != MOE_MISS_PULL)
    return fail(MOE_ERR_INVALID_ARG, "unknown miss_mode");
  if (cfg->miss_mode == MOE_MISS_PULL && !c->hblob_ok)
    return fail(MOE_ERR_UNSUPPORTED, "MOE_MISS_PULL needs device-accessible pinned expert blobs");
  if (cfg->miss_mode == MOE_MISS_HOST_COMPUTE && !c->fused)
    return fail(MOE_ERR_UNSUPPORTED, "MOE_MISS_HOST_COMPUTE needs the fused expert kernel (K <= 2)");
  if (cfg->policy != MOE_POLICY_LRU && cfg->policy != MOE_POLICY_FIFO && cfg->policy != MOE_POLICY_STATIC_RANDOM)
    return fail(MOE_ERR_INVALID_ARG, "unknown policy");
  long long S;
  int Nraw;
  if (cfg->cache_bytes >= 0) {
    S = cfg->cache_bytes / c->slot_bytes;
    Nraw = (int)(S / M);
  } else if (cfg->cache_bytes == -1) {
    if (cfg->indexes < 0 || cfg->indexes > c->L) return fail(MOE_ERR_INVALID_ARG, "indexes out of [0, L]");
    Nraw = cfg->indexes;
    S = (long long)Nraw * M;
  } else {
    return fail(MOE_ERR_INVALID_ARG, "cache_bytes must be >= 0 or -1");
  }
  const int Ncov = Nraw < c->L ? Nraw : c->L;
  const long long nslots = (long long)Ncov * M + c->K;  // + K staging slots
  const long long need = nslots * c->slot_bytes;
  if (cfg->pool && cfg->pool_bytes < need)
    return fail(MOE_ERR_INVALID_ARG, "caller pool too small: need " + std::to_string(need) + " bytes");
  moe_status st = drain(c);
  if (st != MOE_OK) return st;
  free_cache(c);
  if (cfg->pool) {
    c->pool = (uint8_t*)cfg->pool;
    c->pool_owned = false;
  } else {
    cudaError_t e = cudaMalloc(&c->pool, (size_t)need);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c->pool = nullptr;
      return fail(MOE_ERR_OUT_OF_MEMORY, "slot pool cudaMalloc(" + std::to_string(need) + ") failed");
    }
    c->pool_owned = true;
  }
  c->M = M; c->Ncov = Ncov; c->Nraw = Nraw; c->S = S; c->nslots = nslots;
  c->policy = cfg->policy; c->pool_bytes = need;
  c->miss_mode = cfg->miss_mode;
  if (c->miss_mode == MOE_MISS_HOST_COMPUTE && !c->host) c->host = new HostExpert(cfg->host_threads);
  CUDA_TRY(cudaMemset(c->d_hflag, 0, sizeof(uint32_t) * kMaxK));
  const long long nways = (long long)(Ncov > 0 ? Ncov : 1) * M;
  CUDA_TRY(cudaMalloc(&c->d_tag, sizeof(int32_t) * nways));
  CUDA_TRY(cudaMalloc(&c->d_stamp, sizeof(unsigned long long) * nways));
  CUDA_TRY(cudaMalloc(&c->d_gen, sizeof(uint32_t) * nslots));
  CUDA_TRY(cudaMalloc(&c->d_ready, sizeof(uint32_t) * nslots));
  CUDA_TRY(cudaMalloc(&c->d_clock, sizeof(unsigned long long)));
  CUDA_TRY(cudaMalloc(&c->d_stats, sizeof(DevStats) * c->L));
  const char* tc = getenv("MOE_TRACE_CAP");
  c->trace_cap = tc ? atoll(tc) : (1ll << 20);
  if (c->trace_cap < 0) c->trace_cap = 0;
  CUDA_TRY(cudaMalloc(&c->d_trace, sizeof(moe_access_record) * (c->trace_cap > 0 ? c->trace_cap : 1)));
  // directory: cold = all invalid; warm = experts 0..M-1 in ways 0..M-1, stamps 1..M (R9)
  std::vector<int32_t> tag(nways, -1);
  std::vector<unsigned long long> stamp(nways, 0);
  std::vector<uint32_t> gen(nslots, 0);
  unsigned long long clock = 0;
  if (cfg->policy == MOE_POLICY_STATIC_RANDOM) {
    // "randomly selecting a set of expert networks to be stored in the cache
    // statically": per covered layer, M distinct experts drawn with a seeded partial
    // Fisher-Yates shuffle (counter-based splitmix64 keyed by (seed, layer, i)), way i holds
    // the i-th draw; loaded once here, never replaced.
    for (int s = 0; s < Ncov; ++s) {
      std::vector<int> perm(c->n);
      for (int e = 0; e < c->n; ++e) perm[e] = e;
      for (int i = 0; i < M; ++i) {
        uint64_t z = cfg->seed ^ ((uint64_t)(uint32_t)s << 32) ^ (uint64_t)(uint32_t)i;
        z += 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const int j = i + (int)(z % (uint64_t)(c->n - i));
        std::swap(perm[i], perm[j]);
      }
      for (int wy = 0; wy < M; ++wy) {
        tag[(size_t)s * M + wy] = perm[wy];
        stamp[(size_t)s * M + wy] = 0;
        gen[(size_t)s * M + wy] = 1;
        CUDA_TRY(cudaMemcpyAsync(c->pool + ((long long)s * M + wy) * c->slot_bytes,
                                 c->blobs[(size_t)s * c->n + perm[wy]], (size_t)c->slot_bytes,
                                 cudaMemcpyHostToDevice, c->fetch_stream));
      }
    }
  } else if (cfg->warm_start) {
    for (int s = 0; s < Ncov; ++s)
      for (int wy = 0; wy < M; ++wy) {
        tag[(size_t)s * M + wy] = wy;
        stamp[(size_t)s * M + wy] = wy + 1;
        gen[(size_t)s * M + wy] = 1;
        CUDA_TRY(cudaMemcpyAsync(c->pool + ((long long)s * M + wy) * c->slot_bytes,
                                 c->blobs[(size_t)s * c->n + wy], (size_t)c->slot_bytes,
                                 cudaMemcpyHostToDevice, c->fetch_stream));
      }
    clock = M;
  }
  CUDA_TRY(cudaMemcpyAsync(c->d_tag, tag.data(), sizeof(int32_t) * nways, cudaMemcpyHostToDevice, c->fetch_stream));
  CUDA_TRY(cudaMemcpyAsync(c->d_stamp, stamp.data(), sizeof(unsigned long long) * nways, cudaMemcpyHostToDevice, c->fetch_stream));
  CUDA_TRY(cudaMemcpyAsync(c->d_gen, gen.data(), sizeof(uint32_t) * nslots, cudaMemcpyHostToDevice, c->fetch_stream));
  CUDA_TRY(cudaMemcpyAsync(c->d_ready, gen.data(), sizeof(uint32_t) * nslots, cudaMemcpyHostToDevice, c->fetch_stream));
  CUDA_TRY(cudaMemcpyAsync(c->d_clock, &clock, sizeof(clock), cudaMemcpyHostToDevice, c->fetch_stream));
  CUDA_TRY(cudaMemsetAsync(c->d_stats, 0, sizeof(DevStats) * c->L, c->fetch_stream));
  CUDA_TRY(cudaStreamSynchronize(c->fetch_stream));
  CUDA_TRY(cudaDeviceSynchronize());
  c->trace_count = 0;
  std::fill(c->tokens.begin(), c->tokens.end(), 0u);
  c->configured = true;
  c->pool_maps = false;
  if (out) {
    out->slots_S = S;
    out->slot_bytes = c->slot_bytes;
    out->pool_bytes = need;
    out->ways_M = M;
    out->indexes_N_raw = Nraw;
    out->covered_layers = Ncov;
    out->reserved = 0;
  }
  return MOE_OK;
}

// Virtual warps of the gate-logit summation order (gate_gemv.cuh): the fused kernel's
// consumer warps, so that every path (fused, split, prefill) rounds the logits alike.
static int gate_warps(const moe_ctx* c) { return c->fused ? 2 * c->plan.NS : kGateWarpsDefault; }

// xhost / yhost (moe_layer_forward_host, fused path): device-accessible pinned host buffers;
// the kernel reads x from xhost into the staging buffer x and writes y straight to yhost.
static moe_status forward_impl(moe_ctx* c, int32_t layer, const void* x, float* y, cudaStream_t s,
                               const uint16_t* xhost = nullptr, float* yhost = nullptr, uint32_t donetag = 0) {
  if (!c->configured) return fail(MOE_ERR_STATE, "cache_configure() has not been called");
  if (layer < 0 || layer >= c->L) return fail(MOE_ERR_INVALID_ARG, "layer out of range");
  if (!x || !y) return fail(MOE_ERR_INVALID_ARG, "NULL x or y");
  if (((uintptr_t)x & 15) || ((uintptr_t)y & 15)) return fail(MOE_ERR_INVALID_ARG, "x and y must be 16-byte aligned");
  if (c->fetch_error.load()) return fail(MOE_ERR_CUDA, c->fetch_error_msg);
  const bool tpf = c->P > 1 && c->tp_fused && c->fused;  // y summed in the kernel's epilogue (f3)
  const bool ll1 = yhost && !tpf && c->fused;             // single-rank LL: y -> host memory
  if (c->P > 1 && !tpf && !c->comm)
    return fail(MOE_ERR_STATE, "tp_size > 1 without an NCCL communicator needs moe_tp_connect_* (fused path)");
  // host-side back-pressure: never let the GPU overwrite an unconsumed mailbox entry
  const unsigned long long seq = c->issued.load() + 1;
  while (seq - c->consumed.load(std::memory_order_acquire) >= (unsigned long long)kMailRing - 1)
    std::this_thread::yield();
  const bool covered = layer < c->Ncov;
  RouteArgs ra;
  ra.Wg = c->d_gate + (size_t)layer * c->n * c->d;
  ra.x = (const uint16_t*)x;
  ra.d = c->d; ra.n = c->n; ra.K = c->K; ra.M = c->M; ra.layer = layer;
  ra.covered = covered; ra.policy = c->policy; ra.miss_mode = c->miss_mode;
  ra.gw = gate_warps(c);
  ra.xmail = c->d_xring + (size_t)(seq % kMailRing) * c->d;
  ra.tag = covered ? c->d_tag + (size_t)layer * c->M : nullptr;
  ra.stamp = covered ? c->d_stamp + (size_t)layer * c->M : nullptr;
  ra.slot_base = covered ? layer * c->M : 0;
  ra.staging_base = c->Ncov * c->M;
  ra.gen = c->d_gen;
  ra.ready = c->d_ready;
  ra.clock = c->d_clock;
  ra.stats = c->d_stats + layer;
  ra.route = c->d_route;
  ra.trace = c->d_trace;
  ra.trace_idx = c->trace_count;
  ra.trace_cap = c->trace_cap;
  ra.token = c->tokens[layer];
  ra.mail = c->d_mail + (seq % kMailRing);
  ra.seq = seq;
  ra.sts = c->d_sts ? c->d_sts + (seq % kStsRing) * (kStsHead + 2 * c->fused_grid) : nullptr;
  ra.slot_bytes = c->slot_bytes;
  ra.hblob = c->d_hblob + (size_t)layer * c->n;
  ra.last_seq = c->d_last;

  ExpertArgs ea;
  ea.route = c->d_route;
  ea.pool = c->pool;
  ea.slot_bytes = c->slot_bytes;
  ea.x = (const uint16_t*)x;
  ea.d = c->d; ea.ffr = c->ffr; ea.K = c->K;
  ea.h = c->d_h;
  ea.y = (tpf || ll1) ? c->d_ypart : y;
  ea.ready = c->d_ready;
  ea.last_seq = c->d_last;
  ea.seq = seq;
  ea.host_out = c->d_hout;
  ea.host_flag = c->d_hflag;

  ProfEv pe;
  if (c->fused) {
    // ONE kernel per call: every CTA takes the routing decision itself (CTA 0 writes the
    // directory, trace, counters and mailbox), then streams the experts
    FusedArgs fa;
    fa.r = ra;
    fa.e = ea;
    fa.bar = c->d_bar;
    fa.hf = c->d_hf;
    fa.calls = c->fused_calls;
    fa.ctr = c->d_ctr;
    fa.NS = c->plan.NS;
    fa.SB = c->plan.SB;
    fa.xh_bytes = c->plan.xh_bytes;
    fa.pctA = c->plan.pctA;
    fa.pctB = c->plan.pctB;
    fa.RB = c->plan.RB;
    fa.RBp = c->plan_RBp;
    fa.xsep = c->plan.xsep;
    fa.claim_ahead = c->plan.claim_ahead;
    fa.lazy_marks = c->plan.lazy_marks;
    fa.merge = c->plan.merge;
    fa.prefetchB = c->plan.prefetchB;
    fa.pfA = c->plan.pfA;
    fa.pfB = c->plan.pfB;
    {  // the next call in decode order is layer + 1 (wrapping: the next token's layer 0)
      const int nl = (layer + 1) % c->L;
      // default: one row pair per way when the set has at most 8 ways (interleaved A/B, warm:
      // Mixtral -0.57 us, 8x22B P = 4 / 8 slices -0.57 / -0.42; with Phi's 16 ways the 38 MB of
      // mostly unused rows cost +0.38 us); MOE_PREFETCH_NEXT=rows overrides (0 = off)
      const int rows = c->plan.next_rows >= 0 ? c->plan.next_rows : 0;
      const bool ok = rows > 0 && nl < c->Ncov && c->miss_mode != MOE_MISS_HOST_COMPUTE;
      fa.next_pool = ok ? c->pool + (long long)nl * c->M * c->slot_bytes : nullptr;
      fa.next_ways = c->M;
      fa.next_rows = rows;
    }
    {
      // default: one row pair per way of a set with at most 8 ways, issued by each CTA before
      // its PDL wait (the bytes land while the previous call drains and this one routes)
      const int rows = c->plan.start_rows >= 0 ? c->plan.start_rows : (c->M <= 8 ? 1 : 0);
      const bool ok = rows > 0 && layer < c->Ncov && c->miss_mode != MOE_MISS_HOST_COMPUTE;
      fa.cur_pool = ok ? c->pool + (long long)layer * c->M * c->slot_bytes : nullptr;
      fa.cur_ways = c->M;
      fa.start_rows = rows;
      fa.pfx = c->plan.pfx;
    }
    fa.hoff = c->plan.hoff;
    fa.hstride = c->plan.hstride;
    fa.dbg = c->d_dbg;
    fa.dbg_stale = c->dbg_stale;
    fa.ts = c->d_ts;
    fa.ev = c->d_ev;
    fa.sts = ra.sts;
    fa.tpP = tpf ? c->P : ll1 ? 1 : 0;
    fa.tp_rank = tpf ? c->rank : 0;
    fa.tp_calls = tpf ? c->tp_calls : c->ll_calls;
    for (int p = 0; p < 8; ++p) fa.peer[p] = tpf && p < c->P ? c->tp_peer[p] : nullptr;
    if (ll1) fa.peer[0] = c->d_ll1;
    fa.yout = yhost ? yhost : y;
    fa.xhost = xhost;
    fa.xflag = c->d_xflag;
    fa.xseq = xhost ? ++c->xseq : 0u;
    fa.donef = donetag ? c->d_done : nullptr;
    fa.donetag = donetag;
    prof_begin(c, 1, s, &pe);
    TlRec tr;
    tl_begin(c, TL_KERNEL, seq, 0, s, &tr);
    cudaError_t e = launch_expert_fused(fa, c->plan, c->fused_grid, s, c->pdl, c->coop);
    if (e != cudaSuccess && c->pdl) {  // PDL not accepted: retry without it
      cudaGetLastError();
      c->pdl = false;
      e = launch_expert_fused(fa, c->plan, c->fused_grid, s, false, c->coop);
    }
    tl_end(c, s, &tr);
    prof_end(c, s, &pe);
    if (e != cudaSuccess) return fail(MOE_ERR_CUDA, std::string("expert_fused launch: ") + cudaGetErrorString(e));
    c->fused_calls += 1;
    if (tpf) c->tp_calls += 1;
    if (ll1) c->ll_calls += 1;
    c->issued.store(seq, std::memory_order_release);  // the fetch thread may now wait for it
  } else {
    prof_begin(c, 0, s, &pe);
    CUDA_TRY(launch_route_probe(ra, s, c->pdl));
    prof_end(c, s, &pe);
    c->issued.store(seq, std::memory_order_release);
    if (c->miss_mode == MOE_MISS_PULL) {  // missed experts: host store -> slots, by the SMs
      PullJob j{};
      j.count = &c->d_route->K;
      j.expert = c->d_route->expert;
      j.slot = c->d_route->slot;
      j.gen = c->d_route->gen;
      j.flag = c->d_route->wait;
      j.hblob = ra.hblob;
      j.pool = c->pool;
      j.slot_bytes = c->slot_bytes;
      j.ready = c->d_ready;
      j.done = c->d_pull_done;
      CUDA_TRY(launch_pull(j, c->num_sms, s));
    }
    prof_begin(c, 1, s, &pe);
    launch_expert_gateup(ea, s, c->num_sms);
    prof_end(c, s, &pe);
    prof_begin(c, 2, s, &pe);
    launch_expert_down(ea, s, c->num_sms);
    prof_end(c, s, &pe);
    CUDA_TRY(cudaGetLastError());
  }
  c->tokens[layer] += 1;
  c->trace_count += c->K;
  if (c->P > 1 && !tpf) {
    prof_begin(c, 3, s, &pe);
    ncclResult_t r = g_nccl.AllReduce(y, y, (size_t)c->d, ncclFloat32, ncclSum, c->comm, s);
    prof_end(c, s, &pe);
    if (r != ncclSuccess) return fail(MOE_ERR_NCCL, "ncclAllReduce failed");
  }
  CUDA_TRY(cudaEventRecord(c->done_ev, s));
  c->any_call = true;
  return MOE_OK;
}

MOE_API moe_status moe_layer_forward(moe_ctx* c, int32_t layer, const void* x, float* y, void* stream) {
  if (!c) return fail(MOE_ERR_INVALID_ARG, "NULL ctx");
  DeviceGuard g(c->device);
  nvtxRangePushA("moe_layer_forward");
  const moe_status st = forward_impl(c, layer, x, y, (cudaStream_t)stream);
  nvtxRangePop();
  return st;
}

// Debug only (not in moe.h): the stream timeline recorded since the last read
// (MOE_STREAM_TIMELINE=1). out: [cap][5] doubles {kind (0 kernel on the caller's stream,
// 1 weight copy on the fetch stream, 2 host-result copy on the activation stream), call seq,
// start ms, end ms (relative to the context's base event), bytes}. Synchronizes. Returns the
// number of records written (and clears them), or -1.
MOE_API int64_t moe_debug_stream_timeline(moe_ctx* c, double* out, int64_t cap) {
  if (!c || !c->tl || (cap > 0 && !out)) return -1;
  DeviceGuard g(c->device);
  if (drain(c) != MOE_OK) return -1;
  std::lock_guard<std::mutex> lk(c->tl_mu);
  int64_t n = 0;
  for (auto& r : c->tl_recs) {
    float t0 = 0.f, t1 = 0.f;
    if (n < cap && cudaEventElapsedTime(&t0, c->tl_base, r.a) == cudaSuccess &&
        cudaEventElapsedTime(&t1, c->tl_base, r.b) == cudaSuccess) {
      out[5 * n + 0] = r.kind;
      out[5 * n + 1] = (double)r.seq;
      out[5 * n + 2] = t0;
      out[5 * n + 3] = t1;
      out[5 * n + 4] = (double)r.bytes;
      ++n;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  cudaGetLastError();
  c->tl_recs.clear();
  return n;
}

// m-tiles per CTA tile of the prefill GEMMs: 0 = chosen on the device from the exact tile
// counts (prefill_gemm.cu); MOE_PREFILL_MT=1|2 forces one variant (A/B runs).
static int prefill_mt() {
  const char* e = getenv("MOE_PREFILL_MT");  // (read per call: prefill calls are few and large)
  const int v = e ? atoi(e) : 0;
  return v == 1 || v == 2 ? v : 0;
}

MOE_API moe_status moe_layer_prefill(moe_ctx* c, int32_t layer, const void* x, float* y, int32_t T, void* stream) {
  if (!c) return fail(MOE_ERR_INVALID_ARG, "NULL ctx");
  if (!c->configured) return fail(MOE_ERR_STATE, "cache_configure() has not been called");
  if (layer < 0 || layer >= c->L) return fail(MOE_ERR_INVALID_ARG, "layer out of range");
  if (!x || !y || T < 1) return fail(MOE_ERR_INVALID_ARG, "bad x / y / T");
  if (((uintptr_t)x & 15) || ((uintptr_t)y & 15)) return fail(MOE_ERR_INVALID_ARG, "x and y must be 16-byte aligned");
  if (layer >= c->Ncov || c->miss_mode == MOE_MISS_HOST_COMPUTE || c->K > 2 || c->d % 64 || c->ffr % 128 ||
      c->policy == MOE_POLICY_STATIC_RANDOM)
    return fail(MOE_ERR_UNSUPPORTED,
                "prefill needs a covered layer, MOE_MISS_FETCH or PULL, LRU/FIFO, K <= 2, d % 64 == 0, "
                "(ff/P) % 128 == 0");
  if (c->P > 1 && !c->comm)
    return fail(MOE_ERR_UNSUPPORTED, "prefill with tp_size > 1 reduces y with NCCL: create the ctx with nccl_unique_id");
  if (c->fetch_error.load()) return fail(MOE_ERR_CUDA, c->fetch_error_msg);
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  // ---- buffers (grow on demand) and tensor maps
  const int rows_cap = ((T * c->K + c->n * 128 + 127) / 128) * 128;
  if (T > c->pf_T || rows_cap > c->pf_rows) {
    CUDA_TRY(cudaDeviceSynchronize());
    cudaFree(c->d_rt_e); cudaFree(c->d_rt_w); cudaFree(c->d_tok); cudaFree(c->d_wrow);
    cudaFree(c->d_xg); cudaFree(c->d_hg);
    c->d_rt_e = nullptr; c->d_rt_w = nullptr; c->d_tok = nullptr; c->d_wrow = nullptr;
    c->d_xg = nullptr; c->d_hg = nullptr;
    c->pf_T = 0; c->pf_rows = 0;
    if (!c->d_pfscratch) CUDA_TRY(cudaMalloc(&c->d_pfscratch, prefill_scratch_bytes()));
    CUDA_TRY(cudaMalloc(&c->d_rt_e, sizeof(int) * (size_t)T * c->K));
    CUDA_TRY(cudaMalloc(&c->d_rt_w, sizeof(float) * (size_t)T * c->K));
    CUDA_TRY(cudaMalloc(&c->d_tok, sizeof(int) * (size_t)rows_cap));
    CUDA_TRY(cudaMalloc(&c->d_wrow, sizeof(float) * (size_t)rows_cap));
    CUDA_TRY(cudaMalloc(&c->d_xg, sizeof(uint16_t) * (size_t)rows_cap * c->d));
    CUDA_TRY(cudaMalloc(&c->d_hg, sizeof(uint16_t) * (size_t)rows_cap * c->ffr));
    if (!c->d_plan) CUDA_TRY(cudaMalloc(&c->d_plan, sizeof(PrefillPlan)));
    PrefillPlan hp;
    memset(&hp, 0, sizeof(hp));
    hp.tok = c->d_tok;
    hp.wrow = c->d_wrow;
    CUDA_TRY(cudaMemcpy(c->d_plan, &hp, sizeof(hp), cudaMemcpyHostToDevice));
    if (!encode_map_2d(&c->map_xg, c->d_xg, c->d, rows_cap, (uint64_t)c->d * 2, 128) ||
        !encode_map_2d(&c->map_hg, c->d_hg, c->ffr, rows_cap, (uint64_t)c->ffr * 2, 128))
      return fail(MOE_ERR_CUDA, "cuTensorMapEncodeTiled failed (prefill buffers)");
    c->pf_T = T;
    c->pf_rows = rows_cap;
  }
  const bool mn = c->M < c->n;  // evictions possible inside the prompt
  if (mn && (T > c->zbuf_T || c->pfstage_slots != c->n - c->M)) {
    CUDA_TRY(cudaDeviceSynchronize());
    if (T > c->zbuf_T) {
      cudaFree(c->d_zbuf);
      c->d_zbuf = nullptr;
      c->zbuf_T = 0;
      CUDA_TRY(cudaMalloc(&c->d_zbuf, sizeof(float) * (size_t)T * c->n));
      c->zbuf_T = T;
    }
    if (c->pfstage_slots != c->n - c->M) {
      cudaFree(c->d_pfstage);
      c->d_pfstage = nullptr;
      c->pfstage_slots = 0;
      const int ns = c->n - c->M;
      cudaError_t e = cudaMalloc(&c->d_pfstage, (size_t)ns * c->slot_bytes);
      if (e != cudaSuccess) {
        cudaGetLastError();
        c->d_pfstage = nullptr;
        return fail(MOE_ERR_OUT_OF_MEMORY, "prefill staging area (n - M slots) cudaMalloc failed");
      }
      if (!c->d_pfready) CUDA_TRY(cudaMalloc(&c->d_pfready, sizeof(uint32_t) * MOE_MAX_EXPERTS));
      CUDA_TRY(cudaMemset(c->d_pfready, 0, sizeof(uint32_t) * MOE_MAX_EXPERTS));
      const uint64_t st_elems = (uint64_t)ns * c->slot_bytes / 2;
      if (!encode_map_2d(&c->map_stage_d, c->d_pfstage, c->d, st_elems / c->d, (uint64_t)c->d * 2, 128) ||
          !encode_map_2d(&c->map_stage_f, c->d_pfstage, c->ffr, st_elems / c->ffr, (uint64_t)c->ffr * 2, 256) ||
          !encode_map_2d(&c->map_stage_f128, c->d_pfstage, c->ffr, st_elems / c->ffr, (uint64_t)c->ffr * 2, 128))
        return fail(MOE_ERR_CUDA, "cuTensorMapEncodeTiled failed (prefill staging area)");
      c->pfstage_slots = ns;
    }
  }
  if (!c->pool_maps) {
    const uint64_t pool_elems = (uint64_t)c->pool_bytes / 2;
    if (!encode_map_2d(&c->map_pool_d, c->pool, c->d, pool_elems / c->d, (uint64_t)c->d * 2, 128) ||
        !encode_map_2d(&c->map_pool_f, c->pool, c->ffr, pool_elems / c->ffr, (uint64_t)c->ffr * 2, 256) ||
        !encode_map_2d(&c->map_pool_f128, c->pool, c->ffr, pool_elems / c->ffr, (uint64_t)c->ffr * 2, 128))
      return fail(MOE_ERR_CUDA, "cuTensorMapEncodeTiled failed (slot pool)");
    c->pool_maps = true;
  }
  // host-side back-pressure on the miss mailbox (as in moe_layer_forward)
  const unsigned long long seq = c->issued.load() + 1;
  while (seq - c->consumed.load(std::memory_order_acquire) >= (unsigned long long)kMailRing - 1)
    std::this_thread::yield();
  // ---- router + cache pass (token order) + plan
  PrefillArgs pa;
  pa.T = T; pa.n = c->n; pa.K = c->K; pa.M = c->M; pa.layer = layer; pa.policy = c->policy;
  pa.miss_mode = c->miss_mode;
  pa.gw = gate_warps(c);
  pa.zbuf = mn ? c->d_zbuf : nullptr;
  pa.ready = c->d_ready;
  pa.staging_base = c->Ncov * c->M;
  pa.stage_slots = mn ? c->pfstage_slots : 0;
  pa.last_seq = c->d_last;
  pa.scratch = c->d_pfscratch;
  pa.tag = c->d_tag + (size_t)layer * c->M;
  pa.stamp = c->d_stamp + (size_t)layer * c->M;
  pa.slot_base = layer * c->M;
  pa.gen = c->d_gen;
  pa.clock = c->d_clock;
  pa.stats = c->d_stats + layer;
  pa.rt_e = c->d_rt_e;
  pa.rt_w = c->d_rt_w;
  pa.trace = c->d_trace;
  pa.trace_idx = c->trace_count;
  pa.trace_cap = c->trace_cap;
  pa.token0 = c->tokens[layer];
  pa.mail = c->d_mail + (seq % kMailRing);
  pa.seq = seq;
  pa.slot_bytes = c->slot_bytes;
  pa.plan = c->d_plan;
  CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(float) * (size_t)T * c->d, s));
  ProfEv pe;
  prof_begin(c, 0, s, &pe);
  CUDA_TRY(launch_prefill_route(pa, c->d_gate + (size_t)layer * c->n * c->d, (const uint16_t*)x, c->d, s));
  prof_end(c, s, &pe);
  c->issued.store(seq, std::memory_order_release);  // (the plan kernel publishes seq)
  c->tokens[layer] += (uint32_t)T;
  c->trace_count += (long long)T * c->K;
  if (c->miss_mode == MOE_MISS_PULL) {  // experts to fill: host store -> slots, by the SMs
    for (int stg = 0; stg < (mn ? 2 : 1); ++stg) {  // pool slots, then (M < n) staging slots
      PullJob j{};
      j.count = &c->d_plan->nblk;
      j.expert = c->d_plan->expert;
      j.slot = c->d_plan->slot;
      j.gen = c->d_plan->gen;
      j.flag = c->d_plan->wait;
      j.only = c->d_plan->stage;
      j.only_val = stg;
      j.hblob = c->d_hblob + (size_t)layer * c->n;
      j.pool = stg ? c->d_pfstage : c->pool;
      j.slot_bytes = c->slot_bytes;
      j.ready = stg ? c->d_pfready : c->d_ready;
      j.done = c->d_pull_done;
      CUDA_TRY(launch_pull(j, c->num_sms, s));
    }
  }
  CUDA_TRY(launch_prefill_gather((const uint16_t*)x, c->d, c->d_plan, c->d_xg, rows_cap, s));
  // ---- tensor-core expert FFN: GEMM1 (SwiGLU) then GEMM2 (down + combine)
  const int max_mtiles = rows_cap / 128;
  const int mt = prefill_mt();
  TcArgs ta;
  memset(&ta, 0, sizeof(ta));
  ta.d = c->d; ta.ffr = c->ffr; ta.ldh = c->ffr;
  ta.num_sms = c->num_sms;
  ta.plan = c->d_plan;
  ta.ready = c->d_ready;
  ta.mode = TC_MODE_SWIGLU;
  ta.mapA = c->map_xg;
  ta.mapB = c->map_pool_d;
  ta.has_stage = mn ? 1 : 0;
  ta.mapB2 = c->map_stage_d;
  ta.ready2 = c->d_pfready;
  ta.N = c->ffr; ta.K = c->d;
  ta.H = reinterpret_cast<__nv_bfloat16*>(c->d_hg);
  prof_begin(c, 1, s, &pe);
  CUDA_TRY(launch_tc_swiglu(ta, max_mtiles, mt, s));
  prof_end(c, s, &pe);
  ta.mode = TC_MODE_DOWN;
  ta.mapA = c->map_hg;
  ta.mapB = c->map_pool_f;
  ta.mapB2 = c->map_stage_f;
  ta.mapBp = c->map_pool_f128;
  ta.mapB2p = c->map_stage_f128;
  ta.has_pair_maps = 1;
  ta.N = c->d; ta.K = c->ffr;
  ta.y = y;
  prof_begin(c, 2, s, &pe);
  CUDA_TRY(launch_tc_down(ta, max_mtiles, mt, s));
  prof_end(c, s, &pe);
  if (c->P > 1) {
    prof_begin(c, 3, s, &pe);
    ncclResult_t r = g_nccl.AllReduce(y, y, (size_t)T * c->d, ncclFloat32, ncclSum, c->comm, s);
    prof_end(c, s, &pe);
    if (r != ncclSuccess) return fail(MOE_ERR_NCCL, "ncclAllReduce failed");
  }
  CUDA_TRY(cudaEventRecord(c->done_ev, s));
  c->any_call = true;
  return MOE_OK;
}

MOE_API moe_status moe_layer_forward_host(moe_ctx* c, int32_t layer, const uint16_t* x_host, float* y_host) {
  if (!c || !x_host || !y_host) return fail(MOE_ERR_INVALID_ARG, "NULL argument");
  if (!c->configured) return fail(MOE_ERR_STATE, "cache_configure() has not been called");
  if (layer < 0 || layer >= c->L) return fail(MOE_ERR_INVALID_ARG, "layer out of range");
  DeviceGuard g(c->device);
  cudaStream_t s = c->own_stream;
  moe_status st;
  // Zero-copy (fused path, pinned host buffers): the kernel reads x from the host buffer and
  // writes y straight into it — no copy-engine transfer queued in front of or behind it.
  void* xd = nullptr;
  void* yd = nullptr;
  // host -> device pointer of a pinned buffer: a driver call per pointer the first time, then
  // from a small direct-mapped cache (decode calls cycle over a few buffers). Only identity
  // mappings are cached (pinned memory under unified addressing, where the device pointer is
  // the host pointer whatever allocation later reuses the address); others ask every call.
  auto devptr = [&](const void* h, void** out) -> bool {
    const size_t slot = ((uintptr_t)h >> 4) % moe_ctx::kDevPtrCache;
    if (c->dp_host[slot] == h) {
      *out = const_cast<void*>(h);
      return true;
    }
    if (cudaHostGetDevicePointer(out, (void*)h, 0) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (*out == h) c->dp_host[slot] = h;
    return true;
  };
  const bool zc = c->fused && (c->P == 1 || c->tp_fused) && devptr(x_host, &xd) && devptr(y_host, &yd) &&
                  c->d % 8 == 0 && ((uintptr_t)xd & 15) == 0 && ((uintptr_t)yd & 15) == 0;
  if (zc && !c->tp_fused && !c->d_ll1) {
    const long long bytes = tp_xchg_bytes(1, c->K, c->d);
    CUDA_TRY(cudaMalloc(&c->d_ll1, (size_t)bytes));
    CUDA_TRY(cudaMemset(c->d_ll1, 0, (size_t)bytes));
    if (!c->d_ypart) CUDA_TRY(cudaMalloc(&c->d_ypart, sizeof(float) * c->d));
    CUDA_TRY(cudaDeviceSynchronize());
  }
  // single-rank zero-copy: every CTA flags its slice of y in host memory; the host spins on
  // those words (no driver call in the loop) instead of on a CUDA event
  const bool flags = zc && !c->tp_fused && c->fused_grid <= 1024 && getenv("MOE_E2E_EVENT") == nullptr;
  if (flags && !c->h_done) {
    uint32_t* hd = nullptr;
    CUDA_TRY(cudaHostAlloc((void**)&hd, sizeof(uint32_t) * 1024, cudaHostAllocMapped));
    memset(hd, 0, sizeof(uint32_t) * 1024);
    c->h_done = hd;
    CUDA_TRY(cudaHostGetDevicePointer((void**)&c->d_done, hd, 0));
  }
  if (zc) {
    const uint32_t tag = flags ? ++c->done_tag : 0u;
    st = forward_impl(c, layer, c->d_x_e2e, c->d_y_e2e, s, (const uint16_t*)xd, (float*)yd, tag);
    if (st != MOE_OK) return st;
    if (flags) {
      const int G = c->fused_grid;
      const auto t0 = std::chrono::steady_clock::now();
      bool recorded = false;                 // (the event only for a call that takes > 2 s)
      for (int b = 0; b < G; ++b) {
        while (c->h_done[b] != tag) {
          // a kernel that failed never writes its flags: fall back to the event's verdict (an
          // event recorded now completes after the kernel, or reports its error)
          if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) {
            if (!recorded) {
              CUDA_TRY(cudaEventRecord(c->host_ev, s));
              recorded = true;
            }
            cudaError_t q = cudaEventQuery(c->host_ev);
            if (q != cudaErrorNotReady && c->h_done[b] != tag) {
              CUDA_TRY(q);
              return fail(MOE_ERR_CUDA, "forward_host: kernel completed without its completion flags");
            }
          }
        }
      }
      std::atomic_thread_fence(std::memory_order_acquire);
      return MOE_OK;
    }
  } else {
    CUDA_TRY(cudaMemcpyAsync(c->d_x_e2e, x_host, sizeof(uint16_t) * c->d, cudaMemcpyHostToDevice, s));
    st = forward_impl(c, layer, c->d_x_e2e, c->d_y_e2e, s);
    if (st != MOE_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(y_host, c->d_y_e2e, sizeof(float) * c->d, cudaMemcpyDeviceToHost, s));
  }
  // Latency-oriented wait (single-request decode): poll the completion event instead of a
  // blocking synchronize, whose OS wake-up costs ~10 us per call.
  CUDA_TRY(cudaEventRecord(c->host_ev, s));
  cudaError_t q;
  while ((q = cudaEventQuery(c->host_ev)) == cudaErrorNotReady) {
  }
  CUDA_TRY(q);
  return MOE_OK;
}

MOE_API moe_status cache_stats(moe_ctx* c, int32_t layer, moe_layer_stats* out) {
  if (!c || !out) return fail(MOE_ERR_INVALID_ARG, "NULL argument");
  if (!c->configured) return fail(MOE_ERR_STATE, "cache_configure() has not been called");
  if (layer < -1 || layer >= c->L) return fail(MOE_ERR_INVALID_ARG, "layer out of range");
  DeviceGuard g(c->device);
  moe_status st = drain(c);
  if (st != MOE_OK) return st;
  std::vector<DevStats> all(c->L);
  CUDA_TRY(cudaMemcpy(all.data(), c->d_stats, sizeof(DevStats) * c->L, cudaMemcpyDeviceToHost));
  DevStats acc;
  memset(&acc, 0, sizeof(acc));
  for (int l = 0; l < c->L; ++l) {
    if (layer >= 0 && l != layer) continue;
    const unsigned long long* src = (const unsigned long long*)&all[l];
    unsigned long long* dst = (unsigned long long*)&acc;
    for (size_t k = 0; k < sizeof(DevStats) / 8; ++k) dst[k] += src[k];
  }
  memcpy(out, &acc, sizeof(acc));
  return MOE_OK;
}

MOE_API moe_status cache_trace(moe_ctx* c, moe_access_record* host_out, int64_t cap, int64_t* n_out) {
  if (!c || (cap > 0 && !host_out) || cap < 0) return fail(MOE_ERR_INVALID_ARG, "bad argument");
  if (!c->configured) return fail(MOE_ERR_STATE, "cache_configure() has not been called");
  DeviceGuard g(c->device);
  moe_status st = drain(c);
  if (st != MOE_OK) return st;
  long long avail = c->trace_count < c->trace_cap ? c->trace_count : c->trace_cap;
  long long m = avail < cap ? avail : cap;
  if (m > 0)
    CUDA_TRY(cudaMemcpy(host_out, c->d_trace, sizeof(moe_access_record) * m, cudaMemcpyDeviceToHost));
  if (n_out) *n_out = c->trace_count;
  return MOE_OK;
}

MOE_API moe_status moe_get_runtime_info(moe_ctx* c, moe_runtime_info* out) {
  if (!c || !out) return fail(MOE_ERR_INVALID_ARG, "NULL argument");
  memset(out, 0, sizeof(*out));
  out->expert_path = c->fused ? 1 : 0;
  out->pdl = c->pdl ? 1 : 0;
  out->ring_stages = c->fused ? c->plan.NS : 0;
  out->stage_bytes = c->fused ? c->plan.SB : 0;
  out->grid = c->fused ? c->fused_grid : 0;
  out->tp_reduce = c->P == 1 ? 0 : (c->tp_fused && c->fused) ? 2 : c->comm ? 1 : 0;
  return MOE_OK;
}

// ------------------------------------------------------------ fused TP reduction (f3)
static moe_status tp_ensure_buffer(moe_ctx* c) {
  if (c->d_xchg) return MOE_OK;
  const long long bytes = tp_xchg_bytes(c->P, c->K, c->d);
  cudaError_t e = cudaMalloc(&c->d_xchg, (size_t)bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_ypart, sizeof(float) * c->d);
  if (e == cudaSuccess) e = cudaMemset(c->d_xchg, 0, (size_t)bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaFree(c->d_xchg);
    cudaFree(c->d_ypart);
    c->d_xchg = nullptr;
    c->d_ypart = nullptr;
    return fail(e == cudaErrorMemoryAllocation ? MOE_ERR_OUT_OF_MEMORY : MOE_ERR_CUDA,
                std::string("exchange buffer: ") + cudaGetErrorString(e));
  }
  return MOE_OK;
}

static moe_status tp_check(moe_ctx* c) {
  if (c->P == 1) return fail(MOE_ERR_STATE, "tp_size == 1: nothing to reduce");
  if (!c->fused) return fail(MOE_ERR_UNSUPPORTED, "the fused TP reduction needs the fused decode kernel (K <= 2)");
  return MOE_OK;
}

// Zero this rank's counters and restart its call count: every rank must connect before any
// rank's first call (multi-process: a barrier after moe_tp_connect_ipc).
static moe_status tp_reset(moe_ctx* c) {
  moe_status st = drain(c);
  if (st != MOE_OK) return st;
  // all of it: a slot word left by an earlier connection could carry a tag this one reuses
  CUDA_TRY(cudaMemset(c->d_xchg, 0, (size_t)tp_xchg_bytes(c->P, c->K, c->d)));
  // the fused kernel's monotonic per-call counters assume a fixed grid: restart them (the
  // grid may have changed in moe_tp_connect_local)
  CUDA_TRY(cudaMemset(c->d_bar, 0, sizeof(unsigned long long) * 16 * kMaxK));
  CUDA_TRY(cudaMemset(c->d_ctr, 0, sizeof(unsigned) * kCtrWords));
  CUDA_TRY(cudaMemset(c->d_hf, 0xff, sizeof(float) * 2 * (size_t)c->K * c->ffr));  // call parity restarts
  CUDA_TRY(cudaDeviceSynchronize());
  c->fused_calls = 0;
  c->tp_calls = 0;
  c->tp_fused = true;
  return MOE_OK;
}

MOE_API moe_status moe_tp_exchange_buffer(moe_ctx* c, moe_tp_exchange* out) {
  if (!c || !out) return fail(MOE_ERR_INVALID_ARG, "NULL argument");
  moe_status st = tp_check(c);
  if (st != MOE_OK) return st;
  DeviceGuard g(c->device);
  st = tp_ensure_buffer(c);
  if (st != MOE_OK) return st;
  memset(out, 0, sizeof(*out));
  out->dev_ptr = c->d_xchg;
  out->bytes = tp_xchg_bytes(c->P, c->K, c->d);
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "ipc handle size");
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->d_xchg));
  memcpy(out->ipc_handle, &h, 64);
  return MOE_OK;
}

MOE_API moe_status moe_tp_connect_ipc(moe_ctx* c, const uint8_t* handles) {
  if (!c || !handles) return fail(MOE_ERR_INVALID_ARG, "NULL argument");
  moe_status st = tp_check(c);
  if (st != MOE_OK) return st;
  DeviceGuard g(c->device);
  st = tp_ensure_buffer(c);
  if (st != MOE_OK) return st;
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  c->ipc_opened.clear();
  c->tp_fused = false;
  for (int p = 0; p < c->P; ++p) {
    if (p == c->rank) {
      c->tp_peer[p] = c->d_xchg;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + 64 * p, 64);
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      for (void* q : c->ipc_opened) cudaIpcCloseMemHandle(q);
      c->ipc_opened.clear();
      return fail(MOE_ERR_CUDA, "cudaIpcOpenMemHandle(rank " + std::to_string(p) + "): " + cudaGetErrorString(e));
    }
    c->ipc_opened.push_back(ptr);
    c->tp_peer[p] = (uint8_t*)ptr;
  }
  return tp_reset(c);
}

MOE_API moe_status moe_tp_disconnect(moe_ctx* c) {
  if (!c) return fail(MOE_ERR_INVALID_ARG, "NULL ctx");
  DeviceGuard g(c->device);
  moe_status st = drain(c);
  if (st != MOE_OK) return st;
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  c->ipc_opened.clear();
  for (auto& p : c->tp_peer) p = nullptr;
  c->tp_fused = false;
  return MOE_OK;
}

MOE_API moe_status moe_tp_connect_local(moe_ctx* const* ctxs, int32_t P) {
  if (!ctxs || P < 2 || P > 8) return fail(MOE_ERR_INVALID_ARG, "need 2 <= P <= 8 contexts");
  moe_ctx* by_rank[8] = {};
  for (int i = 0; i < P; ++i) {
    moe_ctx* c = ctxs[i];
    if (!c) return fail(MOE_ERR_INVALID_ARG, "NULL context");
    if (c->P != P) return fail(MOE_ERR_INVALID_ARG, "every context must have tp_size == P");
    if (by_rank[c->rank]) return fail(MOE_ERR_INVALID_ARG, "tp_rank must be a permutation of 0..P-1");
    by_rank[c->rank] = c;
    if (c->L != ctxs[0]->L || c->d != ctxs[0]->d || c->ff != ctxs[0]->ff || c->n != ctxs[0]->n ||
        c->K != ctxs[0]->K)
      return fail(MOE_ERR_INVALID_ARG, "contexts of one TP group must share the model shape");
    moe_status st = tp_check(c);
    if (st != MOE_OK) return st;
  }
  for (int r = 0; r < P; ++r) {
    DeviceGuard g(by_rank[r]->device);
    moe_status st = tp_ensure_buffer(by_rank[r]);
    if (st != MOE_OK) return st;
  }
  for (int r = 0; r < P; ++r) {
    moe_ctx* c = by_rank[r];
    DeviceGuard g(c->device);
    int same = 0;
    for (int q = 0; q < P; ++q) {
      moe_ctx* o = by_rank[q];
      c->tp_peer[q] = o->d_xchg;
      if (o->device == c->device) {
        ++same;
        continue;
      }
      int can = 0;
      CUDA_TRY(cudaDeviceCanAccessPeer(&can, c->device, o->device));
      if (!can) return fail(MOE_ERR_UNSUPPORTED, "no peer access between devices of the TP group");
      cudaError_t e = cudaDeviceEnablePeerAccess(o->device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return fail(MOE_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
    }
    if (same > 1) {
      // ranks sharing this GPU wait on each other inside their kernels: split the SMs so all
      // of their grids are co-resident, and launch each call only after the previous one of
      // the same rank has completed (no PDL early start, no cooperative launch)
      FusedPlan plan;
      const int grid = c->num_sms / same;
      if (!plan_fused(c->d, c->ffr, c->n, c->K, grid, &plan))
        return fail(MOE_ERR_UNSUPPORTED, "fused plan does not fit the per-rank grid");
      c->fused_grid = grid;
      c->pdl = false;
      c->coop = false;
    }
  }
  for (int r = 0; r < P; ++r) {
    DeviceGuard g(by_rank[r]->device);
    moe_status st = tp_reset(by_rank[r]);
    if (st != MOE_OK) return st;
  }
  return MOE_OK;
}

MOE_API moe_status moe_profile_enable(moe_ctx* c, int32_t enable) {
  if (!c) return fail(MOE_ERR_INVALID_ARG, "NULL ctx");
  c->prof = enable != 0;
  return MOE_OK;
}

MOE_API moe_status moe_profile_read(moe_ctx* c, moe_profile_t* out) {
  if (!c || !out) return fail(MOE_ERR_INVALID_ARG, "NULL argument");
  DeviceGuard g(c->device);
  for (auto& p : c->prof_events) {
    float ms = 0;
    CUDA_TRY(cudaEventSynchronize(p.b));
    CUDA_TRY(cudaEventElapsedTime(&ms, p.a, p.b));
    c->prof_ms[p.kind] += ms;
    c->prof_launches[p.kind] += 1;
    c->ev_free.push_back(p.a);
    c->ev_free.push_back(p.b);
  }
  c->prof_events.clear();
  for (int k = 0; k < MOE_PROF_KINDS; ++k) {
    out->ms[k] = c->prof_ms[k];
    out->launches[k] = c->prof_launches[k];
    c->prof_ms[k] = 0;
    c->prof_launches[k] = 0;
  }
  return MOE_OK;
}

}  // extern "C"
