// route_probe.cu — K1: fused router + cache probe + on-device LRU update (sm_100a).
//
// Router of the split expert path (MOE_EXPERT_PATH=split, or shapes the fused kernel does
// not cover; the fused decode kernel evaluates the same decision itself). One CTA per
// call. Warps compute the gate GEMV z = Wg x (16-byte loads, fp32 accumulation,
// warp-shuffle reduction); warp 0 then takes the routing decision (route_core.cuh: top-K,
// softmax, cache probe, LRU/FIFO/static update, miss handling) and writes the route
// record for the expert kernels, the access trace, the per-layer counters and the miss
// mailbox (host-mapped; P:200's post-fetch is issued by the runtime's fetch thread from it).
#include <math.h>

#include "moe_internal.cuh"
#include "gate_gemv.cuh"
#include "ptx.cuh"
#include "route_core.cuh"

namespace moe {
namespace {

using ptx::griddep_launch_dependents;
using ptx::griddep_wait;

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;

__global__ void __launch_bounds__(kThreads) route_probe_kernel(const RouteArgs a) {
  __shared__ float zpart[kGateWarpsMax * MOE_MAX_EXPERTS];
  __shared__ int sS[kMaxK];
  __shared__ float sZ[kMaxK], sW[kMaxK];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = a.n;
  // The set of this layer was last written by the router of an EARLIER call, which
  // completed before the previous expert kernels passed their own griddepcontrol.wait,
  // i.e. before this grid could launch: it can be read before this grid's wait, too.
  // The gate rows do not depend on x either: pulled towards L2 before the wait.
  DirState ds;
  if (warp == 0) ds = dir_load(a, lane);
  for (int i = threadIdx.x; i < (n * a.d) >> 6; i += kThreads)  // one 128-B line per thread and step
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a.Wg + (size_t)i * 64));
  griddep_launch_dependents();  // let the expert kernel's CTAs get resident early
  griddep_wait();               // x (written by the caller's previous kernel) is visible now
  const long long ck0 = clock64();
  if (a.sts && threadIdx.x == 0) a.sts[0] = ptx::globaltimer();
  // ---- gate GEMV z = Wg x in the shared summation order (gate_gemv.cuh): real warp w
  // evaluates virtual warp w (a.gw <= 32 virtual warps), warp 0 sums them in order
  gate_virtual_warps(a.Wg, a.x, a.d, n, a.gw, warp, kWarps, zpart);
  __syncthreads();
  if (warp != 0) return;
  if (a.sts && lane == 0) a.sts[2] = clock64() - ck0;
  const float zsum = lane < n ? gate_sum_warps(zpart + lane, n, a.gw) : 0.f;
  LaneRoute lr;
  const int nmiss = route_decide(a, zsum, ds, true, sS, sZ, sW, &lr);
  if (a.sts && lane == 0) a.sts[4] = clock64() - ck0;
  if (lane < a.K) {
    a.route->expert[lane] = lr.expert;
    a.route->w[lane] = lr.w;
    a.route->slot[lane] = lr.slot;
    a.route->gen[lane] = lr.gen;
    a.route->wait[lane] = lr.wait;
    a.route->host[lane] = lr.host;
  }
  if (lane == 0) a.route->K = a.K;
  __syncwarp();
  if (a.sts && lane == 0) {
    a.sts[1] = ptx::globaltimer();
    a.sts[5] = clock64() - ck0;
  }
  // miss mailbox entry (host-mapped; FETCH / HOST_COMPUTE misses) and the progress word
  if (lane == 0) publish_progress(a, nmiss);
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
