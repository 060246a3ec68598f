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
#include "ptx.cuh"
#include "route_core.cuh"

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
  // The set of this layer was last written by the router of an EARLIER call, which
  // completed before the previous expert kernels passed their own griddepcontrol.wait,
  // i.e. before this grid could launch: it can be read before this grid's wait, too.
  DirState ds;
  if (warp == 0) ds = dir_load(a, lane);
  griddep_launch_dependents();  // let the expert kernel's CTAs get resident early
  griddep_wait();               // x (written by the caller's previous kernel) is visible now
  const long long ck0 = clock64();
  if (a.sts && threadIdx.x == 0) a.sts[0] = ptx::globaltimer();
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
  if (a.sts && lane == 0) a.sts[2] = clock64() - ck0;
  float zsum = 0.f;
  if (lane < n)
    for (int q = 0; q < G; ++q) zsum += part[lane][q];  // fixed order: deterministic
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
