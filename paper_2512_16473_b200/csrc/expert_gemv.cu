// expert_gemv.cu — K2/K3: SwiGLU expert FFN GEMVs over cache-resident slots (sm_100a).
//
// Decode batch 1 makes every expert matrix a GEMV (~1 FLOP/B): the kernels are HBM
// bound, so they are written as streaming reductions on the CUDA cores — 16-byte
// L1-bypassing loads with deep per-lane unrolling (memory-level parallelism), fp32
// accumulation, warp-shuffle reductions. Tensor cores are not the roofline here.
//
//   K2 expert_gateup : h_r[j] = silu(W1_r[j,:] x) * (W3_r[j,:] x)        (R4)
//                      one warp per (expert r, row j); waits for the slots' fills.
//   K3 expert_down   : y[c] = sum_r w_r * (W2_r[c,:] h_r)
//                      one warp per output row c, rank-ordered combine.
// Slot layout (moe.h): { W1[ffr][d], W3[ffr][d], W2[d][ffr] } bf16.
#include <math.h>

#include "moe_internal.cuh"

namespace moe {
namespace {

__device__ __forceinline__ float bf_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// Streaming 16-byte load: read-only path, no L1 allocation, 256-B L2 prefetch.
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float dot8(const int4 w, const float4 a, const float4 b, float s) {
  s = fmaf(bf_lo(w.x), a.x, s);
  s = fmaf(bf_hi(w.x), a.y, s);
  s = fmaf(bf_lo(w.y), a.z, s);
  s = fmaf(bf_hi(w.y), a.w, s);
  s = fmaf(bf_lo(w.z), b.x, s);
  s = fmaf(bf_hi(w.z), b.y, s);
  s = fmaf(bf_lo(w.w), b.z, s);
  s = fmaf(bf_hi(w.w), b.w, s);
  return s;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Spin until the slot's fill generation has landed (hit: immediate; miss / hit-under-
// fill: the fetch stream publishes it after the H2D copy). 60 s timeout -> trap.
__device__ void wait_ready(const uint32_t* ready, int slot, uint32_t gen) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 64;
  while (true) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + slot) : "memory");
    if (v >= gen) break;
    __nanosleep(ns);
    if (ns < 4096) ns <<= 1;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 60ull * 1000000000ull) __trap();
  }
}

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnrollA = 8;  // 16 x 16-B loads in flight per lane in K2
constexpr int kUnrollB = 8;  // 8 x 16-B loads in flight per lane per expert in K3

__global__ void __launch_bounds__(kThreads) expert_gateup_kernel(const ExpertArgs a) {
  extern __shared__ float4 xs4[];  // x as fp32, d floats
  __shared__ const uint8_t* base[kMaxK];
  const int K = a.K, d = a.d, ffr = a.ffr;
  float* xs = reinterpret_cast<float*>(xs4);
  for (int i = threadIdx.x; i < d; i += kThreads) xs[i] = __uint_as_float((uint32_t)a.x[i] << 16);
  if (threadIdx.x < K) {
    const int slot = a.route->slot[threadIdx.x];
    wait_ready(a.ready, slot, a.route->gen[threadIdx.x]);
    base[threadIdx.x] = a.pool + (long long)slot * a.slot_bytes;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nchunk = d >> 3;
  const int rows = K * ffr;
  for (int q = blockIdx.x * kWarps + warp; q < rows; q += gridDim.x * kWarps) {
    const int r = q / ffr, j = q - r * ffr;
    const int4* w1 = reinterpret_cast<const int4*>(base[r]) + (long long)j * nchunk;
    const int4* w3 = w1 + (long long)ffr * nchunk;
    float g = 0.f, u = 0.f;
    for (int c0 = lane; c0 < nchunk; c0 += 32 * kUnrollA) {
      int4 wa[kUnrollA], wb[kUnrollA];
#pragma unroll
      for (int k = 0; k < kUnrollA; ++k) {
        const int c = c0 + 32 * k;
        if (c < nchunk) {
          wa[k] = ld_stream(w1 + c);
          wb[k] = ld_stream(w3 + c);
        }
      }
#pragma unroll
      for (int k = 0; k < kUnrollA; ++k) {
        const int c = c0 + 32 * k;
        if (c < nchunk) {
          const float4 x0 = xs4[2 * c], x1 = xs4[2 * c + 1];
          g = dot8(wa[k], x0, x1, g);
          u = dot8(wb[k], x0, x1, u);
        }
      }
    }
    g = warp_sum(g);
    u = warp_sum(u);
    if (lane == 0) a.h[q] = g / (1.0f + expf(-g)) * u;
  }
}

__global__ void __launch_bounds__(kThreads) expert_down_kernel(const ExpertArgs a) {
  __shared__ const uint8_t* base[kMaxK];
  __shared__ float wgt[kMaxK];
  const int K = a.K, d = a.d, ffr = a.ffr;
  if (threadIdx.x < K) {
    base[threadIdx.x] = a.pool + (long long)a.route->slot[threadIdx.x] * a.slot_bytes;
    wgt[threadIdx.x] = a.route->w[threadIdx.x];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nchunk = ffr >> 3;
  const long long w2off = 2ll * ffr * d * 2;  // bytes of W1 + W3
  for (int c = blockIdx.x * kWarps + warp; c < d; c += gridDim.x * kWarps) {
    float y = 0.f;
    for (int r = 0; r < K; ++r) {
      const int4* w2 = reinterpret_cast<const int4*>(base[r] + w2off) + (long long)c * nchunk;
      const float4* h4 = reinterpret_cast<const float4*>(a.h + (long long)r * ffr);
      float acc = 0.f;
      for (int c0 = lane; c0 < nchunk; c0 += 32 * kUnrollB) {
        int4 wv[kUnrollB];
#pragma unroll
        for (int k = 0; k < kUnrollB; ++k) {
          const int cc = c0 + 32 * k;
          if (cc < nchunk) wv[k] = ld_stream(w2 + cc);
        }
#pragma unroll
        for (int k = 0; k < kUnrollB; ++k) {
          const int cc = c0 + 32 * k;
          if (cc < nchunk) acc = dot8(wv[k], __ldg(h4 + 2 * cc), __ldg(h4 + 2 * cc + 1), acc);
        }
      }
      acc = warp_sum(acc);
      y = fmaf(wgt[r], acc, y);  // rank-ordered combine (fp32)
    }
    if (lane == 0) a.y[c] = y;
  }
}

}  // namespace

cudaError_t preload_expert_kernels() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, expert_gateup_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, expert_down_kernel);
  return e;
}

void launch_expert_gateup(const ExpertArgs& a, cudaStream_t s, int num_sms) {
  const int rows = a.K * a.ffr;
  int grid = (rows + kWarps - 1) / kWarps;
  if (grid > num_sms * 8) grid = num_sms * 8;
  expert_gateup_kernel<<<grid, kThreads, a.d * sizeof(float), s>>>(a);
}

void launch_expert_down(const ExpertArgs& a, cudaStream_t s, int num_sms) {
  int grid = (a.d + kWarps - 1) / kWarps;
  if (grid > num_sms * 8) grid = num_sms * 8;
  expert_down_kernel<<<grid, kThreads, 0, s>>>(a);
}

}  // namespace moe
