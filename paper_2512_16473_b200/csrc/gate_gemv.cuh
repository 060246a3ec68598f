// gate_gemv.cuh — the ONE summation order of the router's gate logits z_e = sum_i Wg[e,i] x_i
// (P:44), shared by every kernel that computes them: the fused decode kernel
// (expert_fused.cu), the split-path router (route_probe.cu) and the prefill router
// (prefill.cu). moe.h promises that a prefill of T tokens routes exactly like T decode
// calls; near-tied logits make that a statement about rounding, so every path sums the same
// products in the same order (DESIGN R25):
//
//   W "virtual warps" of 32 lanes (V = 32 W virtual lanes; W = the fused plan's consumer
//   warps, 2 * NS, or kGateWarpsDefault without a fused plan). With x and Wg[e] read as
//   16-B chunks of 8 bf16 (nch = d / 8 chunks):
//   1. lane v accumulates two fp32 sums from 0, over chunks ch = v, v + V, v + 2V, ...:
//        for k = 0..3:  s_even = fma(w[2k], x[2k], s_even);  s_odd = fma(w[2k+1], x[2k+1], s_odd)
//      (bf16 x bf16 products are exact in fp32, so every fma rounds once), p_v = s_even + s_odd;
//   2. per virtual warp: butterfly over its 32 lanes, xor 16, 8, 4, 2, 1 (s += partner);
//   3. z_e = ((0 + zw_0) + zw_1) + ... + zw_{W-1}, in virtual-warp order.
// The fused kernel runs it with one real consumer warp per virtual warp (mixed-precision
// FHFMA.BF16 and a warp reduce-scatter that evaluates the same butterfly tree per expert);
// the other kernels emulate the W virtual warps with whatever warps they have.
//
// Tensor-core form (gate_mma_form: 9-16 experts, d a multiple of 16), replacing steps 1-2:
// virtual warp vw runs one mma.sync m16n8k16 (bf16 x bf16 -> fp32, legacy HMMA) per k-block
// kb = vw, vw + W, vw + 2W, ... < d / 16 into one accumulator from 0, A = the gate rows
// (row e = expert e, rows >= n zero or ignored), x in every column of B, and takes column 0
// (the same instruction sequence on the same values in every kernel: the same bits). Step 3 is
// unchanged. 16 gate rows x 4096 with 20 warps: ~2100 cycles against ~3100 for the FHFMA
// form (tools/gate_mma_rate.cu); with 8 rows half of every MMA is wasted and it is slower.
#pragma once
#include <stdint.h>

namespace moe {

constexpr int kGateWarpsDefault = 20;
constexpr int kGateWarpsMax = 32;

__device__ __forceinline__ float gate_bf_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float gate_bf_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// step 1 for one virtual lane: returns s_even + s_odd
__device__ __forceinline__ float gate_lane_partial(const int4* __restrict__ w, const int4* __restrict__ x, int v, int V,
                                                   int nch) {
  float se = 0.f, so = 0.f;
  for (int ch = v; ch < nch; ch += V) {
    const int4 a = w[ch], b = x[ch];
    se = fmaf(gate_bf_lo(a.x), gate_bf_lo(b.x), se);
    so = fmaf(gate_bf_hi(a.x), gate_bf_hi(b.x), so);
    se = fmaf(gate_bf_lo(a.y), gate_bf_lo(b.y), se);
    so = fmaf(gate_bf_hi(a.y), gate_bf_hi(b.y), so);
    se = fmaf(gate_bf_lo(a.z), gate_bf_lo(b.z), se);
    so = fmaf(gate_bf_hi(a.z), gate_bf_hi(b.z), so);
    se = fmaf(gate_bf_lo(a.w), gate_bf_lo(b.w), se);
    so = fmaf(gate_bf_hi(a.w), gate_bf_hi(b.w), so);
  }
  return se + so;
}

__host__ __device__ constexpr bool gate_mma_form(int n, int d) { return n > 8 && n <= 16 && (d & 15) == 0; }

// Tensor-core form, one virtual warp vw of W: lane (g = lane / 4, c = lane % 4) passes
// r0 = row g + 4c bytes, r1 = row g + 8 (any row when g + 8 >= n) + 4c, xp = x + 4c; nkb = d / 16.
// Returns (z_part of row g, z_part of row g + 8) in lanes with c == 0.
__device__ __forceinline__ float2 gate_mma_warp(const uint8_t* r0, const uint8_t* r1, const uint8_t* xp, int nkb, int vw,
                                                int W) {
  float c[4] = {0.f, 0.f, 0.f, 0.f};
  for (int kb = vw; kb < nkb; kb += W) {
    const int o = kb * 32;
    const uint32_t a0 = *reinterpret_cast<const uint32_t*>(r0 + o);
    const uint32_t a2 = *reinterpret_cast<const uint32_t*>(r0 + o + 16);
    const uint32_t a1 = *reinterpret_cast<const uint32_t*>(r1 + o);
    const uint32_t a3 = *reinterpret_cast<const uint32_t*>(r1 + o + 16);
    const uint32_t b0 = *reinterpret_cast<const uint32_t*>(xp + o);
    const uint32_t b1 = *reinterpret_cast<const uint32_t*>(xp + o + 16);
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  return make_float2(c[0], c[2]);
}

// step 2: butterfly over the (real) warp's 32 lanes; every lane returns the same value
__device__ __forceinline__ float gate_butterfly(float s) {
  s += __shfl_xor_sync(0xffffffffu, s, 16);
  s += __shfl_xor_sync(0xffffffffu, s, 8);
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}

// step 3: zw[w * stride] for w = 0 .. W-1, summed in order (loads issued up front)
__device__ __forceinline__ float gate_sum_warps(const float* zw, int stride, int W) {
  float p[kGateWarpsMax];
#pragma unroll
  for (int w = 0; w < kGateWarpsMax; ++w) p[w] = w < W ? zw[w * stride] : 0.f;
  float z = 0.f;
#pragma unroll
  for (int w = 0; w < kGateWarpsMax; ++w)
    if (w < W) z += p[w];
  return z;
}

// Steps 1-2 for n experts and the virtual warps vw = vw0, vw0 + step, ... < W, by one real
// warp: zpart[vw * n + e] = butterfly of virtual warp vw for expert e. x chunks are reused
// across the experts. Wg: [n][d] rows; x: [d].
__device__ __forceinline__ void gate_virtual_warps(const uint16_t* __restrict__ Wg, const uint16_t* __restrict__ x,
                                                   int d, int n, int W, int vw0, int step, float* zpart) {
  const int lane = threadIdx.x & 31;
  if (gate_mma_form(n, d)) {
    const int g = lane >> 2, c4 = lane & 3;
    const bool hi = g + 8 < n;
    const uint8_t* r0 = reinterpret_cast<const uint8_t*>(Wg + (size_t)g * d) + 4 * c4;
    const uint8_t* r1 = reinterpret_cast<const uint8_t*>(Wg + (size_t)(hi ? g + 8 : g) * d) + 4 * c4;
    const uint8_t* xp = reinterpret_cast<const uint8_t*>(x) + 4 * c4;
    for (int vw = vw0; vw < W; vw += step) {
      const float2 z = gate_mma_warp(r0, r1, xp, d >> 4, vw, W);
      if (c4 == 0) {
        zpart[vw * n + g] = z.x;
        if (hi) zpart[vw * n + g + 8] = z.y;
      }
    }
    return;
  }
  const int nch = d >> 3, V = 32 * W;
  const int4* xq = reinterpret_cast<const int4*>(x);
  for (int vw = vw0; vw < W; vw += step) {
    const int v = 32 * vw + lane;
    for (int e = 0; e < n; ++e) {
      const float p = gate_lane_partial(reinterpret_cast<const int4*>(Wg + (size_t)e * d), xq, v, V, nch);
      const float s = gate_butterfly(p);
      if (lane == 0) zpart[vw * n + e] = s;
    }
  }
}

}  // namespace moe
