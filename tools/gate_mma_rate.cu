// Gate GEMV z = Wg x on one SM, whole prologue step (per-warp partials + the in-order
// cross-warp sum), in cycles, for the decode kernel's routing: 20 consumer warps, n gate
// rows x d bf16 in shared memory at the kernel's padded stride (2d + 16 B), x in shared memory.
//   mode 0  the kernel's FHFMA.BF16 form (16-B chunks per thread, warp reduce-scatter)
//   mode 1  mma.sync m16n8k16 bf16 -> fp32 (legacy HMMA), warp w takes k-blocks w, w + 20, ...,
//           A fragments by 32-bit shared loads, B = x in every column
//   mode 2  as 1 with two accumulators (even / odd k-blocks of the warp) summed at the end
//   mode 3  (8 experts) paired k-blocks: rows 0-7 = the experts at the warp's k-block 2i,
//           rows 8-15 = the same experts at k-block 2i + 1, B column 0 / 1 = x at those
//           k-blocks; z = D[e][0] + D[e + 8][1]: every MMA does 16 useful rows
//   mode 4  as 1 with the k index permuted inside each block of 16 (MMA k-pair 2c <-> columns
//           4c, 4c+1, k-pair 2c+8 <-> 4c+2, 4c+3): A and B fragments by 64-bit shared loads,
//           3 loads per MMA instead of 6 (same sum, another order)
// Prints the median CTA's cycles and the max relative error against an fp64 host GEMV.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gate_mma_rate tools/gate_mma_rate.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <vector>
#include <algorithm>

constexpr int W = 20, T = 32 * W;

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
__device__ __forceinline__ float2 dot8_bf(const int4 w, const int4 x, float2 acc) {
  acc = fma_bf16x2((uint32_t)w.x, (uint32_t)x.x, acc);
  acc = fma_bf16x2((uint32_t)w.y, (uint32_t)x.y, acc);
  acc = fma_bf16x2((uint32_t)w.z, (uint32_t)x.z, acc);
  acc = fma_bf16x2((uint32_t)w.w, (uint32_t)x.w, acc);
  return acc;
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int MODE>
__global__ void __launch_bounds__(T, 1) gemv(const uint16_t* Wg, const uint16_t* x, int d, int n, float* out,
                                             long long* cyc) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int gstride = 2 * d + 16;
  uint8_t* xs = sm + (size_t)16 * gstride;
  float* zpart = reinterpret_cast<float*>(xs + 2 * d);
  for (int i = threadIdx.x; i < 16 * (gstride / 4); i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < n * (d / 8); i += blockDim.x) {
    const int e = i / (d / 8), c = i % (d / 8);
    reinterpret_cast<int4*>(sm + (size_t)e * gstride)[c] = reinterpret_cast<const int4*>(Wg + (size_t)e * d)[c];
  }
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) reinterpret_cast<int4*>(xs)[i] = reinterpret_cast<const int4*>(x)[i];
  __syncthreads();
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  float z = 0.f;
  long long c0 = 0;
  for (int rep = 0; rep < 17; ++rep) {
    if (rep == 1) c0 = clock64();
    if (MODE == 0) {
      const int nch = d >> 3;
      const int4* xq = reinterpret_cast<const int4*>(xs);
      for (int e0 = 0; e0 < n; e0 += 8) {
        float2 acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = make_float2(0.f, 0.f);
        for (int ch = t; ch < nch; ch += T) {
          const int4 xv = xq[ch];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (e0 + j < n) acc[j] = dot8_bf(reinterpret_cast<const int4*>(sm + (size_t)(e0 + j) * gstride)[ch], xv, acc[j]);
        }
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = acc[j].x + acc[j].y;
        const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
        float w4[4], w2[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) w4[i] = (b4 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, b4 ? v[i] : v[i + 4], 16);
#pragma unroll
        for (int i = 0; i < 2; ++i) w2[i] = (b3 ? w4[i + 2] : w4[i]) + __shfl_xor_sync(0xffffffffu, b3 ? w4[i] : w4[i + 2], 8);
        float zz = (b2 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? w2[0] : w2[1], 4);
        zz += __shfl_xor_sync(0xffffffffu, zz, 2);
        zz += __shfl_xor_sync(0xffffffffu, zz, 1);
        const int e = e0 + (b4 ? 4 : 0) + (b3 ? 2 : 0) + (b2 ? 1 : 0);
        if ((lane & 3) == 0 && e < n) zpart[warp * 16 + e] = zz;
      }
    } else if (MODE == 4) {
      const int g = lane >> 2, c = lane & 3;
      const uint8_t* r0 = sm + (size_t)g * gstride + 8 * c;
      const uint8_t* r1 = sm + (size_t)(g + 8) * gstride + 8 * c;
      const uint8_t* xp = xs + 8 * c;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const int nkb = d >> 4;
      for (int kb = warp; kb < nkb; kb += W) {
        const int o = kb * 32;
        const uint2 a02 = *reinterpret_cast<const uint2*>(r0 + o);
        const uint2 a13 = n > 8 ? *reinterpret_cast<const uint2*>(r1 + o) : make_uint2(0u, 0u);
        const uint2 b01 = *reinterpret_cast<const uint2*>(xp + o);
        mma16816(acc, a02.x, a13.x, a02.y, a13.y, b01.x, b01.y);
      }
      if (c == 0) {
        zpart[warp * 16 + g] = acc[0];
        if (g + 8 < n) zpart[warp * 16 + g + 8] = acc[2];
      }
    } else if (MODE == 3) {
      const int g = lane >> 2, c = lane & 3;
      const uint8_t* r0 = sm + (size_t)g * gstride + 4 * c;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const int nkb = d >> 4;
      for (int kb = warp; kb < nkb; kb += 2 * W) {
        const int kb2 = kb + W;
        const bool two = kb2 < nkb;
        const int o = kb * 32, o2 = (two ? kb2 : kb) * 32;
        const uint32_t a0 = *reinterpret_cast<const uint32_t*>(r0 + o);
        const uint32_t a2 = *reinterpret_cast<const uint32_t*>(r0 + o + 16);
        const uint32_t a1 = two ? *reinterpret_cast<const uint32_t*>(r0 + o2) : 0u;
        const uint32_t a3 = two ? *reinterpret_cast<const uint32_t*>(r0 + o2 + 16) : 0u;
        const int ob = g == 1 ? o2 : o;
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(xs + 4 * c + ob);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(xs + 4 * c + ob + 16);
        mma16816(acc, a0, a1, a2, a3, b0, b1);
      }
      if (c == 0) zpart[warp * 16 + g] = acc[0] + acc[3];
    } else {
      const int g = lane >> 2, c = lane & 3;
      const uint8_t* r0 = sm + (size_t)g * gstride + 4 * c;
      const uint8_t* r1 = sm + (size_t)(g + 8) * gstride + 4 * c;
      const uint8_t* xp = xs + 4 * c;
      float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      const int nkb = d >> 4;
      int i = 0;
      for (int kb = warp; kb < nkb; kb += W, ++i) {
        const int o = kb * 32;
        const uint32_t a0 = *reinterpret_cast<const uint32_t*>(r0 + o);
        const uint32_t a2 = *reinterpret_cast<const uint32_t*>(r0 + o + 16);
        const uint32_t a1 = n > 8 ? *reinterpret_cast<const uint32_t*>(r1 + o) : 0u;
        const uint32_t a3 = n > 8 ? *reinterpret_cast<const uint32_t*>(r1 + o + 16) : 0u;
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(xp + o);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(xp + o + 16);
        if (MODE == 2 && (i & 1)) mma16816(acc[1], a0, a1, a2, a3, b0, b1);
        else mma16816(acc[0], a0, a1, a2, a3, b0, b1);
      }
      if (MODE == 2) {
        acc[0][0] += acc[1][0];
        acc[0][2] += acc[1][2];
      }
      if (c == 0) {  // column 0: rows g and g + 8
        zpart[warp * 16 + g] = acc[0][0];
        if (g + 8 < n) zpart[warp * 16 + g + 8] = acc[0][2];
      }
    }
    __syncthreads();
    if (t < n) {
      float s = 0.f;
      for (int w = 0; w < W; ++w) s += zpart[w * 16 + t];
      z = s;
    }
    __syncthreads();
  }
  const long long c1 = clock64();
  if (t < 16) out[blockIdx.x * 16 + t] = z;
  if (t == 0) cyc[blockIdx.x] = (c1 - c0) / 16;
}

static float bf2f(uint16_t v) {
  uint32_t u = (uint32_t)v << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main() {
  const int G = 148;
  const int shapes[3][2] = {{8, 6144}, {8, 4096}, {16, 4096}};
  for (auto& sh : shapes) {
    const int n = sh[0], d = sh[1];
    std::vector<uint16_t> hw((size_t)n * d), hx(d);
    uint32_t s = 12345;
    auto rnd = [&] { s = s * 1664525u + 1013904223u; return (uint16_t)(0x3c00 + (s >> 22) % 0x200 + ((s >> 10) & 1 ? 0x8000 : 0)); };
    for (auto& v : hw) v = rnd();
    for (auto& v : hx) v = rnd();
    std::vector<double> ref(n, 0.0);
    for (int e = 0; e < n; ++e)
      for (int i = 0; i < d; ++i) ref[e] += (double)bf2f(hw[(size_t)e * d + i]) * (double)bf2f(hx[i]);
    uint16_t *dw, *dx;
    float* dout;
    long long* dc;
    cudaMalloc(&dw, hw.size() * 2);
    cudaMalloc(&dx, hx.size() * 2);
    cudaMalloc(&dout, (size_t)G * 16 * 4);
    cudaMalloc(&dc, G * 8);
    cudaMemcpy(dw, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
    const int smem = 16 * (2 * d + 16) + 2 * d + W * 16 * 4;
    for (int mode = 0; mode < 5; ++mode) {
      if (mode == 3 && n > 8) continue;
      auto k = mode == 0 ? gemv<0> : mode == 1 ? gemv<1> : mode == 2 ? gemv<2> : mode == 3 ? gemv<3> : gemv<4>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k<<<G, T, smem>>>(dw, dx, d, n, dout, dc);
      k<<<G, T, smem>>>(dw, dx, d, n, dout, dc);
      std::vector<long long> c(G);
      std::vector<float> o((size_t)G * 16);
      cudaMemcpy(c.data(), dc, G * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
      std::sort(c.begin(), c.end());
      double err = 0.0, mx = 0.0;
      for (int e = 0; e < n; ++e) {
        err = std::max(err, std::fabs((double)o[e] - ref[e]));
        mx = std::max(mx, std::fabs(ref[e]));
      }
      printf("{\"n\": %d, \"d\": %d, \"mode\": %d, \"cycles_median\": %lld, \"rel_err\": %.3g, \"err\": \"%s\"}\n", n, d, mode,
             c[G / 2], err / mx, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(dw);
    cudaFree(dx);
    cudaFree(dout);
    cudaFree(dc);
  }
  return 0;
}
