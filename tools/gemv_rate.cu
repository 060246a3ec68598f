// Gate-GEMV arithmetic rates on one SM (the decode kernel's routing prologue): 20 consumer
// warps, 16 gate rows x 4096 bf16 in shared memory, each thread one 16-B chunk of x and of
// every row, accumulated into even/odd fp32 lanes in the same order four ways:
//   0  fma.rn.f32.bf16 (mixed precision, SASS FHFMA.BF16)
//   1  bf16 -> fp32 by shift/mask, then fma.rn.f32x2 (FFMA2)
//   2  bf16 -> fp32 by shift/mask, then two FFMA
//   3  a third of the rows as 0, the rest as 1 (fma and alu pipes both busy)
// Prints SM cycles per pass (clock64, median CTA) and checks the four give identical bits.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gemv_rate tools/gemv_rate.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

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
__device__ __forceinline__ float2 ffma2(const float2 a, const float2 b, const float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
        "l"(*reinterpret_cast<const unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 bf2(uint32_t v) { return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xffff0000u)); }

template <int MODE>
__device__ __forceinline__ float2 dot8(const int4 w, const float2 (&xf)[4], const int4 x, float2 acc) {
  const uint32_t ww[4] = {(uint32_t)w.x, (uint32_t)w.y, (uint32_t)w.z, (uint32_t)w.w};
  const uint32_t xx[4] = {(uint32_t)x.x, (uint32_t)x.y, (uint32_t)x.z, (uint32_t)x.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (MODE == 0) acc = fma_bf16x2(ww[i], xx[i], acc);
    if (MODE == 1) acc = ffma2(bf2(ww[i]), xf[i], acc);
    if (MODE == 2) {
      const float2 wf = bf2(ww[i]);
      acc.x = fmaf(wf.x, xf[i].x, acc.x);
      acc.y = fmaf(wf.y, xf[i].y, acc.y);
    }
    if (MODE == 3) acc = ffma2(bf2(ww[i]), xf[i], acc);   // (mode 3 mixes: see the kernel)
  }
  return acc;
}

template <int MODE>
__global__ void __launch_bounds__(640, 1) gemv(const uint16_t* Wg, const uint16_t* x, int d, int n, float* out,
                                               long long* cyc) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int gstride = 2 * d + 16;
  for (int i = threadIdx.x; i < n * (d / 8); i += blockDim.x) {
    const int e = i / (d / 8), c = i % (d / 8);
    reinterpret_cast<int4*>(sm + (size_t)e * gstride)[c] = reinterpret_cast<const int4*>(Wg + (size_t)e * d)[c];
  }
  __syncthreads();
  const int t = threadIdx.x, nthr = blockDim.x, nch = d / 8;
  int4 xr = make_int4(0, 0, 0, 0);
  if (t < nch) xr = reinterpret_cast<const int4*>(x)[t];
  float2 xf[4] = {bf2(xr.x), bf2(xr.y), bf2(xr.z), bf2(xr.w)};
  float res = 0.f;
  __syncthreads();
  const long long c0 = clock64();
  for (int rep = 0; rep < 16; ++rep) {
    for (int e0 = 0; e0 < n; e0 += 8) {
      float2 acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = make_float2(0.f, 0.f);
      if (t < nch) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (e0 + j < n) {
            const int4 w = reinterpret_cast<const int4*>(sm + (size_t)(e0 + j) * gstride)[t];
            // mode 3: rows j % 3 == 0 on the mixed-precision FMA (fma pipe only), the others
            // converted on the ALU pipe and accumulated with packed FFMA2 (half the fma slots)
            if (MODE == 3) acc[j] = (j % 3 == 0) ? dot8<0>(w, xf, xr, acc[j]) : dot8<3>(w, xf, xr, acc[j]);
            else acc[j] = dot8<MODE>(w, xf, xr, acc[j]);
          }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) res += (acc[j].x + acc[j].y) * (rep == 0 ? 1.f : 0.f);
    }
    __syncthreads();
  }
  const long long c1 = clock64();
  out[blockIdx.x * nthr + t] = res;
  if (t == 0) cyc[blockIdx.x] = (c1 - c0) / 16;
}

int main() {
  const int d = 4096, n = 16, G = 148, T = 640;
  std::vector<uint16_t> hw((size_t)n * d), hx(d);
  uint32_t s = 12345;
  auto rnd = [&] { s = s * 1664525u + 1013904223u; return (uint16_t)(0x3c00 + (s >> 22) % 0x200 + ((s >> 10) & 1 ? 0x8000 : 0)); };
  for (auto& v : hw) v = rnd();
  for (auto& v : hx) v = rnd();
  uint16_t *dw, *dx;
  float* dout;
  long long* dc;
  cudaMalloc(&dw, hw.size() * 2);
  cudaMalloc(&dx, hx.size() * 2);
  cudaMalloc(&dout, (size_t)G * T * 4 * 4);
  cudaMalloc(&dc, G * 8);
  cudaMemcpy(dw, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  const int smem = n * (2 * d + 16);
  std::vector<float> outs[4];
  for (int mode = 0; mode < 4; ++mode) {
    auto k = mode == 0 ? gemv<0> : mode == 1 ? gemv<1> : mode == 2 ? gemv<2> : gemv<3>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<G, T, smem>>>(dw, dx, d, n, dout + (size_t)mode * G * T, dc);
    k<<<G, T, smem>>>(dw, dx, d, n, dout + (size_t)mode * G * T, dc);
    std::vector<long long> c(G);
    cudaMemcpy(c.data(), dc, G * 8, cudaMemcpyDeviceToHost);
    std::sort(c.begin(), c.end());
    outs[mode].resize((size_t)G * T);
    cudaMemcpy(outs[mode].data(), dout + (size_t)mode * G * T, (size_t)G * T * 4, cudaMemcpyDeviceToHost);
    printf("{\"mode\": %d, \"cycles_per_gemv_median\": %lld, \"err\": \"%s\"}\n", mode, c[G / 2],
           cudaGetErrorString(cudaGetLastError()));
  }
  const bool same = outs[0] == outs[1] && outs[0] == outs[2] && outs[0] == outs[3];
  printf("{\"bit_identical\": %s}\n", same ? "true" : "false");
  return 0;
}
