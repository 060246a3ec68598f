// host_expert.cpp — host-CPU expert FFN for the paper's miss handling (PAPER.md:199-201,
// "offloads the intermediate state ... to the CPU side for expert computation",
// "CPU multithreading optimizations"). Used by the runtime in MOE_MISS_HOST_COMPUTE mode:
// while the missed expert's weights are post-fetched to the GPU cache, the host cores
// compute its output from the pinned backing store.
//
// Memory-bound on host DRAM (a Mixtral expert is 352 MB of bf16): AVX-512 BF16 dot
// products (vdpbf16ps: exact bf16 products, fp32 accumulation) for W1/W3 x, fp32 FMAs for
// W2 h, rows split over a small persistent thread pool. Scalar fallback without AVX-512.
#include <immintrin.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "host_expert.h"

namespace moe {
namespace {

inline float bf(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

// ---------------------------------------------------------------------------- kernels
float dot_bf16_scalar(const uint16_t* a, const uint16_t* b, int n) {
  float s = 0.f;
  for (int i = 0; i < n; ++i) s += bf(a[i]) * bf(b[i]);
  return s;
}

float dot_bf16_f32_scalar(const uint16_t* a, const float* h, int n) {
  float s = 0.f;
  for (int i = 0; i < n; ++i) s += bf(a[i]) * h[i];
  return s;
}

__attribute__((target("avx512f,avx512bw,avx512bf16"))) float dot_bf16_avx512(const uint16_t* a, const uint16_t* b,
                                                                              int n) {
  __m512 acc0 = _mm512_setzero_ps(), acc1 = _mm512_setzero_ps();
  int i = 0;
  for (; i + 64 <= n; i += 64) {
    const __m512i a0 = _mm512_loadu_si512(a + i), b0 = _mm512_loadu_si512(b + i);
    const __m512i a1 = _mm512_loadu_si512(a + i + 32), b1 = _mm512_loadu_si512(b + i + 32);
    acc0 = _mm512_dpbf16_ps(acc0, (__m512bh)a0, (__m512bh)b0);
    acc1 = _mm512_dpbf16_ps(acc1, (__m512bh)a1, (__m512bh)b1);
  }
  float s = _mm512_reduce_add_ps(_mm512_add_ps(acc0, acc1));
  for (; i < n; ++i) s += bf(a[i]) * bf(b[i]);
  return s;
}

__attribute__((target("avx512f,avx512bw"))) float dot_bf16_f32_avx512(const uint16_t* a, const float* h, int n) {
  __m512 acc0 = _mm512_setzero_ps(), acc1 = _mm512_setzero_ps();
  int i = 0;
  for (; i + 32 <= n; i += 32) {
    const __m512i w = _mm512_loadu_si512(a + i);                                // 32 bf16
    const __m512 lo = _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(_mm512_castsi512_si256(w)), 16));
    const __m512 hi =
        _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(_mm512_extracti64x4_epi64(w, 1)), 16));
    acc0 = _mm512_fmadd_ps(lo, _mm512_loadu_ps(h + i), acc0);
    acc1 = _mm512_fmadd_ps(hi, _mm512_loadu_ps(h + i + 16), acc1);
  }
  float s = _mm512_reduce_add_ps(_mm512_add_ps(acc0, acc1));
  for (; i < n; ++i) s += bf(a[i]) * h[i];
  return s;
}

bool have_avx512bf16() {
  static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                         __builtin_cpu_supports("avx512bf16");
  return ok;
}

// ---------------------------------------------------------------------------- thread pool
class Pool {
 public:
  explicit Pool(int n) : n_(std::max(1, n)) {
    for (int i = 1; i < n_; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++epoch_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return n_; }
  // Runs fn(lo, hi) over [0, total) in chunks; the calling thread participates.
  void run(int total, int chunk, const std::function<void(int, int)>& fn) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      total_ = total;
      chunk_ = chunk;
      next_.store(0);
      pending_ = n_ - 1;
      ++epoch_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void work() {
    while (true) {
      const int lo = next_.fetch_add(chunk_);
      if (lo >= total_) break;
      (*fn_)(lo, std::min(total_, lo + chunk_));
    }
  }
  void loop(int) {
    uint64_t seen = 0;
    while (true) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return epoch_ != seen; });
        seen = epoch_;
        if (stop_) return;
      }
      work();
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  int n_;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  uint64_t epoch_ = 0;
  bool stop_ = false;
  const std::function<void(int, int)>* fn_ = nullptr;
  int total_ = 0, chunk_ = 1;
  std::atomic<int> next_{0};
  int pending_ = 0;
};

}  // namespace

struct HostExpert::Impl {
  Pool pool;
  std::vector<float> h;
  explicit Impl(int threads) : pool(threads) {}
};

HostExpert::HostExpert(int threads) {
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  impl_ = new Impl(threads);
}

HostExpert::~HostExpert() { delete impl_; }

int HostExpert::threads() const { return impl_->pool.size(); }

// o[c] = sum_j W2[c][j] * silu(W1[j] . x) * (W3[j] . x)   (reading R4; fp32 accumulate)
void HostExpert::ffn(const uint16_t* blob, const uint16_t* x, int d, int ffr, float* o) {
  const uint16_t* W1 = blob;
  const uint16_t* W3 = blob + (size_t)ffr * d;
  const uint16_t* W2 = blob + 2 * (size_t)ffr * d;
  impl_->h.resize(ffr);
  float* h = impl_->h.data();
  const bool v = have_avx512bf16();
  impl_->pool.run(ffr, 64, [&](int lo, int hi) {
    for (int j = lo; j < hi; ++j) {
      const float g = v ? dot_bf16_avx512(W1 + (size_t)j * d, x, d) : dot_bf16_scalar(W1 + (size_t)j * d, x, d);
      const float u = v ? dot_bf16_avx512(W3 + (size_t)j * d, x, d) : dot_bf16_scalar(W3 + (size_t)j * d, x, d);
      h[j] = g / (1.0f + expf(-g)) * u;
    }
  });
  impl_->pool.run(d, 32, [&](int lo, int hi) {
    for (int c = lo; c < hi; ++c)
      o[c] = v ? dot_bf16_f32_avx512(W2 + (size_t)c * ffr, h, ffr) : dot_bf16_f32_scalar(W2 + (size_t)c * ffr, h, ffr);
  });
}

}  // namespace moe
