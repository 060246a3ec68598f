// host_expert.h — host-CPU SwiGLU expert (miss handling of PAPER.md:199-201).
#pragma once
#include <stdint.h>

namespace moe {

class HostExpert {
 public:
  explicit HostExpert(int threads);  // <= 0: all hardware threads
  ~HostExpert();
  HostExpert(const HostExpert&) = delete;
  HostExpert& operator=(const HostExpert&) = delete;
  int threads() const;
  // blob: { W1[ffr][d], W3[ffr][d], W2[d][ffr] } bf16 (moe.h slot layout); x: bf16 [d];
  // o: fp32 [d] = W2 (silu(W1 x) * (W3 x)).
  void ffn(const uint16_t* blob, const uint16_t* x, int d, int ffr, float* o);

 private:
  struct Impl;
  Impl* impl_;
};

}  // namespace moe
