// expert_fused_mma.cu — the fused decode kernel with the gate GEMV's tensor-core form
// (gate_gemv.cuh: gate_mma_form, 9-16 experts), compiled from the same source as
// expert_fused.cu in a translation unit of its own (see there).
#define MOE_FUSED_MMA_GATE 1
#include "expert_fused.cu"
