// tcgen05 binary16 GEMM (fp32 accumulation in TMEM) for KP_ACCUM_TENSOR.
// Same operand / epilogue contract as gemm_f16ref (gemm_f16ref.cuh).
#pragma once

#include "gemm_f16ref.cuh"

namespace kp {
int gemm_f16tc_num_ctas(int M, int N);
void gemm_f16tc(const F16GemmArgs& a, int kernel_class);
}  // namespace kp
