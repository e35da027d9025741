// FP64 GEMM on the DMMA tensor pipe (mma.sync.m16n8k16 f64) for the
// Kronecker-sum operator (kron.cpp:62-88) and FP64-format preconditioner.
#pragma once

#include "common.cuh"

namespace kp {

// K-major operand with "K batches": element (row, kk) with kk = b*Kb + k is at
// p[b*bstride + row*ld + k]. A plain K-major matrix has one batch.
struct F64Operand {
  const double* p = nullptr;
  long ld = 0;
  long bstride = 0;
};

// Fused epilogue. C(m,n) at C[m*cm + n*cn]; auxiliary vectors use
// (m*vm + n*vn). Per-CTA partial sums (deterministic order) go to
// partials[cta*4 + {0,1,2}]: 0: sum acc*d0 (or acc^2 if d0_self),
// 1: sum acc*(d1a - d1b), 2: count of non-finite outputs.
struct F64Epilogue {
  double* C = nullptr;
  long cm = 1, cn = 0;
  long vm = 1, vn = 0;
  const double* mul = nullptr;
  const double* addv = nullptr;
  double addc = 0.0;
  const double* d0 = nullptr;
  int d0_self = 0;
  const double* d1a = nullptr;
  const double* d1b = nullptr;
  int count_nonfinite = 0;
  double* partials = nullptr;
  // Batched banded operator (band_rows, grid.z = image): C and the vectors of
  // image z start at z * img, its partials at slot z * part_img, and the
  // addv coefficient is addc_img[z] when given (per-image lambda^2).
  long img = 0;
  int part_img = 0;
  const double* addc_img = nullptr;
};

struct F64GemmArgs {
  int M = 0, N = 0, nb = 1, Kb = 0;
  F64Operand A, B;
  F64Epilogue epi;
  const int* status = nullptr;  // kernel is a no-op when *status != 0
};

// Number of CTAs the launch will use (size of the partials array / 4).
int gemm_f64_num_ctas(int M, int N);
void gemm_f64(const F64GemmArgs& a, int kernel_class);

}  // namespace kp
