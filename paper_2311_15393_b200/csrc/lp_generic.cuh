// Emulated low-precision arithmetic for ANY PrecisionFormat (t, emax,
// subnormals) on the device: round_value (precision.cpp:15-41,82-86) and the
// lp_matmul tree (lpblas.cpp:13-70) computed per output element in FP64 with
// the format's rounding after every product and every pairwise sum.
//
// fp16 preconditioners run on the f16x2 GEMM (gemm_f16ref); this module is
// the exact path for every other format (bfloat16, fp32, custom, and the
// unrounded FP64 tree), and for lp_matmul calls on inputs that are not
// binary16-representable.
#pragma once

#include "common.cuh"

namespace kp {

struct LpFormat {
  int t = 53, emax = 1023, sub = 1;
  __host__ __device__ bool covers_double() const { return t >= 53 && emax >= 1023 && sub; }
};

// out[i] = round_value(x[i], f) (device pointers; in place allowed).
void lp_round_array(const double* x, size_t count, LpFormat f, double* out, int kernel_class);

// C(i,j) = tree over k of round(A(i,k) * B(k,j)), each pairwise sum rounded
// (no rounding at all when f covers double). A(i,k) = a[i*ai + k*ak],
// B(k,j) = b[k*bk + j*bj], C(i,j) = c[i + j*ldc]. With `scale`, the stored
// value is round(scale[i + j*ls] * C(i,j)) (the preconditioner's S .* t2).
struct LpGemmArgs {
  int M = 0, N = 0, K = 0;
  const double* a = nullptr;
  long ai = 1, ak = 0;
  const double* b = nullptr;
  long bk = 1, bj = 0;
  double* c = nullptr;
  long ldc = 0;
  const double* scale = nullptr;
  long ls = 0;
  LpFormat f;
  bool round_leaves = true;  // false: leaves are pre-rounded addends (pairwise_sum)
  const int* status = nullptr;
};
void lp_gemm_generic(const LpGemmArgs& g, int kernel_class);

// Fixed-grid partial sums over z (n*n): part[cta*4 + q], q = 0: z.d0,
// 1: z.(d1a - d1b) (d1b optional), 2: #non-finite z. LP_PART_CTAS CTAs.
constexpr int LP_PART_CTAS = 296;
void lp_vector_partials(const double* z, size_t count, const double* d0, const double* d1a,
                        const double* d1b, double* part, const int* status, int kernel_class);

// Number of entries of x (device, count) that are not exactly representable
// in binary16 (NaN counts as not representable).
long long count_not_f16(const double* x, size_t count);

// dst[r*ld + c] = half(src[r*rs + c*cs]) for r < rows, c < cols; columns
// [cols, ld) filled with `pad` (0x8000 = -0 for A operands, 0 for B).
void pack_f16(const double* src, long rs, long cs, int rows, int cols, __half* dst, long ld,
              uint16_t pad);

}  // namespace kp
