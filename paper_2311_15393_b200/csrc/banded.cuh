// Banded-Toeplitz Kronecker-sum operator.
#pragma once

#include "common.cuh"
#include "gemm_f64.cuh"

namespace kp {

constexpr int BAND_MAX_TAPS = 64;   // padded tap count limit (multiple of 8)
constexpr int BAND_MAX_TERMS = 8;

// One direction of a correlation y(a) = sum_u w[k][u] x(a + shift + u),
// u in [0, taps); taps padded to a multiple of 8 with zeros at the end.
struct BandTaps {
  int taps = 0;   // padded to a multiple of 8 (shared-memory halo sizing)
  int real = 0;   // actual tap count (the correlation loops)
  int shift = 0;
  double w[BAND_MAX_TERMS][BAND_MAX_TAPS];
};

// Y_k = column correlation of X (n-by-n, column-major) for all r terms;
// Y holds r stacked n-by-n column-major blocks. batch > 1: `batch` images,
// X and Y of image z at z * n^2 and z * r * n^2.
void band_cols(const double* X, double* Y, int n, int r, const BandTaps& t, const int* status,
               int batch = 1);
// out = sum_k row correlation of Y_k, with the GEMM epilogue contract
// (F64Epilogue; C indexed column-major like out; batched images per
// F64Epilogue::img / part_img / addc_img).
void band_rows(const double* Y, int n, int r, const BandTaps& t, const F64Epilogue& e,
               const int* status, int batch = 1);
int band_rows_num_ctas(int n);
// Both passes in one kernel (short bands, where the two-pass form is HBM-
// bound): out = sum_k row-correlation(column-correlation(X)), epilogue as
// band_rows. Supported tap counts: band_fused_supported(); partial slots per
// image: band_fused_num_ctas(n).
bool band_fused_supported(int col_taps, int row_taps);
int band_fused_num_ctas(int n);
void band_fused(const double* X, int n, int r, const BandTaps& tc, const BandTaps& tr, const F64Epilogue& e,
                const int* status, int batch = 1);

}  // namespace kp
