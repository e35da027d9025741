// Reference-exact binary16 matrix product: the device form of lp_matmul
// (lpblas.cpp:13-70) for fmt = fp16.
#pragma once

#include "common.cuh"

namespace kp {

// K-major binary16 operand: element (row, k) at p[row*ld + k]. Requirements
// (all internal buffers satisfy them): ld % 64 == 0, ld >= K, 16-byte aligned,
// and the padding columns k in [K, ld) hold -0 for A and +0 for B, so every
// padded product is exactly -0 — a neutral element of the pairwise tree.
struct F16Operand {
  const __half* p = nullptr;
  long ld = 0;
};

enum F16OutMode { F16OUT_HALF = 0, F16OUT_HALF_SCALED = 1, F16OUT_F64 = 2 };

struct F16Epilogue {
  int mode = F16OUT_HALF;
  __half* Ch = nullptr;  // F16OUT_HALF[_SCALED]: Ch[m*cm + n*cn]
  double* Cd = nullptr;  // F16OUT_F64:           Cd[m*cm + n*cn]
  long cm = 1, cn = 0;
  const __half* scale = nullptr;  // HALF_SCALED: out = round16(scale(m,n) * acc)
  long sm = 1, sn = 0;
  // F64 partials (vectors indexed m*vm + n*vn), per CTA at partials[cta*4+q]:
  // 0: sum out*d0, 1: sum out*(d1a - d1b) (d1b optional), 2: #non-finite.
  long vm = 1, vn = 0;
  const double* d0 = nullptr;
  const double* d1a = nullptr;
  const double* d1b = nullptr;
  double* partials = nullptr;
  // Batched products: N stacks independent images of n_img columns each (the
  // B operand holds their rows back to back). Output column n = img * n_img
  // + nl is addressed as image img's column nl: C at img * c_img + m*cm +
  // nl*cn, the scale at img * s_img + ..., the dot vectors at img * v_img +
  // ..., and partials per image in slots [img * part_img, (img+1) * part_img)
  // (fixed-order per-image reductions). n_img must be a multiple of the tile
  // width (64), so no tile straddles two images. n_img = 0: one product.
  int n_img = 0;
  long c_img = 0, s_img = 0, v_img = 0;
  int part_img = 0;
  // gemm_f16tc only: the images stacked along M instead (the A operand holds
  // their rows back to back; m_img rows each, a multiple of 128); same
  // per-image offsets c_img / s_img. Binary16 outputs only.
  int m_img = 0;
};

// Image index and image-local column of global output column n.
__host__ __device__ __forceinline__ int epi_image(const F16Epilogue& e, int n, int& nl) {
  if (!e.n_img) {
    nl = n;
    return 0;
  }
  const int img = n / e.n_img;
  nl = n - img * e.n_img;
  return img;
}

struct F16GemmArgs {
  int M = 0, N = 0, K = 0;
  F16Operand A, B;  // C(m,n) = tree_k round16(A(m,k) * B(n,k))
  F16Epilogue epi;
  const int* status = nullptr;
  // gemm_f16x only: zero-sign fix-up workspace, f16x_zfix_words(M, N) + 2
  // unsigned words with [0] = [1] = 0 ([0] listed outputs, [1] fix-up
  // completion counter, [2..] the list); every launch leaves [0] = [1] = 0.
  unsigned* zfix = nullptr;
  // gemm_f16x only: row sign hashes of A (M words; computed by the call unless
  // hash_a_ready) and B (N words, computed by the call), and their target sum.
  unsigned long long* hash_a = nullptr;
  bool hash_a_ready = false;
  unsigned long long* hash_b = nullptr;
  unsigned long long hsum = 0;
};

int gemm_f16ref_num_ctas(int M, int N);
// Batched products: partial slots per image (F16Epilogue::part_img).
int gemm_f16ref_partials_per_image(int M, int N, int n_img);
void gemm_f16ref(const F16GemmArgs& a, int kernel_class);
// Fill helper for padded binary16 buffers (bits = 0x8000 for -0, 0 for +0).
void fill_u16(__half* p, size_t count, uint16_t bits);

}  // namespace kp
